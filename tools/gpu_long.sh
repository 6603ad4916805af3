#!/bin/bash
# long runs: ablations (C1 frames, C4 first Newton iterations), C4 whole frames (chi=0, chi=0.3)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out profiles
timeout 600 python tools/ablation.py c1 10 > gpurun_out/ablation_c1.log 2>&1
timeout 900 python tools/ablation.py c4 20 > gpurun_out/ablation_c4.log 2>&1
timeout 900 python tools/c4_frames.py 1 --chi 0.0 --out gpurun_out/c4_frames_chi0.json > gpurun_out/c4_frames_chi0.log 2>&1
timeout 1500 python tools/c4_frames.py 1 --max-newton 300 --out gpurun_out/c4_frames.json > gpurun_out/c4_frames.log 2>&1
echo done
