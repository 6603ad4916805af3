#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python tools/c4_frames.py 3 --chi 0.0 --out gpurun_out/c4_frames_chi0_3f.json > gpurun_out/c4_frames_chi0_3f.log 2>&1
timeout 2400 python tools/c4_frames.py 1 --out gpurun_out/c4_frames_1000.json > gpurun_out/c4_frames_1000.log 2>&1
echo done
