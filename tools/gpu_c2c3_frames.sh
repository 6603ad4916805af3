#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python tools/c4_frames.py 2 --scene c3 --max-newton 300 --out gpurun_out/c3_frames.json > gpurun_out/c3_frames.log 2>&1
timeout 900 python tools/c4_frames.py 3 --scene c2 --max-newton 200 --out gpurun_out/c2_frames.json > gpurun_out/c2_frames.log 2>&1
timeout 600 python tools/c4_frames.py 3 --scene c2 --lagged-friction --max-newton 200 --out gpurun_out/c2_frames_lagged.json > gpurun_out/c2_frames_lagged.log 2>&1
echo done
