#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python tools/c4_frames.py 2 --lagged-friction --max-newton 400 --out gpurun_out/c4_frames_lagged.json > gpurun_out/c4_frames_lagged.log 2>&1
echo done
