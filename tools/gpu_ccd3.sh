#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_parity.py tests/test_gpu_c2c3.py -q -x > gpurun_out/pytest_ccd3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ccd3.log
timeout 600 python tools/c4_frames.py 3 --scene c2 --max-newton 200 --out gpurun_out/c2_frames.json > gpurun_out/c2_frames.log 2>&1
echo done
