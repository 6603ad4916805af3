#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_c2c3.py -v --durations=0 > gpurun_out/pytest_c2c3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c2c3.log
timeout 900 bash tools/spmv_variants.sh
echo done
