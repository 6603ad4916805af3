#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
BAL_PCG_UNFUSED=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_unfused.log 2>&1
echo done
