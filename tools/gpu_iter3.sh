#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/prof_spmv.py > gpurun_out/spmv_sym.log 2>&1
BAL_SPMV_V1=1 timeout 300 python tools/prof_spmv.py > gpurun_out/spmv_v1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 20 -c 1 -o gpurun_out/spmv_sym -f python tools/prof_spmv.py > gpurun_out/ncu_sym.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
echo done
