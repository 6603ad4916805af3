#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/spmv_modes.log
for m in sym full staged; do
  echo "$m: $(BAL_SPMV=$m timeout 300 python tools/prof_spmv.py 2>&1 | grep 'bench spmv')" >> gpurun_out/spmv_modes.log
done
BAL_SPMV=staged timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_staged.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_staged.log
BAL_SPMV=staged timeout 600 ncu --set full --clock-control none -k regex:k_spmv -s 20 -c 1 -o gpurun_out/spmv_staged -f python tools/prof_spmv.py > gpurun_out/ncu_staged.log 2>&1
BAL_SPMV=staged timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_staged.log 2>&1
echo done
