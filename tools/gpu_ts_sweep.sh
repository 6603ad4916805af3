#!/bin/bash
# SpMV tile-budget sweep on the C4 first Newton system + ncu of the default configuration
mkdir -p gpurun_out
for b in ${BUDGETS:-0}; do
  echo "== budget $b" >> gpurun_out/sweep.log
  BAL_TS_BUDGET=$b BAL_VERBOSE=1 timeout 300 python tools/prof_spmv.py 2>&1 | grep -v "^\[bal-pcg\]" >> gpurun_out/sweep.log
done
if [ -z "$NO_NCU" ]; then bash tools/gpu_ncu_spmv.sh; fi
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
grep -h "budget\|bal-ts\|bench spmv\|iters" gpurun_out/sweep.log
