#!/bin/bash
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
  timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants4.log 2>&1
  BAL_TS_CONTACT_INLINE=1 timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants4.log 2>&1
done
timeout 1800 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_gpu_c2c3.py tests/test_gpu_additive.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_sep.log 2>&1; echo rc=$? >> gpurun_out/pytest_sep.log
grep "^{" gpurun_out/variants4.log | cut -c1-330; tail -3 gpurun_out/pytest_sep.log
