#!/bin/bash
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
for L in paper_2407_00046_b200/libbal.so variants/libbal_vec.so variants/libbal_split.so variants/libbal_both.so; do
  BAL_LIB_PATH=$L timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants2.log 2>&1
done
BAL_LIB_PATH=variants/libbal_both_timing.so timeout 300 python tools/spmv_variants.py $cfg > gpurun_out/timing2_$cfg.log 2>&1
done
BAL_LIB_PATH=variants/libbal_both.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py tests/test_gpu_step.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_5.log 2>&1; echo rc=$? >> gpurun_out/pytest_5.log
grep "^{" gpurun_out/variants2.log | cut -c1-300; grep -h "ts-timing" gpurun_out/timing2_*.log | tail -4; tail -3 gpurun_out/pytest_5.log
