#!/bin/bash
# round-2 follow-up: SpMV producer/consumer cycle breakdown (BAL_TS_TIMING build), partitioned-path
# and parity tests
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
  BAL_LIB_PATH=variants/libbal_timing.so timeout 300 python tools/spmv_variants.py $cfg > gpurun_out/timing_$cfg.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_step.py tests/test_gpu_parity.py tests/test_gpu_degenerate.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_4.log 2>&1; echo rc=$? >> gpurun_out/pytest_4.log
grep "ts-timing" gpurun_out/timing_c4.log | tail -2; grep "ts-timing" gpurun_out/timing_c4-drop.log | tail -2; tail -3 gpurun_out/pytest_4.log
