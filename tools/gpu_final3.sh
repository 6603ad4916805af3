#!/bin/bash
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
  timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants5.log 2>&1
  BAL_LIB_PATH=variants/libbal_cearly.so timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants5.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_final3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final3.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_final3.log 2>&1
grep "^{" gpurun_out/variants5.log | cut -c1-330; tail -2 gpurun_out/bench_final3.log | cut -c1-400
