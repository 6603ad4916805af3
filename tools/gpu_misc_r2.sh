#!/bin/bash
# ncu of the SpMV on the bench workload (traffic per launch) + NEXT-1 ablations on C2 / C3 frames
mkdir -p gpurun_out
python tools/prof_spmv_settled.py > gpurun_out/prof_settled.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_ts -c 1 \
  -o gpurun_out/ncu_r02_settled -f python tools/prof_spmv_settled.py > gpurun_out/ncu_settled.log 2>&1
timeout 900 python tools/ablation.py c2 10 > gpurun_out/ablation_c2.log 2>&1
timeout 1200 python tools/ablation.py c3 3 > gpurun_out/ablation_c3.log 2>&1
tail -3 gpurun_out/prof_settled.log; tail -2 gpurun_out/ncu_settled.log; cat gpurun_out/ablation_c2.log gpurun_out/ablation_c3.log | cut -c1-300
