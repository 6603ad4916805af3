#!/bin/bash
# ncu --set full of the SpMV / PCG kernels on the C4 first Newton system (tools/prof_spmv.py)
mkdir -p gpurun_out
BAL_VERBOSE=1 python tools/prof_spmv.py > gpurun_out/prof_spmv.log 2>&1
K=${NCU_K:-"regex:k_spmv_ts|k_cg_update"}
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -s ${NCU_S:-6} -c ${NCU_C:-3} \
  -o gpurun_out/${NCU_OUT:-ncu_ts} -f python tools/prof_spmv.py > gpurun_out/ncu_run.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_run.log
tail -3 gpurun_out/prof_spmv.log; tail -3 gpurun_out/ncu_run.log
