#!/bin/bash
# SpMV A/B + ncu of k_spmv, bench (C4 default), ncu launch list of one bench step
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/prof_spmv.py > gpurun_out/spmv_sym.log 2>&1
BAL_SPMV_FULL=1 timeout 300 python tools/prof_spmv.py > gpurun_out/spmv_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 20 -c 1 -o gpurun_out/spmv_sym -f python tools/prof_spmv.py > gpurun_out/ncu_sym.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
