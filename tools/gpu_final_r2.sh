#!/bin/bash
# round-2 measurement pass on the final tree: bench line, launch list of a short bench, ncu --set full
# of k_spmv_ts on the bench system, NEXT-1 ablations (incl. App. A additive preconditioner) on C2 / C3
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_LAUNCHES:-3000} --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_ts -c 1 \
  -o gpurun_out/ncu_final_settled -f python tools/prof_spmv_settled.py > gpurun_out/ncu_settled_final.log 2>&1
if [ -z "$NO_ABL" ]; then
timeout 900 python tools/ablation.py c2 10 > gpurun_out/ablation_c2_final.log 2>&1
timeout 1200 python tools/ablation.py c3 3 > gpurun_out/ablation_c3_final.log 2>&1
fi
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_7.log 2>&1; echo rc=$? >> gpurun_out/pytest_7.log
tail -2 gpurun_out/bench_final.log | cut -c1-600; tail -2 gpurun_out/ncu_settled_final.log; tail -3 gpurun_out/pytest_7.log
