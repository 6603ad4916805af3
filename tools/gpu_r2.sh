#!/bin/bash
# round-2 verification: GPU tests, bench, ncu (launch list of a short bench + full capture of the SpMV
# and the PCG update on the C4 first Newton system)
mkdir -p gpurun_out
T=${PYTEST_TARGETS:-tests}
if [ -z "$NO_TESTS" ]; then
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest $T -m gpu -q -p no:cacheprovider ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_LAUNCHES:-3000} --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
NCU_OUT=ncu_r02 bash tools/gpu_ncu_spmv.sh
fi
tail -5 gpurun_out/pytest_gpu.log 2>/dev/null; tail -2 gpurun_out/bench.log 2>/dev/null | cut -c1-1500
