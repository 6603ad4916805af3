#!/bin/bash
# final-tree verification: full GPU suite, smoke, bench line, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final2.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_final2.log 2>&1
tail -3 gpurun_out/pytest_final.log; tail -2 gpurun_out/smoke_final.log; tail -2 gpurun_out/bench_final2.log | cut -c1-400
