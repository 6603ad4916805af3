#!/bin/bash
# NEXT-3 FP32 storage measurements + the full GPU suite and smoke on the final tree
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
  BAL_FLAGS=256 timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/fp32.log 2>&1
done
timeout 900 python bench.py --fp32-matrix --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1
timeout 900 python tools/ablation.py c2 10 > gpurun_out/ablation_c2_fp32.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
grep "^{" gpurun_out/fp32.log | cut -c1-300; tail -1 gpurun_out/bench_fp32.log | cut -c1-300; tail -3 gpurun_out/pytest_all.log; tail -2 gpurun_out/smoke.log
