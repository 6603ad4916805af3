#!/bin/bash
# artifacts for profiles/: GPU tests, smoke, bench (both arms), ncu k_spmv full + launch list of one bench step
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 20 -c 1 -o gpurun_out/spmv_sym -f python tools/prof_spmv.py > gpurun_out/ncu_sym.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_pcg_update_fused" -s 5 -c 1 -o gpurun_out/upd_full -f python tools/prof_spmv.py > gpurun_out/ncu_upd.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 25000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
