#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_gpu_c4.py -q -x > gpurun_out/pytest_fuse4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fuse4.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_fuse4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_pcg_update_fused" -s 5 -c 1 -o gpurun_out/upd4_full -f python tools/prof_spmv.py > gpurun_out/ncu_upd4.log 2>&1
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
echo done
