#!/bin/bash
# Round-2 GPU passes (one B200 via gpurun), in the order the profiles/ files were produced.
#   bash tools/gpu_round2.sh tests|bench|ncu|variants|ablation|rods|frames
# tests    : the full -m gpu suite and smoke()                          -> gpurun_out/pytest_gpu.log, smoke.log
# bench    : python bench.py (+ --fp32-matrix) and the ncu launch list   -> bench*.log, launches.csv
# ncu      : ncu --set full of k_spmv_ts on the bench system            -> ncu_settled.ncu-rep (profiles/ncu_r02_*)
# variants : SpMV variants (BAL_LIB_PATH=variants/libbal_*.so builds with BAL_NVCC_EXTRA=-D...; BAL_FLAGS;
#            BAL_TS_* env switches) on the contact-rich and drop C4 systems -> variants.log (profiles/spmv_variants_r02.md)
# ablation : NEXT-1 / NEXT-3 / NEXT-4 variants on C2 (10 frames) and C3 (3 frames) -> profiles/ablation_r02.md
# rods     : NEXT-2 twisting rods frames and the stall diagnosis           -> profiles/rods_r02.md
# frames   : whole C4 frames at the paper's chi = 0.3 (tools/gpu_frames.sh) -> profiles/c4-drop_frames_*.json
mkdir -p gpurun_out
case "$1" in
  tests)
    timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
    timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log ;;
  bench)
    timeout 900 python bench.py > gpurun_out/bench.log 2>&1
    timeout 900 python bench.py --fp32-matrix --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1 ;;
  ncu)
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_ts -c 1 \
      -o gpurun_out/ncu_settled -f python tools/prof_spmv_settled.py > gpurun_out/ncu_settled.log 2>&1 ;;
  variants)
    for cfg in c4 c4-drop; do
      for L in paper_2407_00046_b200/libbal.so variants/libbal_*.so; do
        [ -f "$L" ] && BAL_LIB_PATH=$L timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants.log 2>&1
      done
      BAL_FLAGS=256 timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants.log 2>&1
    done ;;
  ablation)
    timeout 1500 python tools/ablation.py c2 10 > gpurun_out/ablation_c2.log 2>&1
    timeout 1500 python tools/ablation.py c3 3 > gpurun_out/ablation_c3.log 2>&1
    timeout 1500 python tools/probe_as_c4.py 3 > gpurun_out/probe_as_c4.log 2>&1 ;;
  rods)
    timeout 1500 python tools/rods_frames.py 90 1200 gpurun_out/rods_frames.json > gpurun_out/rods_frames.log 2>&1
    BAL_FLAGS=16 timeout 1500 python tools/rods_frames.py 150 1300 gpurun_out/rods_frames_sigmamin.json > gpurun_out/rods_frames_sm.log 2>&1
    timeout 600 python tools/rods_diag.py 24 400 25 0 > gpurun_out/rods_diag0.log 2>&1
    BAL_LS_ROUND=0 timeout 600 python tools/rods_diag.py 24 400 25 0 > gpurun_out/rods_diag_ls0.log 2>&1 ;;
  frames)
    FRAME_TIMEOUT=3300 bash tools/gpu_frames.sh "c4-drop_frames_r02b_chi0.3 6 --scene c4" ;;
esac
