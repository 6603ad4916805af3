#!/bin/bash
# A/B of the SpMV tile geometry: rebuild with -D overrides on the GPU box, time tools/prof_spmv.py
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/spmv_variants.log
for v in "128 16 16 320" "64 32 8 160" "256 8 32 640" "64 24 8 160" "128 12 16 320"; do
  set -- $v
  export BAL_NVCC_EXTRA="-DBAL_SPMV_THREADS=$1 -DBAL_SPMV_MINBLOCKS=$2 -DBAL_SPMV_TILE_ROWS=$3 -DBAL_SPMV_TILE_CAP=$4"
  rm -f paper_2407_00046_b200/build/k_linalg.o
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed $v" >> gpurun_out/spmv_variants.log; continue; }
  echo "variant threads=$1 minblocks=$2 rows=$3 cap=$4: $(timeout 300 python tools/prof_spmv.py 2>&1 | grep 'bench spmv')" >> gpurun_out/spmv_variants.log
done
unset BAL_NVCC_EXTRA
rm -f paper_2407_00046_b200/build/k_linalg.o
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo done >> gpurun_out/spmv_variants.log
