#!/bin/bash
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
  timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants6.log 2>&1
  BAL_LIB_PATH=variants/libbal_split2.so timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants6.log 2>&1
  timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants6.log 2>&1
  BAL_LIB_PATH=variants/libbal_split2.so timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants6.log 2>&1
done
grep "^{" gpurun_out/variants6.log | cut -c1-330
