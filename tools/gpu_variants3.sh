#!/bin/bash
mkdir -p gpurun_out
for cfg in c4 c4-drop; do
for L in paper_2407_00046_b200/libbal.so variants/libbal_m3.so variants/libbal_m4.so variants/libbal_c128m4.so; do
  BAL_LIB_PATH=$L timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants3.log 2>&1
done
done
timeout 1500 python tools/probe_as_c4.py 3 > gpurun_out/probe_as_c4.log 2>&1
grep "^{" gpurun_out/variants3.log | cut -c1-330; cat gpurun_out/probe_as_c4.log | cut -c1-400
