mkdir -p gpurun_out
for cfg in c4 c4-drop; do
for L in paper_2407_00046_b200/libbal.so variants/libbal_s3.so variants/libbal_sb2.so; do
  BAL_LIB_PATH=$L timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants.log 2>&1
done
BAL_TS_NO_CPREFETCH=1 timeout 300 python tools/spmv_variants.py $cfg >> gpurun_out/variants.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_degenerate.py tests/test_gpu_step.py tests/test_gpu_c4.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_3.log 2>&1; echo rc=$? >> gpurun_out/pytest_3.log
grep "^{" gpurun_out/variants.log | cut -c1-400; tail -3 gpurun_out/pytest_3.log
