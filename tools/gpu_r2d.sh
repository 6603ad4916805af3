#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all2.log 2>&1; echo rc=$? >> gpurun_out/pytest_all2.log
BAL_ABL_ONLY="bal+warmstart,criterion" timeout 1500 python tools/ablation.py c2 10 > gpurun_out/ablation_c2_crit.log 2>&1
BAL_ABL_ONLY="bal+warmstart,criterion" timeout 1500 python tools/ablation.py c3 3 > gpurun_out/ablation_c3_crit.log 2>&1
tail -3 gpurun_out/pytest_all2.log; cat gpurun_out/ablation_c2_crit.log gpurun_out/ablation_c3_crit.log | cut -c1-250
