#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rods.py tests/test_gpu_criteria.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_rods.log 2>&1; echo rc=$? >> gpurun_out/pytest_rods.log
timeout 1500 python tools/rods_frames.py 90 1200 gpurun_out/rods_frames.json > gpurun_out/rods_frames.log 2>&1
tail -3 gpurun_out/pytest_rods.log; tail -4 gpurun_out/rods_frames.log | cut -c1-400
