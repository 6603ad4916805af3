#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/verify_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/verify_smoke.log
timeout 900 python bench.py > gpurun_out/verify_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/verify_bench.log
echo done
