#!/bin/bash
# session-e baseline: full -m gpu suite, smoke, default bench (both arms)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02ba_smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02ba_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02ba_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ba_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02ba_smoke.log
timeout 900 python bench.py > gpurun_out/r02ba_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r02ba_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r02ba_bench_ref.log 2>&1
echo "rc=$?" >> gpurun_out/r02ba_bench_ref.log
