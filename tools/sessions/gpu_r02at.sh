#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py tests/test_sharded_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02at_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02at_pytest.log
timeout 900 python tools/stress_parity.py 150 > gpurun_out/r02at_stress.log 2>&1
echo "rc=$?" >> gpurun_out/r02at_stress.log
for sp in 4 8 12 16 32; do
  QS_CORE_SPLIT=$sp timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 0 > gpurun_out/r02at_bench_$sp.log 2>&1
done
