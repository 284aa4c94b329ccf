#!/bin/bash
# small-bucket kernel: parity (search tests + randomised sweep), class timings, QS_SMALL=0 A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py tests/test_sharded_gpu.py tests/test_buckets_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02an_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02an_pytest.log
timeout 900 python tools/stress_parity.py 150 > gpurun_out/r02an_stress.log 2>&1
echo "rc=$?" >> gpurun_out/r02an_stress.log
timeout 900 python tools/pair_classes.py 8000000 matched,distinct > gpurun_out/r02an_classes.log 2>&1
echo "rc=$?" >> gpurun_out/r02an_classes.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint > gpurun_out/r02an_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r02an_bench.log
