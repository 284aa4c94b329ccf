#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py tests/test_minmax_gpu.py tests/test_fingerprint_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02i_lsh.log 2>&1
echo "lsh rc=$?" >> gpurun_out/r02i_lsh.log
B='python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fingerprint --no-e2e --full-steps 1'
timeout 600 $B > gpurun_out/r02i_bench.log 2>&1
timeout 900 python tools/stress_parity.py 60 > gpurun_out/r02i_stress.log 2>&1
