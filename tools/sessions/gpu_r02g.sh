#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_buckets_gpu.py tests/test_capi_fingerprint_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02g_buckets.log 2>&1
echo "buckets rc=$?" >> gpurun_out/r02g_buckets.log
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py tests/test_sharded_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02g_lsh.log 2>&1
echo "lsh rc=$?" >> gpurun_out/r02g_lsh.log
B='python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fingerprint --no-e2e --full-steps 0'
timeout 600 $B > gpurun_out/r02g_bench_bins.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bb_|k_rs_" -c 9 python tools/one_search.py > gpurun_out/r02g_ncu_bb.log 2>&1
