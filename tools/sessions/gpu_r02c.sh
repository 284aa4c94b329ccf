#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_capi_search_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02c_capi.log 2>&1
echo "capi rc=$?" >> gpurun_out/r02c_capi.log
QS_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --fingerprints 400000 --no-fingerprint --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/r02c_spawn.log 2> gpurun_out/r02c_spawn.err
echo "spawn rc=$?" >> gpurun_out/r02c_spawn.err
timeout 2400 python tools/cpu_scaling.py > gpurun_out/r02c_cpu_scaling.log 2>&1
echo "cpu rc=$?" >> gpurun_out/r02c_cpu_scaling.log
