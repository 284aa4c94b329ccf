#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_demo_golden_gpu.py tests/test_files.py tests/test_bandpass.py -q -x -p no:cacheprovider > gpurun_out/r02t_fp.log 2>&1
echo "fp rc=$?" >> gpurun_out/r02t_fp.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02t_bench.log 2> gpurun_out/r02t_bench.err
echo "bench rc=$?" >> gpurun_out/r02t_bench.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02t_ref.log 2> gpurun_out/r02t_ref.err
echo "ref rc=$?" >> gpurun_out/r02t_ref.err
