#!/bin/bash
# round-2: new bench (both arms), tightened fingerprint tests, spawn path, 4e5 parity
cd "$GRAFT_REPO_ROOT"
(free -g; nproc; lscpu | head -20) > gpurun_out/r02b_host.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02b_bench.log 2> gpurun_out/r02b_bench.err
echo "bench rc=$?" >> gpurun_out/r02b_bench.err
timeout 600 python -m pytest tests/test_fingerprint_gpu.py -q -s -p no:cacheprovider > gpurun_out/r02b_fp.log 2>&1
echo "fp rc=$?" >> gpurun_out/r02b_fp.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 2 > gpurun_out/r02b_ref.log 2> gpurun_out/r02b_ref.err
echo "ref rc=$?" >> gpurun_out/r02b_ref.err
QS_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --fingerprints 400000 --no-fingerprint --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/r02b_spawn.log 2> gpurun_out/r02b_spawn.err
echo "spawn rc=$?" >> gpurun_out/r02b_spawn.err
timeout 1200 python tools/parity_cfg1.py 400000 > gpurun_out/r02b_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r02b_parity.log
