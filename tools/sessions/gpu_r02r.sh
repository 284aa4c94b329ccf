#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_capi_fingerprint_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02r_fp.log 2>&1
echo "fp rc=$?" >> gpurun_out/r02r_fp.log
B='python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --full-steps 0 --fingerprints 1000000'
timeout 900 $B > gpurun_out/r02r_bench.log 2>&1
QS_MAD_SELECT=radix timeout 900 $B > gpurun_out/r02r_bench_radixmad.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_fp.py > gpurun_out/r02r_launches.csv 2> gpurun_out/r02r_launches.err
timeout 1800 python tools/cfg3_run.py > gpurun_out/r02r_cfg3.log 2>&1; echo "cfg3 rc=$?" >> gpurun_out/r02r_cfg3.log
timeout 600 python tools/pair_table_bench.py 30 4e9 > gpurun_out/r02r_pairtable.log 2>&1
