#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_capi_fingerprint_gpu.py tests/test_demo_golden_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02q_fp.log 2>&1
echo "fp rc=$?" >> gpurun_out/r02q_fp.log
B='python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --full-steps 0 --fingerprints 1000000'
for k in cta32; do QS_WIN_KERNEL=$k timeout 900 $B > gpurun_out/r02q_bench_$k.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_fp.py > gpurun_out/r02q_launches.csv 2> gpurun_out/r02q_launches.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win_cta --launch-skip 1 -c 1 -o gpurun_out/r02q_wincta python tools/prof_fp.py > gpurun_out/r02q_ncu.log 2>&1
