#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_demo_golden_gpu.py tests/test_capi_fingerprint_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02al_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02al_pytest.log
timeout 900 python tools/stress_fingerprint.py 40 > gpurun_out/r02al_stress.log 2>&1
echo "rc=$?" >> gpurun_out/r02al_stress.log
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:"^k_" --clock-control none --csv --log-file gpurun_out/r02al_fp_launches.csv python tools/prof_fp_cfg2.py > gpurun_out/r02al_ncu.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --full-steps 0 > gpurun_out/r02al_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r02al_bench.log
