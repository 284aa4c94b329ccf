#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/fp_time.py > gpurun_out/r02be_fp.log 2>&1
echo "rc=$?" >> gpurun_out/r02be_fp.log
timeout 900 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_capi_fingerprint_gpu.py tests/test_demo_golden_gpu.py -q -x -s -p no:cacheprovider > gpurun_out/r02be_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02be_pytest.log
timeout 900 python tools/stress_fingerprint.py 40 > gpurun_out/r02be_stress_fp.log 2>&1
echo "rc=$?" >> gpurun_out/r02be_stress_fp.log
