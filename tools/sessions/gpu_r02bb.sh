#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/fp_time.py > gpurun_out/r02bb_fp.log 2>&1
echo "rc=$?" >> gpurun_out/r02bb_fp.log
timeout 900 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_capi_fingerprint_gpu.py tests/test_demo_golden_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02bb_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02bb_pytest.log
timeout 1500 python tools/cfg4_run.py > gpurun_out/r02bb_cfg4.log 2>&1
echo "cfg4 rc=$?" >> gpurun_out/r02bb_cfg4.log
