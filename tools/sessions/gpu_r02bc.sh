#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
( QS_STFT_KERNEL=fma timeout 300 python tools/stft_ab.py fma; timeout 300 python tools/stft_ab.py mma; python tools/stft_ab.py cmp ) > gpurun_out/r02bc_stft.log 2>&1
timeout 600 python tools/fp_time.py > gpurun_out/r02bc_fp.log 2>&1
echo "rc=$?" >> gpurun_out/r02bc_fp.log
timeout 900 python -m pytest tests/test_fingerprint_gpu.py tests/test_fingerprint_day.py tests/test_capi_fingerprint_gpu.py tests/test_demo_golden_gpu.py -q -x -s -p no:cacheprovider > gpurun_out/r02bc_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02bc_pytest.log
