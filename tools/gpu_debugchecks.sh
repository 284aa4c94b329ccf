#!/bin/bash
# Sanitizer substitute (compute-sanitizer is closed on this pool): the library
# built with -DQS_DEBUG_CHECKS (device bounds asserts in the asynchronous
# kernels; a failed assert traps the kernel) runs the randomised search and
# fingerprint parity sweeps and the small all-modes run.
cd "$GRAFT_REPO_ROOT"
export QS_LIB_PATH=$GRAFT_REPO_ROOT/paper_1803_09835_b200/lib/debug/libquakescan_b200.so
timeout 600 python tools/sanitize_run.py > gpurun_out/dbg_sanitize_run.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_sanitize_run.log
timeout 1200 python tools/stress_parity.py 200 > gpurun_out/dbg_stress_parity.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_stress_parity.log
timeout 1200 python tools/stress_fingerprint.py 40 > gpurun_out/dbg_stress_fp.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_stress_fp.log
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_buckets_gpu.py tests/test_capi_search_gpu.py -q -x -p no:cacheprovider > gpurun_out/dbg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_pytest.log
