#!/bin/bash
# session 5, call f: 12-bit host narrowing of the bit indices: tests + e2e timing (split sweep)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_native_abi.py tests/test_capi_search_gpu.py -q -x -p no:cacheprovider -k "host or e2e or abi or pack" 2>&1 | tail -5 | tee $O/s5f_pytest.log
QS_E2E_SPLITS=0.6,0.7,0.8,0.9,1 timeout 900 python tools/e2e_time.py 8000000 3 2>&1 | tail -8 | tee $O/s5f_e2e.log
QS_H2D_NARROW=16 QS_E2E_SPLITS=0.7 timeout 900 python tools/e2e_time.py 8000000 3 2>&1 | tail -3 | sed 's/^/u16: /' | tee -a $O/s5f_e2e.log
