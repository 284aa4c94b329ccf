#!/bin/bash
# session 5, call k: adaptive narrowed share (no QS_H2D_SPLIT) against fixed splits; host-transfer tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py -q -x -p no:cacheprovider -k "host or e2e" 2>&1 | tail -3 | tee $O/s5k_pytest.log
QS_E2E_SPLITS=auto,0.6,0.7,auto,0.7,auto timeout 900 python tools/e2e_time.py 8000000 3 2>&1 | grep pinned | tee $O/s5k_e2e.log
