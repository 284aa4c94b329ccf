#!/bin/bash
# session 5, call i: k_col_median with a sampled first-digit range (lib/vc) against the default build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
V=$PWD/paper_1803_09835_b200/lib/vc/libquakescan_b200.so
for i in 1 2; do
  timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/base: /' | tee -a $O/s5i_fp.log
  QS_LIB_PATH=$V timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/sampled: /' | tee -a $O/s5i_fp.log
done
QS_LIB_PATH=$V timeout 900 python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "fingerprint or demo or golden" 2>&1 | tail -2 | tee -a $O/s5i_fp.log
QS_LIB_PATH=$V timeout 900 python tools/stress_fingerprint.py 40 2>&1 | tail -1 | tee -a $O/s5i_fp.log
