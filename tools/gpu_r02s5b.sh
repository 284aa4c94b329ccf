#!/bin/bash
# session 5, call b: k_win_cta resident-CTA A/B (lib/v3 = -DWC_MINB=3 -> up to 85 registers)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
for i in 1 2; do
  timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/minb4: /' | tee -a $O/s5b_fp.log
  QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/v3/libquakescan_b200.so timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/minb3: /' | tee -a $O/s5b_fp.log
done
