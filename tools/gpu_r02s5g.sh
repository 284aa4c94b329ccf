#!/bin/bash
# session 5, call g: staging thread-pool size against the e2e time (12-bit narrowing)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
nproc | tee $O/s5g_e2e.log; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA" | tee -a $O/s5g_e2e.log
for T in 8 16 24 32; do
  QS_COPY_THREADS=$T QS_E2E_SPLITS=0.7,0.85 timeout 900 python tools/e2e_time.py 8000000 3 2>&1 | grep -E "pinned|narrowed" | sed "s/^/threads=$T: /" | tee -a $O/s5g_e2e.log
done
