#!/bin/bash
# MATCHED ncu capture (source-level) + compute-sanitizer logs (racecheck / synccheck / memcheck)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/one_search.py > gpurun_out/r02d_one.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc -c 1 -o gpurun_out/r02d_matched python tools/one_search.py > gpurun_out/r02d_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r02d_ncu.log
timeout 300 python tools/sanitize_run.py > gpurun_out/r02d_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/r02d_plain.log
for tool in memcheck synccheck racecheck; do
  QS_SAN_N=1500 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/r02d_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02d_san_$tool.log
done
