#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for v in base m4a m4b m4c; do
  if [ $v = base ]; then unset QS_LIB_PATH; else export QS_LIB_PATH=$GRAFT_REPO_ROOT/tools/variants/$v/libquakescan_b200.so; fi
  echo "== $v" >> gpurun_out/r02ao.log
  timeout 300 python tools/pairs_window.py matched 0 1000000000 >> gpurun_out/r02ao.log 2>&1
done
