#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
QS_LIB_PATH=$GRAFT_REPO_ROOT/tools/variants/prof/libquakescan_b200.so timeout 900 python tools/pair_classes.py 8000000 matched > gpurun_out/r02w_prof.log 2>&1
echo "rc=$?" >> gpurun_out/r02w_prof.log
