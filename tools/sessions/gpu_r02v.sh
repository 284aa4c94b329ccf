#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/pair_classes.py 8000000 matched,distinct > gpurun_out/r02v_classes.log 2>&1
echo "rc=$?" >> gpurun_out/r02v_classes.log
