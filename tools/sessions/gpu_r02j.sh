#!/bin/bash
# fingerprint chain: launch list (cfg0 day) + full capture of the mode-3 window kernel
cd "$GRAFT_REPO_ROOT"
timeout 300 python tools/prof_fp.py > gpurun_out/r02j_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_fp.py > gpurun_out/r02j_launches.csv 2> gpurun_out/r02j_launches.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_windows --launch-skip 1 -c 1 -o gpurun_out/r02j_windows python tools/prof_fp.py > gpurun_out/r02j_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02j_ncu.log
