#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:qs:: --clock-control none --csv --log-file gpurun_out/r02af_launches.csv python tools/pairs_window.py matched 2 8 > gpurun_out/r02af_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02af_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_small -c 1 -o /tmp/ncu/small python tools/pairs_window.py matched 2 8 > gpurun_out/r02af_ncu2.log 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page details --csv > gpurun_out/r02af_small_details.csv 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page raw --csv > gpurun_out/r02af_small_raw.csv 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page source --csv --print-source sass > gpurun_out/r02af_small_sass.csv 2>&1
gzip -f gpurun_out/r02af_small_sass.csv gpurun_out/r02af_small_raw.csv
