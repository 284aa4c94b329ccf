#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/pairs_window.py matched 2 8 > gpurun_out/r02y_w.log 2>&1
QS_SMALL=0 timeout 300 python tools/pairs_window.py matched 2 8 >> gpurun_out/r02y_w.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r02y_launches.csv python tools/pairs_window.py matched 2 8 > gpurun_out/r02y_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02y_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_small -c 1 -o /tmp/ncu/small python tools/pairs_window.py matched 2 8 > gpurun_out/r02y_ncu2.log 2>&1
echo "rc=$?" >> gpurun_out/r02y_ncu2.log
ncu -i /tmp/ncu/small.ncu-rep --page details --csv > gpurun_out/r02y_small_details.csv 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page source --csv --print-source sass > gpurun_out/r02y_small_sass.csv 2>&1
gzip -f gpurun_out/r02y_small_sass.csv
ls -la gpurun_out >> gpurun_out/r02y_ncu2.log
