#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win_cta --launch-skip 1 -c 1 -o /tmp/ncu/win3 python tools/prof_fp_cfg2.py 40000000 > gpurun_out/r02aj_ncu.log 2>&1
ncu -i /tmp/ncu/win3.ncu-rep --page details --csv > gpurun_out/r02aj_win3_details.csv 2>&1
ncu -i /tmp/ncu/win3.ncu-rep --page raw --csv > gpurun_out/r02aj_win3_raw.csv 2>&1
ncu -i /tmp/ncu/win3.ncu-rep --page source --csv --print-source sass > gpurun_out/r02aj_win3_sass.csv 2>&1
ncu -i /tmp/ncu/win3.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02aj_win3_cuda.csv 2>&1
gzip -f gpurun_out/r02aj_*.csv
