#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_signatures -c 1 -o /tmp/ncu/sig python tools/one_search.py > gpurun_out/r02aw_ncu.log 2>&1
ncu -i /tmp/ncu/sig.ncu-rep --page details --csv > gpurun_out/r02aw_sig_details.csv 2>&1
ncu -i /tmp/ncu/sig.ncu-rep --page raw --csv > gpurun_out/r02aw_sig_raw.csv 2>&1
ncu -i /tmp/ncu/sig.ncu-rep --page source --csv --print-source sass > gpurun_out/r02aw_sig_sass.csv 2>&1
gzip -f gpurun_out/r02aw_sig_sass.csv gpurun_out/r02aw_sig_raw.csv
