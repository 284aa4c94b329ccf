#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc -c 1 -o /tmp/ncu/big python tools/pairs_window.py matched 401 1000000000 > gpurun_out/r02aa_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02aa_ncu.log
ncu -i /tmp/ncu/big.ncu-rep --page details --csv > gpurun_out/r02aa_big_details.csv 2>&1
ncu -i /tmp/ncu/big.ncu-rep --page raw --csv > gpurun_out/r02aa_big_raw.csv 2>&1
ncu -i /tmp/ncu/big.ncu-rep --page source --csv --print-source sass > gpurun_out/r02aa_big_sass.csv 2>&1
gzip -f gpurun_out/r02aa_big_sass.csv gpurun_out/r02aa_big_raw.csv
timeout 900 ncu --set full --clock-control none -k regex:k_pairs_pc -c 1 -o /tmp/ncu/mid python tools/pairs_window.py matched 57 112 > gpurun_out/r02aa_ncu2.log 2>&1
ncu -i /tmp/ncu/mid.ncu-rep --page details --csv > gpurun_out/r02aa_mid_details.csv 2>&1
ls -la gpurun_out >> gpurun_out/r02aa_ncu.log
