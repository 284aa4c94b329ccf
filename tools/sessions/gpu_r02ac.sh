#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/pairs_window.py matched 2 8 > gpurun_out/r02ac_w.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_small -c 1 -o /tmp/ncu/small python tools/pairs_window.py matched 2 8 > gpurun_out/r02ac_ncu2.log 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page details --csv > gpurun_out/r02ac_small_details.csv 2>&1
ncu -i /tmp/ncu/small.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ac_small_sass.csv 2>&1
gzip -f gpurun_out/r02ac_small_sass.csv
timeout 900 python -m pytest tests/test_lsh_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02ac_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02ac_pytest.log
