#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 600 python tools/prof_fp_cfg2.py > gpurun_out/r02ag_fp.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"^k_" --clock-control none --csv --log-file gpurun_out/r02ag_fp_launches.csv python tools/prof_fp_cfg2.py > gpurun_out/r02ag_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win_cta -c 1 -o /tmp/ncu/win python tools/prof_fp_cfg2.py 40000000 > gpurun_out/r02ag_ncu2.log 2>&1
ncu -i /tmp/ncu/win.ncu-rep --page details --csv > gpurun_out/r02ag_win_details.csv 2>&1
ncu -i /tmp/ncu/win.ncu-rep --page raw --csv > gpurun_out/r02ag_win_raw.csv 2>&1
ncu -i /tmp/ncu/win.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ag_win_sass.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_band_stft -c 1 -o /tmp/ncu/stft python tools/prof_fp_cfg2.py 40000000 > gpurun_out/r02ag_ncu3.log 2>&1
ncu -i /tmp/ncu/stft.ncu-rep --page details --csv > gpurun_out/r02ag_stft_details.csv 2>&1
ncu -i /tmp/ncu/stft.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ag_stft_sass.csv 2>&1
gzip -f gpurun_out/r02ag_*sass.csv gpurun_out/r02ag_win_raw.csv
