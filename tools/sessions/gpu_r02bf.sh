#!/bin/bash
# ncu --set full of k_win_cta (main pass, cfg0 day) and k_band_stft_mma
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
for spec in "k_win_cta 3" ; do
  set -- $spec; K=$1; SKIP=$2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 -o /tmp/ncu/$K -f python tools/prof_fp.py > gpurun_out/r02bf_$K.log 2>&1; echo "ncu $K rc=$?" >> gpurun_out/r02bf_$K.log
  ncu -i /tmp/ncu/$K.ncu-rep --page details --csv > gpurun_out/r02bf_${K}_details.csv 2>&1
  ncu -i /tmp/ncu/$K.ncu-rep --page raw --csv > gpurun_out/r02bf_${K}_raw.csv 2>&1
  ncu -i /tmp/ncu/$K.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02bf_${K}_cuda.csv 2>&1
  ncu -i /tmp/ncu/$K.ncu-rep --page source --csv --print-source sass > gpurun_out/r02bf_${K}_sass.csv 2>&1
  gzip -f gpurun_out/r02bf_${K}_raw.csv gpurun_out/r02bf_${K}_sass.csv gpurun_out/r02bf_${K}_cuda.csv
done
