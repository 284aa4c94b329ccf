#!/bin/bash
# session 5, call q: ncu --set full of k_rs_scatter and k_signatures on the final build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out /tmp/ncu; O=gpurun_out
timeout 600 python tools/prof_buckets.py > $O/s5q_prof_buckets.log 2>&1; echo "plain rc=$?"
for K in k_rs_scatter k_signatures; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o /tmp/ncu/s5q_$K -f python tools/prof_buckets.py > $O/s5q_prof_$K.log 2>&1; echo "$K rc=$?"
  ncu -i /tmp/ncu/s5q_$K.ncu-rep --page details --csv > $O/s5q_prof_${K}_details.csv 2>&1
  ncu -i /tmp/ncu/s5q_$K.ncu-rep --page raw --csv > $O/s5q_prof_${K}_raw.csv 2>&1
done
