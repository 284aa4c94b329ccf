#!/bin/bash
# session 5, call c: cfg2 fingerprint launch list on the final build, cfg4 refresh
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
timeout 600 python tools/prof_fp_cfg2.py > $O/s5c_fp.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"^k_" --clock-control none --csv --log-file $O/s5c_fp_launches.csv python tools/prof_fp_cfg2.py > $O/s5c_ncu.log 2>&1; echo "list rc=$?"
python tools/launch_summary.py $O/s5c_fp_launches.csv --div 2 > $O/s5c_fp_launches.txt 2>&1; rm -f $O/s5c_fp_launches.csv; head -12 $O/s5c_fp_launches.txt
timeout 1500 python tools/cfg4_run.py > $O/s5c_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -1 $O/s5c_cfg4.log | cut -c1-500
