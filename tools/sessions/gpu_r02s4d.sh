#!/bin/bash
# session-4: e2e host-transfer sweep + launch list with DRAM traffic
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/e2e_time.py 8000000 4 > gpurun_out/s4d_e2e.log 2>&1; echo "e2e rc=$?"; cat gpurun_out/s4d_e2e.log | tail -12
timeout 900 python tools/one_search.py > gpurun_out/s4d_one.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -k regex:"^k_|scan" --clock-control none --csv --log-file gpurun_out/s4d_search_launches.csv python tools/one_search.py > gpurun_out/s4d_ncu.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/s4d_search_launches.csv --half --traffic gpurun_out/s4d_traffic.json > gpurun_out/s4d_search_launches.txt 2>&1
head -12 gpurun_out/s4d_search_launches.txt
rm -f gpurun_out/s4d_search_launches.csv
