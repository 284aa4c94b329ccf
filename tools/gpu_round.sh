cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pt_r01.log 2>&1; tail -3 gpurun_out/pt_r01.log
timeout 900 python bench.py > gpurun_out/b_full2.log 2>&1; tail -1 gpurun_out/b_full2.log | cut -c1-600
timeout 300 python bench.py --impl reference > gpurun_out/b_ref2.log 2>&1; tail -1 gpurun_out/b_ref2.log | cut -c1-200
A='python bench.py --steps 1 --warmup 3 --no-cpu-baseline'
timeout 900 $A > gpurun_out/b_small.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $A > gpurun_out/ncu_list_r01.log 2>&1; echo list $?
B='python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint'
timeout 600 $B > gpurun_out/b_B.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc -c 2 -o gpurun_out/prof_pairs_r01 $B > gpurun_out/ncu_pairs_r01.log 2>&1; echo pairs $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_signatures -c 1 -o gpurun_out/prof_sig_r01 $B > gpurun_out/ncu_sig_r01.log 2>&1; echo sig $?
