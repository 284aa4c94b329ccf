# round-end style run: GPU tests, default bench, reference arm, launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pt_final.log 2>&1; tail -2 gpurun_out/pt_final.log
timeout 900 python bench.py > gpurun_out/b_final.log 2>&1; tail -1 gpurun_out/b_final.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/b_ref_final.log 2>&1; tail -1 gpurun_out/b_ref_final.log | cut -c1-200
A='python bench.py --steps 1 --warmup 3 --no-cpu-baseline'
timeout 900 $A > gpurun_out/b_small2.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $A > gpurun_out/ncu_list_final.log 2>&1; echo list $?
