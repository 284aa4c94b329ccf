# round-end style run: GPU tests, default bench, reference arm, launch list, pair-stage traffic, full captures
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pt_final.log 2>&1; tail -2 gpurun_out/pt_final.log
timeout 900 python bench.py > gpurun_out/b_final.log 2>&1; tail -1 gpurun_out/b_final.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/b_ref_final.log 2>&1; tail -1 gpurun_out/b_ref_final.log | cut -c1-200
A='python bench.py --steps 1 --warmup 3 --no-cpu-baseline'
timeout 900 $A > gpurun_out/b_small2.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $A > gpurun_out/ncu_list_final.log 2>&1; echo list $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_pairs_pc --log-file gpurun_out/pair_traffic.csv python tools/one_search.py > gpurun_out/pair_traffic.log 2>&1; echo traffic $?
for KS in k_pairs_pc:tools/one_search.py k_signatures:tools/prof_buckets.py; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K -f python $S > gpurun_out/prof_$K.log 2>&1; echo $K $?
done
