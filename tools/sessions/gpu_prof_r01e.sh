cd $GRAFT_REPO_ROOT
timeout 600 python tools/one_search.py > gpurun_out/os.log 2>&1 || exit 1
# per search: MATCHED words 0, 1, 2 (word 3 holds no first collision at m = 5), then DISTINCT words 0..3
for k in 0 1 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc --launch-skip $k -c 1 -o gpurun_out/prof_pm_l$k python tools/one_search.py > gpurun_out/ncu_pm_l$k.log 2>&1; echo l$k $?
done
