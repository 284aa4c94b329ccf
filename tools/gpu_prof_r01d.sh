cd $GRAFT_REPO_ROOT
timeout 600 python tools/one_search.py > gpurun_out/os.log 2>&1 || exit 1
# launches per search: MATCHED (x2 on the first search: capacity retry), then DISTINCT words 0..3
for k in 0 2 3 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc --launch-skip $k -c 1 -o gpurun_out/prof_pc_l$k python tools/one_search.py > gpurun_out/ncu_l$k.log 2>&1; echo l$k $?
done
