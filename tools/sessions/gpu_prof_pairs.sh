# full ncu captures of the two pair-enumeration launches of one cfg1 search
cd $GRAFT_REPO_ROOT
B='python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint'
timeout 600 $B > gpurun_out/b_B3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc -c 3 -o gpurun_out/prof_pairs_$1 $B > gpurun_out/ncu_pp.log 2>&1; echo prof $?
