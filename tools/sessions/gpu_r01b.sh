cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_sharded_gpu.py tests/test_lsh_gpu.py -x -q > gpurun_out/pt_sh.log 2>&1; tail -3 gpurun_out/pt_sh.log
QS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --n 2000000 --no-cpu-baseline --no-fingerprint > gpurun_out/b_n2.log 2>&1; echo n2 $?; tail -1 gpurun_out/b_n2.log | cut -c1-900
B='python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint'
timeout 600 $B > gpurun_out/b_B2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs_pc --launch-skip 2 -c 1 -o gpurun_out/prof_pairs_dist_r01 $B > gpurun_out/ncu_pd.log 2>&1; echo pd $?
