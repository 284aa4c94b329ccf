# quick GPU iteration: parity tests of the search + timed bench without the CPU/e2e/fingerprint legs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_lsh_gpu.py tests/test_sharded_gpu.py -x -q > gpurun_out/pt_q.log 2>&1; tail -2 gpurun_out/pt_q.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fingerprint > gpurun_out/b_q.log 2>&1; tail -1 gpurun_out/b_q.log | python3 -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], {k: round(v,1) for k,v in l['stages_ms'].items()}, l['roofline']['frac'])"
if [ -n "$QS_N2" ]; then
QS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --fingerprints 2000000 --no-cpu-baseline --no-fingerprint > gpurun_out/b_n2.log 2>&1; echo n2 $?; tail -1 gpurun_out/b_n2.log | cut -c1-1200
fi
