# iteration run: bucket + search parity tests, then the timed search bench (no CPU/e2e/fingerprint legs)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_buckets_gpu.py tests/test_lsh_gpu.py tests/test_sharded_gpu.py -x -q > gpurun_out/pt_iter.log 2>&1; tail -3 gpurun_out/pt_iter.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fingerprint > gpurun_out/b_iter.log 2>&1; tail -1 gpurun_out/b_iter.log | python3 -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], {k: round(v,1) for k,v in l['stages_ms'].items()}, l['roofline']['frac'])"
