# A/B of the FULL-mode (no occurrence filter) search: default build vs tools/variants/nofold
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_lsh_gpu.py tests/test_buckets_gpu.py tests/test_sharded_gpu.py -x -q > gpurun_out/pt_iter.log 2>&1; tail -1 gpurun_out/pt_iter.log
for L in "" tools/variants/nofold/libquakescan_b200.so; do
QS_LIB_PATH=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fingerprint --occ 0 > gpurun_out/b_full.log 2>&1; tail -1 gpurun_out/b_full.log | python3 -c "import json,sys; l=json.loads(sys.stdin.read()); print('$L', l['ms_per_step'], {k: round(v,1) for k,v in l['stages_ms'].items()})"
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fingerprint > gpurun_out/b_iter.log 2>&1; tail -1 gpurun_out/b_iter.log | python3 -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], {k: round(v,1) for k,v in l['stages_ms'].items()}, l['roofline']['frac'])"
