#!/bin/bash
# session-4: host-transfer paths (pinned DMA, uint16 / float32 narrowing): tests + bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_fingerprint_gpu.py tests/test_native_abi.py -x -q -p no:cacheprovider -k "e2e or out_of_range or upload or host_pack or integration" > gpurun_out/s4b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4b_pytest.log; tail -4 gpurun_out/s4b_pytest.log
nproc; free -g | head -2
for T in 8 16 32; do
  QS_COPY_THREADS=$T timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/s4b_bench_t$T.log 2>&1; echo "bench T=$T rc=$?"
  python - <<PY
import json
l=[x for x in open('gpurun_out/s4b_bench_t$T.log') if x.startswith('{')][-1]
d=json.loads(l)
print('T=$T ms/step', d['ms_per_step'], 'e2e', d['e2e']['seconds_per_step'], 'pageable', d['e2e'].get('pageable',{}).get('seconds_per_step'), 'fp', d['fingerprint']['ms_per_step'], 'fp e2e', d['fingerprint']['e2e']['seconds'])
PY
done
