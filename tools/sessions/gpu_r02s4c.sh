#!/bin/bash
# session-4: host-transfer paths, second pass (hybrid pinned path, background MAD draw)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_fingerprint_gpu.py tests/test_native_abi.py tests/test_sharded_gpu.py -x -q -p no:cacheprovider -k "e2e or out_of_range or upload or host_pack or integration or sharded" > gpurun_out/s4c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4c_pytest.log; tail -4 gpurun_out/s4c_pytest.log
for SP in 0.6 0.7 0.8; do
  QS_H2D_SPLIT=$SP timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/s4c_bench_s$SP.log 2>&1; echo "bench split=$SP rc=$?"
  python - <<PY
import json
l=[x for x in open('gpurun_out/s4c_bench_s$SP.log') if x.startswith('{')][-1]
d=json.loads(l)
print('split=$SP ms/step', d['ms_per_step'], 'e2e', d['e2e']['seconds_per_step'], d['e2e']['h2d_bytes_per_step'], 'pageable', d['e2e'].get('pageable',{}).get('seconds_per_step'), 'fp', d['fingerprint']['ms_per_step'], 'fp e2e', d['fingerprint']['e2e']['seconds'])
PY
done
