#!/bin/bash
# quick check of a search-path change: search tests, a short randomised sweep, a short bench (stage split)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out; T=${1:-q}
timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_capi_search_gpu.py tests/test_sharded_gpu.py -q -x -p no:cacheprovider -k "not full_scale" 2>&1 | tail -2 | tee $O/${T}_pytest.log
timeout 900 python tools/stress_parity.py 60 2>&1 | tail -1 | tee $O/${T}_stress.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 1 > $O/${T}_bench.log 2>&1; echo "bench rc=$?"
python - "$O/${T}_bench.log" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        j = json.loads(l)
        print('ms/step', round(j['ms_per_step'], 2), {k: round(v, 1) for k, v in j['stages_ms'].items()})
        if j.get('full_mode'):
            print('full ms/step', round(j['full_mode']['ms_per_step'], 2), {k: round(v, 1) for k, v in j['full_mode']['stages_ms'].items()})
        print('triplets', j['emitted_triplets'], 'filtered', j['filtered_fingerprints'], 'distinct', j['distinct_pairs'])
PY
