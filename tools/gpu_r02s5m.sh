#!/bin/bash
# session 5, call m: core-skip split on the final build (tables in the first MATCHED step)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
for S in 32 24 28 20 32; do
  QS_CORE_SPLIT=$S timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 0 > $O/s5m_$S.log 2>&1
  python - $S $O/s5m_$S.log <<'PY' | tee -a $O/s5m_split.log
import json, sys
for l in open(sys.argv[2]):
    if l.startswith('{'):
        j = json.loads(l); st = j['stages_ms']
        print('split', sys.argv[1], 'ms/step', round(j['ms_per_step'], 2), 'matched', round(st['pairs_matched'], 1), 'filter', round(st['filter'], 1), 'triplets', j['emitted_triplets'], j['distinct_pairs'])
PY
done
