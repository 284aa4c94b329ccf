#!/bin/bash
# A/B of an alternative library build (QS_LIB_PATH) against the default on the cfg1 stage split
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out; V=$1
show() { python - "$1" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        j = json.loads(l)
        print('ms/step', round(j['ms_per_step'], 2), {k: round(v, 1) for k, v in j['stages_ms'].items()})
        if j.get('full_mode'):
            print('full ms/step', round(j['full_mode']['ms_per_step'], 2), {k: round(v, 1) for k, v in j['full_mode']['stages_ms'].items()})
        print('triplets', j['emitted_triplets'], 'filtered', j['filtered_fingerprints'], 'distinct', j['distinct_pairs'])
PY
}
A='python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 1'
timeout 900 $A > $O/ab_base.log 2>&1; echo "base rc=$?"; show $O/ab_base.log
QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/$V/libquakescan_b200.so timeout 900 $A > $O/ab_$V.log 2>&1; echo "$V rc=$?"; show $O/ab_$V.log
