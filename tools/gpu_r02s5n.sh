#!/bin/bash
# session 5, call n: Min-Max kernel with 4 / 8 interleaved bitmap replicas per warp (lib/vb4, lib/vb8)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
for V in base vb4 vb8 base vb4; do
  if [ $V = base ]; then unset QS_LIB_PATH; else export QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/$V/libquakescan_b200.so; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 0 > $O/s5n_$V.log 2>&1
  python - $V $O/s5n_$V.log <<'PY' | tee -a $O/s5n_minhash.log
import json, sys
for l in open(sys.argv[2]):
    if l.startswith('{'):
        j = json.loads(l); st = j['stages_ms']
        print(sys.argv[1], 'ms/step', round(j['ms_per_step'], 2), 'minhash', round(st['minhash'], 2), 'triplets', j['emitted_triplets'], j['distinct_pairs'])
PY
done
export QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/vb4/libquakescan_b200.so
timeout 900 python -m pytest tests/test_minmax_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 | tee -a $O/s5n_minhash.log
