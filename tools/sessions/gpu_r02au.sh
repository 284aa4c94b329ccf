#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for sp in 24 40 48 64; do
  QS_CORE_SPLIT=$sp timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 0 > gpurun_out/r02au_bench_$sp.log 2>&1
done
