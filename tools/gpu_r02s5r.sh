#!/bin/bash
# session 5, call r: radix scatter CTA shapes (lib/ra 512x8 minb2, lib/rc 1024x4, lib/rd 512x8 minb3) against 256x16
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
for V in base ra rc rd base ra rc; do
  if [ $V = base ]; then unset QS_LIB_PATH; else export QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/$V/libquakescan_b200.so; fi
  timeout 600 python tools/prof_buckets.py 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$V: /" | tee -a $O/s5r_scatter.log
done
for V in ra rc; do
  QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/$V/libquakescan_b200.so timeout 900 python -m pytest tests/test_buckets_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/$V: /" | tee -a $O/s5r_scatter.log
done
