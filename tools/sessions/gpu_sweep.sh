cd $GRAFT_REPO_ROOT
for L in paper_1803_09835_b200/lib/libquakescan_b200.so tools/variants/rs*/libquakescan_b200.so; do
  echo -n "$L "; QS_LIB_PATH=$PWD/$L timeout 300 python tools/prof_buckets.py 2>&1 | tail -1
done
python tools/sweep_pairs.py 8000000 paper_1803_09835_b200/lib/libquakescan_b200.so tools/variants/m12/libquakescan_b200.so tools/variants/m20/libquakescan_b200.so tools/variants/bp32/libquakescan_b200.so
