# bucket build: parity tests, stage timing, per-kernel launch list
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_buckets_gpu.py -x -q > gpurun_out/pt_b.log 2>&1; tail -3 gpurun_out/pt_b.log
timeout 300 python tools/prof_buckets.py > gpurun_out/pb.log 2>&1; tail -2 gpurun_out/pb.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_bin|k_listf|k_rs|k_fix|k_flags|k_make|k_scan" --log-file gpurun_out/pb_launches.csv python tools/prof_buckets.py > /dev/null 2>&1
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/pb_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0]; agg[k] = agg.get(k, 0) + float(r[vi].replace(",", ""))
for k, v in agg.items(): print(f"{v/2e6:9.3f} ms/build  {k}")
PY
