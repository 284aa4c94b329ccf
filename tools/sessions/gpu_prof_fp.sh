cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_fp.py > gpurun_out/pfp.log 2>&1; tail -1 gpurun_out/pfp.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pfp_launches.csv python tools/prof_fp.py > /dev/null 2>&1
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/pfp_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
agg = collections.OrderedDict(); c = collections.Counter()
for r in rows[1:]:
    k = r[ki].split("(")[0][:70]; agg[k] = agg.get(k, 0) + float(r[vi].replace(",", "")); c[k] += 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:14]: print(f"{v/2e6:9.3f} ms/call x{c[k]//2} {k}")
PY
bash tools/gpu_prof_kernel.sh k_windows tools/prof_fp.py
