#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02bg_fp_launches.csv python tools/fp_time.py 795000000 1 > gpurun_out/r02bg_ncu.log 2>&1
python3 - <<'PY' > gpurun_out/r02bg_fp_launches.txt
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r02bg_fp_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
agg = collections.OrderedDict(); c = collections.Counter()
for r in rows[1:]:
    k = r[ki][:60]; agg[k] = agg.get(k, 0) + float(r[vi].replace(",", "")); c[k] += 1
tot = sum(agg.values())
print(f"all launches of the run (3 fingerprint_series calls: warm-up, measured, ...): {tot/1e6:.2f} ms")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:20]: print(f"{v/1e6:9.3f} ms  x{c[k]:3d}  {k}")
PY
rm -f gpurun_out/r02bg_fp_launches.csv
