"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --csv) of
tools/one_search.py: per-kernel totals of the LAST search of the run (the first
is the warm-up), and the pair-stage DRAM traffic written to profiles/traffic.json
(the `roofline.traffic` bench.py reports).

usage: launch_summary.py launches.csv [--half] [--div STEPS] [--traffic profiles/traffic.json] [--n 8000000]
"""
import collections
import csv
import json
import re
import sys


def main():
    path = sys.argv[1]
    half = "--half" in sys.argv
    traffic_out = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 8_000_000
    div = float(sys.argv[sys.argv.index("--div") + 1]) if "--div" in sys.argv else 1.0  # steps in the run
    rows = [r for r in csv.reader(open(path, errors="replace")) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID",
                                                  "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        u = r[ui].lower()
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0,
                 "second": 1e3, "byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1.0)
        d[r[mi]] = v * scale
    ls = list(launches.values())
    if half:
        ls = ls[len(ls) // 2:]
    agg = collections.OrderedDict()
    for d in ls:
        k = re.sub(r"^(void )?(qs::)?", "", d["name"])
        k = re.sub(r"\(.*$", "", k)[:48]
        a = agg.setdefault(k, {"n": 0, "ms": 0.0, "inst": 0.0, "dram": 0.0})
        a["n"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0.0)
        a["inst"] += d.get("smsp__inst_executed.sum", 0.0)
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    for a in agg.values():
        for k in ("n", "ms", "inst", "dram"):
            a[k] = a[k] / div
    tot = sum(a["ms"] for a in agg.values())
    if div != 1.0:
        print(f"per step (totals of the run / {div:g} steps)")
    print(f"launches {len(launches)} in part {len(ls)} total ms {tot:.2f}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        print(f"{k:50s} n={a['n']:7.1f} ms={a['ms']:8.2f} inst={a['inst']:.3g} dramGB={a['dram'] / 1e9:7.2f}")
    if traffic_out:
        pair = {k: a for k, a in agg.items() if k.startswith("k_pairs_")}
        out = {"n": n, "kernel": "k_pairs_pc + k_pairs_small (every pair-stage launch of one cfg1 step)",
               "source": ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                          "dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none on "
                          "tools/one_search.py, the second search's launches (tools/launch_summary.py)"),
               "pair_stage_dram_bytes_total": int(sum(a["dram"] for a in pair.values())),
               "pair_stage_ms_under_ncu": sum(a["ms"] for a in pair.values()),
               "pair_stage_dram_bytes": {k: int(a["dram"]) for k, a in pair.items()},
               "launch_ms": {k: round(a["ms"], 3) for k, a in pair.items()}}
        json.dump(out, open(traffic_out, "w"), indent=1)


main()
