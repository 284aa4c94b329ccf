"""Pair-stage cost per bucket-size class at cfg1 (design measurement).

Builds the cfg1 search layout once (N = 8e6 by default), prints the
pair-weighted bucket-size histogram, then times the MATCHED pass (and the
uncompacted DISTINCT pass) restricted to one bucket-size window at a time
(QS_PAIRS_SMIN / QS_PAIRS_SMAX, read by the pair launcher)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["matched", "distinct"]
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
del bits
ds = ls.DeviceSearch(keys, rkeys, tags, n, 100)
ds.buckets()
bs = ds.bsize[: ds.nb].to(torch.int64).cpu().numpy()
bt = ds.btab[: ds.nb].to(torch.int64).cpu().numpy()
edges = torch.tensor([0, n], dtype=torch.int64, device="cuda")
windows = [(2, 8), (9, 16), (17, 32), (33, 56), (57, 112), (113, 200), (201, 400), (401, 1 << 30)]


import ctypes
from paper_1803_09835_b200 import _native as nat
_prof = getattr(nat.lib(), "qs_prof_read", None)
if _prof is not None:
    _prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
_pbuf = (ctypes.c_ulonglong * 8)()


def timed(mode, lo, hi):
    os.environ["QS_PAIRS_SMIN"], os.environ["QS_PAIRS_SMAX"] = str(lo), str(hi)
    ds.pairs(mode, 5, 0, None, edges, 1)  # warm (cap hint)
    torch.cuda.synchronize()
    if _prof is not None:
        _prof(_pbuf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pk, ps, matched, distinct = ds.pairs(mode, 5, 0, None, edges, 1)
    e1.record()
    torch.cuda.synchronize()
    if _prof is not None:
        _prof(_pbuf, 1)
        v = [x / 1e9 for x in _pbuf]
        print("  prof Gcycles: producer wait_empty %.2f build %.2f | consumer wait_full %.2f compute %.2f drain %.2f"
              % (v[0], v[1], v[4], v[5], v[6]), flush=True)
    return e0.elapsed_time(e1), matched, distinct


out = {"n": n, "nb": int(ds.nb)}
for name in modes:
    mode = {"matched": ds.MODE_MATCHED, "distinct": ds.MODE_DISTINCT, "full": ds.MODE_FULL}[name]
    tmax = 95 if name == "matched" else 99
    rows = []
    ms_all, mt_all, di_all = timed(mode, 0, 1 << 30)
    for lo, hi in windows:
        sel = (bs >= lo) & (bs <= hi) & (bt <= tmax)
        pairs = int((bs[sel] * (bs[sel] - 1) // 2).sum())
        ms, mt, di = timed(mode, lo, hi)
        rows.append({"sizes": f"{lo}-{hi}", "buckets": int(sel.sum()), "members": int(bs[sel].sum()),
                     "pairs": pairs, "ms": round(ms, 2), "matched": mt, "distinct": di,
                     "ns_per_kpair": round(1e6 * ms / max(pairs, 1), 3)})
        print(name, rows[-1], flush=True)
    sel = bt <= tmax
    out[name] = {"all_ms": round(ms_all, 2), "pairs": int((bs[sel] * (bs[sel] - 1) // 2).sum()),
                 "matched": mt_all, "distinct": di_all, "classes": rows,
                 "sum_class_ms": round(sum(r["ms"] for r in rows), 2)}
    print(name, "all", out[name]["all_ms"], "ms; sum of classes", out[name]["sum_class_ms"], flush=True)
os.environ.pop("QS_PAIRS_SMIN"); os.environ.pop("QS_PAIRS_SMAX")
print(json.dumps(out))
