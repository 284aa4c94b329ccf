"""Randomised parity sweep of search_signatures against the oracle (more and
larger cases than tests/test_lsh_gpu.py; run on a GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import search as osr
from paper_1803_09835_b200 import lsh_search as ls

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 150
t0 = time.time()
bad = 0
for seed in range(n_cases):
    rng = np.random.default_rng(10_000 + seed)
    n = int(rng.integers(2, 3000))
    t = int(rng.choice([1, 2, 5, 31, 32, 33, 64, 96, 100, 128]))
    alpha = int(rng.choice([2, 3, 5, 10, 40, 200, 5000]))
    sigs = rng.integers(0, alpha, size=(n, t)).astype(np.uint64)
    if rng.random() < 0.3:  # planted near-duplicate blocks
        for _ in range(int(rng.integers(1, 20))):
            a, b = rng.integers(0, n, 2)
            keep = rng.random(t) < rng.uniform(0.2, 0.9)
            sigs[b, keep] = sigs[a, keep]
    m = int(rng.integers(1, min(t, 8) + 1))
    p = int(rng.choice([1, 1, 2, 3, 5]))
    occ = [None, 0.002, 0.02, 0.2, 1.0][int(rng.integers(0, 5))]
    excl = int(rng.choice([0, 0, 1, 3, 10]))
    cfg = ls.SearchConfig(tables=t, hash_funcs=2, min_matches=m, partitions=p,
                          occurrence_threshold=occ)
    rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
    want, wst = osr.search(sigs, tables=t, min_matches=m, partitions=p,
                           occurrence_threshold=occ, exclusion_windows=excl)
    ok = rec.tobytes() == want.tobytes()
    d = st.to_dict()
    for k, v in wst.items():
        if k in ("lookups_per_query", "selectivity"):
            continue
        if isinstance(v, float):
            ok = ok and abs(d[k] - v) <= 1e-12 * max(1.0, abs(v))
        else:
            ok = ok and d[k] == v
    if not ok:
        bad += 1
        print("MISMATCH", dict(seed=seed, n=n, t=t, alpha=alpha, m=m, p=p, occ=occ, excl=excl), flush=True)
print(f"{n_cases - bad}/{n_cases} cases identical ({time.time() - t0:.0f} s)")
