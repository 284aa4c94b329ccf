"""CPU scaling of the reference search (run on the GPU box's host; log ->
profiles/r02_cpu_scaling.log): the reference's own quakescan signatures
(workers = all cores) + search_signatures (baseline/_ref, unmodified) on the
cfg1 generator at N in {1e5, 2e5, 4e5, 8e5}, filter off and at limit 120.
Fits t(N) = a + b N + c N^2 per mode (least squares) and extrapolates to
N = 8e6 — labelled as an extrapolation: the reference cannot run there
(>= 224 GB of pair keys)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import numpy as np  # noqa: E402
from quakescan import lsh_search as rls  # noqa: E402
from quakescan import minmax_hash as rmh  # noqa: E402

from paper_1803_09835_b200 import workloads  # noqa: E402

ns = [int(float(a)) for a in sys.argv[1:]] or [100_000, 200_000, 400_000, 800_000]
threads = len(os.sched_getaffinity(0))
mapping = rmh.gen_hash_mapping(4096, 100, 4, 0)
rows = {"off": [], "on": []}
for n in ns:
    bits, _ = workloads.cfg1_bits(n=n, seed=0)
    t0 = time.perf_counter()
    sigs = rmh.signatures(bits, mapping, workers=threads)
    ts = time.perf_counter() - t0
    for mode, occ in (("off", None), ("on", 120 / n)):
        t1 = time.perf_counter()
        rec, st = rls.search_signatures(sigs, rls.SearchConfig(tables=100, hash_funcs=4,
                                                               min_matches=5,
                                                               occurrence_threshold=occ))
        tq = time.perf_counter() - t1
        rows[mode].append((n, ts, tq))
        print(f"N={n} filter={mode}: signatures {ts:.2f} s ({threads} threads), search {tq:.2f} s, "
              f"{rec.size} triplets, {st.distinct_pairs} distinct pairs -> "
              f"{n / (ts + tq):.0f} fp/s", flush=True)
    del bits, sigs
out = {"threads": threads, "backend": rmh.BACKEND, "points": rows, "fits": {}}
for mode, pts in rows.items():
    N = np.array([p[0] for p in pts], float)
    T = np.array([p[1] + p[2] for p in pts], float)
    A = np.stack([np.ones_like(N), N, N * N], 1)
    coef, *_ = np.linalg.lstsq(A, T, rcond=None)
    t8 = float(coef @ np.array([1.0, 8e6, 6.4e13]))
    out["fits"][mode] = {"a": coef[0], "b": coef[1], "c": coef[2], "t_8e6_s": t8,
                         "fp_per_s_8e6": 8e6 / t8 if t8 > 0 else None}
    print(f"fit filter={mode}: t(N) = {coef[0]:.3g} + {coef[1]:.3g} N + {coef[2]:.3g} N^2 -> "
          f"extrapolated t(8e6) = {t8:.0f} s = {8e6 / t8:.0f} fp/s", flush=True)
print(json.dumps(out))
