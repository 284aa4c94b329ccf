"""cfg1-generator parity at growing N (run on a GPU box; log -> profiles/).

For each N: Min-Max signatures on the GPU vs the C oracle (all rows), then
search_signatures on the GPU vs the numpy oracle (byte-identical triplets,
every SearchStats field) with the filter off (the reference default), on at
limit 120 (the bench's setting), and on with 3 partitions + exclusion.  With
--ref, the reference's OWN search_signatures (baseline/_ref, unmodified) is
run too at the smallest N.

    python tools/parity_cfg1.py 100000 200000 400000 [--ref]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import minmax as omm  # noqa: E402
from oracle import search as osr  # noqa: E402
from paper_1803_09835_b200 import lsh_search as ls  # noqa: E402
from paper_1803_09835_b200 import minmax_hash as mh  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402


def same_stats(d, w):
    for k, v in w.items():
        if k in ("lookups_per_query", "selectivity"):
            continue
        if isinstance(v, float):
            if abs(d[k] - v) > 1e-12 * max(1.0, abs(v)):
                return False
        elif d[k] != v:
            return False
    return True


def main():
    ns = [int(float(a)) for a in sys.argv[1:] if not a.startswith("--")]
    use_ref = "--ref" in sys.argv
    threads = len(os.sched_getaffinity(0))
    m = mh.gen_hash_mapping(4096, 100, 4, 0)
    bad = 0
    for n in ns:
        t0 = time.time()
        bits, _ = workloads.cfg1_bits(n=n, seed=100 + n % 977)
        sigs = mh.signatures(bits, m)
        want_sigs = omm.signatures_c(bits, m.values, 100, 2, threads=threads)
        ok = np.array_equal(sigs, want_sigs)
        print(f"N={n}: signatures {'identical' if ok else 'MISMATCH'} ({time.time() - t0:.0f} s)",
              flush=True)
        bad += not ok
        for occ_limit, p, excl in [(None, 1, 0), (120, 1, 0), (60, 3, 2)]:
            occ = occ_limit / n if occ_limit else None
            cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, partitions=p,
                                  occurrence_threshold=occ)
            t1 = time.time()
            rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
            t2 = time.time()
            want, wst = osr.search(want_sigs, tables=100, min_matches=5, partitions=p,
                                   occurrence_threshold=occ, exclusion_windows=excl)
            t3 = time.time()
            ok = rec.tobytes() == want.tobytes() and same_stats(st.to_dict(), wst)
            bad += not ok
            print(f"  occ_limit={occ_limit} p={p} excl={excl}: {rec.size} triplets, "
                  f"{st.distinct_pairs} distinct pairs, {st.filtered_fingerprints} filtered -> "
                  f"{'IDENTICAL' if ok else 'MISMATCH'} (gpu {t2 - t1:.2f} s, oracle {t3 - t2:.1f} s)",
                  flush=True)
            if use_ref and n == ns[0]:
                ref = os.path.join(ROOT, "baseline", "_ref")
                sys.path.insert(0, ref)
                from quakescan import lsh_search as rls
                rc = rls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, partitions=p,
                                      occurrence_threshold=occ)
                t4 = time.time()
                rrec, rst = rls.search_signatures(want_sigs, rc, exclusion_windows=excl)
                t5 = time.time()
                ok = rec.tobytes() == rrec.tobytes() and same_stats(st.to_dict(), rst.to_dict())
                bad += not ok
                print(f"    reference search_signatures (baseline/_ref): "
                      f"{'IDENTICAL' if ok else 'MISMATCH'} ({t5 - t4:.1f} s)", flush=True)
    print("ALL IDENTICAL" if bad == 0 else f"{bad} MISMATCHES")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
