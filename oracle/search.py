"""ORACLE — test infrastructure only. LSH search restatement (numpy).

Restates reference pkg/src/quakescan/lsh_search.py:
  partition_bounds       :139-144   near-even linspace index ranges
  table build            :157-164   per table stable argsort of member signatures
  bucket sizes           :167-172   run lengths of the sorted column
  pair collection        :175-219   per table, per query: equal-signature members;
                                    lookups counted before masks; canonical c<q,
                                    |q-c| > excl, ~excluded[c]; (q<<32)|c keys,
                                    sorted, run-length = matching tables
  search_signatures      :222-303   partition loop, occurrence filter pass 1
                                    (within-partition degrees, core + matched
                                    neighbours excluded, frozen for later
                                    partitions), pass 2 emission, lexsort (dt, idx1),
                                    bucket statistics
  detection_probability  :112-136   binomial upper tail in log space
Also the all-pairs brute-force oracle of the reference tests
(tests/test_lsh_search.py:25-36).

The numpy traversal is the same vectorised searchsorted algorithm the
reference runs, so `bench.py --impl reference` times a faithful CPU port.
"""

import math

import numpy as np

TRIPLET_DTYPE = np.dtype([("dt", "<u8"), ("idx1", "<u8"), ("sim", "<u4")])


def partition_bounds(n: int, partitions: int):
    edges = np.linspace(0, n, min(partitions, max(1, n)) + 1, dtype=int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def detection_probability(s: float, k: int, m: int, t: int) -> float:
    p = s ** k
    if p <= 0.0:
        return 0.0
    if p >= 1.0:
        return 1.0
    lp, lq, lt = k * math.log(s), math.log1p(-p), math.lgamma(t + 1)
    terms = [lt - math.lgamma(i + 1) - math.lgamma(t - i + 1) + i * lp + (t - i) * lq
             for i in range(m, t + 1)]
    top = max(terms)
    return min(1.0, math.exp(top) * sum(math.exp(x - top) for x in terms))


def _expand(starts, counts):
    total = int(counts.sum())
    if total == 0:
        return np.empty(0, np.int64)
    ends = np.cumsum(counts)
    return np.arange(total, dtype=np.int64) + np.repeat(starts - (ends - counts), counts)


def _pairs(sigs, tables, queries, excl, excluded, want_lookups):
    """(q, c, matches) of distinct canonical pairs; plus lookups before masks."""
    lookups = 0
    chunks = []
    for ti, (col, ids) in enumerate(tables):
        qs = sigs[queries, ti]
        lo = np.searchsorted(col, qs, side="left")
        cnt = np.searchsorted(col, qs, side="right") - lo
        q = np.repeat(queries, cnt)
        c = ids[_expand(lo, cnt)]
        if want_lookups:
            lookups += int((c != q).sum())
        keep = (c < q) & (np.abs(q - c) > excl)
        if excluded is not None:
            keep &= ~excluded[c]
        chunks.append((q[keep].astype(np.uint64) << np.uint64(32)) | c[keep].astype(np.uint64))
    keys = np.concatenate(chunks) if chunks else np.empty(0, np.uint64)
    if keys.size == 0:
        e = np.empty(0, np.int64)
        return e, e, np.empty(0, np.uint32), lookups
    keys.sort()
    first = np.flatnonzero(np.concatenate(([True], keys[1:] != keys[:-1])))
    counts = np.diff(np.append(first, keys.size)).astype(np.uint32)
    u = keys[first]
    return ((u >> np.uint64(32)).astype(np.int64),
            (u & np.uint64(0xFFFFFFFF)).astype(np.int64), counts, lookups)


def search(sigs, tables: int, min_matches: int, partitions: int = 1,
           occurrence_threshold=None, exclusion_windows: int = 0):
    """Returns (triplets TRIPLET_DTYPE sorted by (dt, idx1), stats dict)."""
    sigs = np.ascontiguousarray(sigs, dtype=np.uint64)
    n = sigs.shape[0]
    st = dict(n_fingerprints=n, n_queries=0, partitions=[], lookups_total=0,
              distinct_pairs=0, emitted_triplets=0, filtered_fingerprints=0,
              peak_table_entries=0, n_buckets=0, top_bucket_mass=0.0, max_bucket=0)
    bounds = partition_bounds(n, partitions) if n else []
    st["partitions"] = [list(b) for b in bounds]
    excluded = np.zeros(n, bool) if occurrence_threshold is not None else None
    everyone = np.arange(n, dtype=np.int64)
    sizes_all, out = [], []
    for lo, hi in bounds:
        members = np.arange(lo, hi, dtype=np.int64)
        if excluded is not None:
            members = members[~excluded[lo:hi]]
        if members.size == 0:
            continue
        tbls = []
        for ti in range(tables):
            col = sigs[members, ti]
            order = np.argsort(col, kind="stable")
            scol = col[order]
            tbls.append((scol, members[order]))
            if scol.size:
                edges = np.flatnonzero(np.concatenate(([True], scol[1:] != scol[:-1]), ))
                sizes_all.append(np.diff(np.append(edges, scol.size)))
        st["peak_table_entries"] = max(st["peak_table_entries"], members.size * tables)
        if occurrence_threshold is not None:
            q, c, cnt, _ = _pairs(sigs, tbls, members, exclusion_windows, None, False)
            hit = cnt >= min_matches
            mq, mc = q[hit], c[hit]
            deg = np.bincount(mq, minlength=n) + np.bincount(mc, minlength=n)
            core = deg > occurrence_threshold * members.size
            if core.any():
                new = core.copy()
                touch = core[mq] | core[mc]
                new[mq[touch]] = True
                new[mc[touch]] = True
                st["filtered_fingerprints"] += int((new & ~excluded).sum())
                excluded |= new
        queries = everyone if excluded is None else everyone[~excluded]
        q, c, cnt, looks = _pairs(sigs, tbls, queries, exclusion_windows, excluded, True)
        st["lookups_total"] += looks
        st["distinct_pairs"] += int(q.size)
        hit = cnt >= min_matches
        if hit.any():
            rec = np.empty(int(hit.sum()), TRIPLET_DTYPE)
            rec["dt"] = (q[hit] - c[hit]).astype(np.uint64)
            rec["idx1"] = c[hit].astype(np.uint64)
            rec["sim"] = cnt[hit]
            out.append(rec)
    st["n_queries"] = n if excluded is None else int(n - excluded.sum())
    if out:
        trip = np.concatenate(out)
        trip = trip[np.lexsort((trip["idx1"], trip["dt"]))]
    else:
        trip = np.empty(0, TRIPLET_DTYPE)
    st["emitted_triplets"] = int(trip.size)
    if sizes_all:
        sizes = np.concatenate(sizes_all)
        st["n_buckets"] = int(sizes.size)
        st["max_bucket"] = int(sizes.max())
        top = max(1, int(math.ceil(0.001 * sizes.size)))
        st["top_bucket_mass"] = float(np.sort(sizes)[sizes.size - top:].sum() / sizes.sum())
    st["lookups_per_query"] = st["lookups_total"] / st["n_queries"] if st["n_queries"] else 0.0
    st["selectivity"] = 2.0 * st["distinct_pairs"] / (n * n) if n else 0.0
    return trip, st


def brute_force_triplets(sigs, min_matches: int, excl: int):
    """All-pairs table-match oracle (reference tests/test_lsh_search.py:25-36)."""
    sigs = np.asarray(sigs)
    n = sigs.shape[0]
    res = []
    for b in range(n):
        if b == 0:
            continue
        sims = (sigs[:b] == sigs[b]).sum(axis=1)
        for a in np.flatnonzero(sims >= min_matches):
            if b - a > excl:
                res.append((int(b - a), int(a), int(sims[a])))
    return sorted(res)
