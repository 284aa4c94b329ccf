"""LSH similarity search on the B200 — drop-in for reference lsh_search.py.

Public surface of the reference module (lsh_search.py:35-333): TRIPLET_DTYPE,
PROFILES, SearchConfig, SearchStats, detection_probability, partition_bounds,
search_signatures, exclusion_windows_for, search_fingerprints.  Results are
identical to the reference's: triplets (dt, idx1, sim) sorted by (dt, idx1),
the same occurrence-filter decisions (including the order-dependent
per-partition exclusion semantics of lsh_search.py:244-287) and the same
SearchStats fields.

Every stage runs in sm_100a kernels through the C ABI (csrc/qs_lsh.cu,
csrc/qs_sort.cu); this module only validates, allocates device buffers
(torch's caching allocator) and sequences the launches.
"""

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ConsistencyError, ParameterError
from .minmax_hash import HashMapping, gen_hash_mapping

TRIPLET_DTYPE = np.dtype([("dt", "<u8"), ("idx1", "<u8"), ("sim", "<u4")])

# (hash_funcs, min_matches) presets (lsh_search.py:40-42)
PROFILES = {"baseline": (6, 5), "optimized": (8, 2)}

_HIST_LEN = 1 << 16
# MATCHED pass counts lazily (exact sims completed for filter survivors only)
_LAZY_COUNTS = os.environ.get("QS_LAZY_COUNTS", "1") != "0"
# occurrence-filtered MATCHED pass: tables [0, _CORE_SPLIT) first, then the rest
# with pairs of two already-core fingerprints skipped (matched_core_skip).  At
# cfg1 the first 32 tables prove the noise-group members core (MATCHED 218 ->
# 189 ms); splits of 4-16 tables prove too few of them and only add launches
# (220-199 ms, tools/gpu_r02at.sh)
_CORE_SPLIT = int(os.environ.get("QS_CORE_SPLIT", "32"))
_cap_hint = {}


@dataclass
class SearchConfig:
    tables: int = 100
    hash_funcs: int = 6
    min_matches: int = 5
    seed: int = 0
    partitions: int = 1
    near_repeat_exclusion_s: float | None = None  # None -> window length
    occurrence_threshold: float | None = None

    def validate(self) -> None:
        if self.tables < 1:
            raise ParameterError("tables must be >= 1")
        if self.hash_funcs < 2 or self.hash_funcs % 2:
            raise ParameterError("hash_funcs must be a positive even number")
        if not 1 <= self.min_matches <= self.tables:
            raise ParameterError("min_matches must be in [1, tables]")
        if self.partitions < 1:
            raise ParameterError("partitions must be >= 1")
        if self.occurrence_threshold is not None and not 0 < self.occurrence_threshold <= 1:
            raise ParameterError("occurrence_threshold must be in (0, 1]")
        if self.near_repeat_exclusion_s is not None and self.near_repeat_exclusion_s < 0:
            raise ParameterError("near_repeat_exclusion_s must be >= 0")


@dataclass
class SearchStats:
    n_fingerprints: int = 0
    n_queries: int = 0
    partitions: list = field(default_factory=list)
    lookups_total: int = 0
    distinct_pairs: int = 0
    emitted_triplets: int = 0
    filtered_fingerprints: int = 0
    peak_table_entries: int = 0
    n_buckets: int = 0
    top_bucket_mass: float = 0.0  # share of entries in the largest 0.1% buckets
    max_bucket: int = 0

    @property
    def lookups_per_query(self) -> float:
        return self.lookups_total / self.n_queries if self.n_queries else 0.0

    @property
    def selectivity(self) -> float:
        """Mean fraction of the dataset compared per query."""
        n = self.n_fingerprints
        return 2.0 * self.distinct_pairs / (n * n) if n else 0.0

    def to_dict(self) -> dict:
        return {
            "n_fingerprints": self.n_fingerprints,
            "n_queries": self.n_queries,
            "partitions": [[int(a), int(b)] for a, b in self.partitions],
            "lookups_total": int(self.lookups_total),
            "lookups_per_query": self.lookups_per_query,
            "distinct_pairs": int(self.distinct_pairs),
            "selectivity": self.selectivity,
            "emitted_triplets": int(self.emitted_triplets),
            "filtered_fingerprints": int(self.filtered_fingerprints),
            "peak_table_entries": int(self.peak_table_entries),
            "n_buckets": int(self.n_buckets),
            "top_bucket_mass": self.top_bucket_mass,
            "max_bucket": int(self.max_bucket),
        }


def detection_probability(s: float, k: int, m: int, t: int) -> float:
    """P(a pair with Jaccard s matches in >= m of t tables), p = s**k
    (lsh_search.py:112-136; scalar host math, not a hot path)."""
    if not 0.0 <= s <= 1.0:
        raise ParameterError("similarity must be in [0, 1]")
    if k < 1 or t < 1 or not 1 <= m <= t:
        raise ParameterError("need k >= 1 and 1 <= m <= t")
    p = s ** k
    if p <= 0.0:
        return 0.0
    if p >= 1.0:
        return 1.0
    log_p = k * math.log(s)
    log_q = math.log1p(-p)
    lg_t = math.lgamma(t + 1)
    terms = [lg_t - math.lgamma(i + 1) - math.lgamma(t - i + 1) + i * log_p + (t - i) * log_q
             for i in range(m, t + 1)]
    top = max(terms)
    return min(1.0, math.exp(top) * sum(math.exp(x - top) for x in terms))


def partition_bounds(n: int, partitions: int) -> list[tuple[int, int]]:
    """Split [0, n) into near-even contiguous index ranges (lsh_search.py:139-144)."""
    if partitions < 1:
        raise ParameterError("partitions must be >= 1")
    edges = np.linspace(0, n, min(partitions, max(1, n)) + 1, dtype=int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def exclusion_windows_for(fps, cfg: SearchConfig) -> int:
    """Near-repeat suppression radius in window-index units (lsh_search.py:306-311)."""
    excl_s = cfg.near_repeat_exclusion_s
    if excl_s is None:
        excl_s = fps.window_len_s
    return int(math.ceil(excl_s / fps.window_lag_s)) if excl_s > 0 else 0


# ---------------------------------------------------------------- device path

class DeviceSearch:
    """Device buffers + launches of one search over the search layout.

    keys: (t, n) int64 table-major, rkeys: (n, t) int64 row-major (mix64 of
    the signature words), tags: (2, n, ceil(t/32), 8) int32 CUDA tensors.
    `tables` (optional, ascending global table ids) restricts the buckets to
    those tables — one rank's share of a table-sharded search (sharded.py);
    `keys` then holds either all t tables or only these rows.  rkeys/tags
    always cover all t tables (the first-colliding-table rule looks at every
    earlier table).  Records per-stage CUDA event times when `timing` is set."""

    MODE_FULL, MODE_MATCHED, MODE_DISTINCT = 0, 1, 2

    def __init__(self, keys, rkeys, tags, n: int, t: int, timing: bool = False, tables=None):
        self.torch = nat.torch()
        self.rkeys, self.tags, self.n, self.t = rkeys, tags, n, t
        self.dev = keys.device
        self.table_ids = None
        if tables is not None and list(tables) != list(range(t)):
            ids = self.torch.as_tensor(list(tables), dtype=self.torch.int64)
            if keys.shape[0] != len(ids):
                keys = keys.index_select(0, ids.to(self.dev))
            self.table_ids = ids.to(self.torch.int32).to(self.dev)
        self.keys = keys
        self.kt = int(keys.shape[0])
        self.timing = timing
        self.events = []
        self.launches = 0

    def _mark(self, name):
        if self.timing:
            ev = self.torch.cuda.Event(enable_timing=True)
            ev.record()
            self.events.append((name, ev))

    def stage_times_ms(self):
        out = {}
        for (a, ea), (_, eb) in zip(self.events[:-1], self.events[1:]):
            out[a] = out.get(a, 0.0) + ea.elapsed_time(eb)
        return out

    def _empty(self, nbytes):
        return self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.dev)

    def buckets(self):
        torch, n, t = self.torch, self.n, self.kt
        lib = nat.lib()
        self._mark("buckets")
        self.sids = torch.empty((t, n), dtype=torch.int32, device=self.dev)
        flags = torch.empty((t, n), dtype=torch.uint8, device=self.dev)
        # tables are independent: big searches (cfg3: N = 3.15e7) build them in
        # chunks so the sort workspace (~20 B per member and table) stays bounded
        budget = float(os.environ.get("QS_BUCKET_WS_GB", "24")) * 2**30
        per_table = lib.qs_lsh_bucket_flags_ws_bytes(n, 1)
        tc = max(1, min(t, int(budget // max(1, per_table))))
        ws = self._empty(lib.qs_lsh_bucket_flags_ws_bytes(n, tc))
        for t0 in range(0, t, tc):
            t1 = min(t, t0 + tc)
            nat.call("qs_lsh_build_bucket_flags", nat.ptr(self.keys[t0:t1]), n, t1 - t0,
                     nat.ptr(self.sids[t0:t1]), nat.ptr(flags[t0:t1]), nat.ptr(ws), ws.numel(),
                     nat.stream())
        del ws
        self.launches += 3 * 3 + 5
        self._mark("list")
        lws = self._empty(lib.qs_lsh_list_flags_ws_bytes(n, t))
        counts = torch.zeros(2, dtype=torch.int64, device=self.dev)
        nat.call("qs_lsh_list_buckets_flags", nat.ptr(flags), n, t, None, None, None, None,
                 nat.ptr(counts), nat.ptr(lws), lws.numel(), nat.stream())
        nb, heads = (int(v) for v in counts.tolist())
        self.nb, self.heads = nb, heads
        self.bstart = torch.empty(max(nb, 1), dtype=torch.int64, device=self.dev)
        self.bsize = torch.empty(max(nb, 1), dtype=torch.int32, device=self.dev)
        self.btab = torch.empty(max(nb, 1), dtype=torch.int32, device=self.dev)
        if nb:
            nat.call("qs_lsh_list_buckets_flags", nat.ptr(flags), n, t, nat.ptr(self.bstart),
                     nat.ptr(self.bsize), nat.ptr(self.btab), nat.ptr(self.table_ids),
                     nat.ptr(counts), nat.ptr(lws), lws.numel(), nat.stream())
        self.launches += 7 + 8
        self.full = (self.sids, self.bstart, self.bsize, self.btab, self.nb)

    def compact(self, emask):
        """Bucket list with excluded members removed (partitions == 1).  The same
        pass computes the single-partition bucket statistics for this emask
        (returned later by bucket_stats)."""
        torch, lib = self.torch, nat.lib()
        self._mark("compact")
        nb = self.nb
        sids2 = torch.empty(max(1, self.n * self.kt), dtype=torch.int32, device=self.dev)
        bstart2 = torch.empty(max(nb, 1), dtype=torch.int64, device=self.dev)
        bsize2 = torch.empty(max(nb, 1), dtype=torch.int32, device=self.dev)
        btab2 = torch.empty(max(nb, 1), dtype=torch.int32, device=self.dev)
        counts = torch.zeros(2, dtype=torch.int64, device=self.dev)
        hist = torch.zeros(_HIST_LEN, dtype=torch.int64, device=self.dev)
        big_cap = max(1024, nb // 64)
        big = torch.empty(big_cap, dtype=torch.int32, device=self.dev)
        out = torch.zeros(4, dtype=torch.int64, device=self.dev)
        ws = self._empty(lib.qs_lsh_compact_ws_bytes(nb))
        nat.call("qs_lsh_compact_buckets", nat.ptr(self.sids), nat.ptr(self.bstart),
                 nat.ptr(self.bsize), nat.ptr(self.btab), nb, nat.ptr(emask), nat.ptr(sids2),
                 nat.ptr(bstart2), nat.ptr(bsize2), nat.ptr(btab2), nat.ptr(counts),
                 nat.ptr(hist), _HIST_LEN, nat.ptr(big), big_cap, nat.ptr(out), nat.ptr(ws),
                 ws.numel(), nat.stream())
        self.launches += 2 + 2 * 3
        nb2 = int(counts[0].item())
        self._compact_stats = (emask, hist, big, big_cap, out)
        # sizes of the compacted buckets (the DISTINCT pass's work; bench.py roofline)
        self.compact_sizes = bsize2[:nb2]
        return (sids2, bstart2, bsize2, btab2, nb2)

    def pairs(self, mode, m, excl, emask, edges, p, lists=None, cap=None, table_range=None,
              core_count=None):
        """Enumerate; returns (pair_key int64, pair_sim int32, n_matched, distinct).

        table_range: (lo, hi) restricts the pass to the buckets of tables
        [lo, hi); core_count: per-bucket core counts of core-first `lists`
        (qs_lsh_pairs_ex: pairs of two core members are skipped)."""
        torch, lib = self.torch, nat.lib()
        sids, bstart, bsize, btab, nb = lists if lists is not None else self.full
        self._mark(("pairs_full", "pairs_matched", "pairs_distinct")[mode])
        key = ("cap", self.n, self.t, mode)
        if mode == self.MODE_DISTINCT:
            cap = 0
        elif cap is None:
            cap = max(1 << 16, _cap_hint.get(key, 4 * self.n))
        counters = torch.zeros(2, dtype=torch.int64, device=self.dev)
        ws = self._empty(lib.qs_lsh_pairs_ws_bytes(nb))
        lazy = mode == self.MODE_MATCHED and _LAZY_COUNTS
        W = (self.t + 31) // 32
        while True:
            pk = torch.empty(max(cap, 1), dtype=torch.int64, device=self.dev)
            ps = torch.empty(max(cap, 1), dtype=torch.int32, device=self.dev)
            rest = torch.empty(max(cap, 1) * W, dtype=torch.int32, device=self.dev) if lazy else None
            counters.zero_()
            if table_range is None and core_count is None:
                nat.call("qs_lsh_pairs", nat.ptr(sids), nat.ptr(bstart), nat.ptr(bsize),
                         nat.ptr(btab), nb, nat.ptr(self.rkeys), nat.ptr(self.tags), self.n,
                         self.t, m, excl, nat.ptr(emask), nat.ptr(edges), p, mode, nat.ptr(pk),
                         nat.ptr(ps), nat.ptr(rest), cap, nat.ptr(counters), nat.ptr(ws),
                         ws.numel(), nat.stream())
            else:
                lo, hi = table_range if table_range is not None else (0, 0xFFFFFFFF)
                nat.call("qs_lsh_pairs_ex", nat.ptr(sids), nat.ptr(bstart), nat.ptr(bsize),
                         nat.ptr(btab), nb, nat.ptr(self.rkeys), nat.ptr(self.tags), self.n,
                         self.t, m, excl, nat.ptr(emask), nat.ptr(edges), p, mode, nat.ptr(pk),
                         nat.ptr(ps), nat.ptr(rest), cap, nat.ptr(counters), nat.ptr(ws),
                         ws.numel(), lo, hi, nat.ptr(core_count), nat.stream())
            # word bounds + per launched table word: 7 planning kernels, 2x3 scan kernels, pairs
            words = (self.t + 31) // 32
            if mode == self.MODE_MATCHED:
                words = min(words, (self.t - m) // 32 + 1)
            self.launches += 1 + 14 * words
            distinct, matched = (int(v) for v in counters.tolist())
            if matched <= cap:
                break
            cap = int(matched * 1.1) + 1024
        if mode != self.MODE_DISTINCT:
            _cap_hint[key] = max(_cap_hint.get(key, 0), int(matched * 1.1) + 1024)
        pk, ps = pk[:matched], ps[:matched]
        # lazily counted sims travel with this pk until complete_sims()
        if lazy:
            self._lazy = (pk, rest[: matched * W])
        return pk, ps, matched, distinct

    def core_first(self, core, table_lo):
        """Core-first copies of the member lists of tables >= table_lo and the
        per-bucket core counts (qs_lsh_core_first)."""
        torch = self.torch
        sids2 = torch.empty_like(self.sids)
        nc = torch.empty(max(self.nb, 1), dtype=torch.int32, device=self.dev)
        nat.call("qs_lsh_core_first", nat.ptr(self.sids), nat.ptr(self.bstart), nat.ptr(self.bsize),
                 nat.ptr(self.btab), self.nb, table_lo, nat.ptr(core), nat.ptr(sids2), nat.ptr(nc),
                 nat.stream())
        self.launches += 1
        return (sids2, self.bstart, self.bsize, self.btab, self.nb), nc

    def matched_core_skip(self, m, excl, edges, threshold):
        """Pass 1 of the occurrence filter (partitions == 1) in two steps: the
        buckets of the first _CORE_SPLIT tables as usual; then, with the fingerprints
        whose degree over those pairs already exceeds the limit marked core, the
        later tables over core-first lists with pairs of two core members
        skipped.  A partial degree is a lower bound of the full one, so those
        fingerprints are core in the full count too; a skipped pair only joins
        two excluded fingerprints and changes no degree decision, exclusion or
        emitted triplet (lsh_search.py:256-287).  Returns what pairs() returns
        for the whole MATCHED pass (the pair list is a different but equally
        sufficient set: the same core set, exclusions and surviving pairs)."""
        torch = self.torch
        t1 = min(self.t, _CORE_SPLIT)
        pk0, ps0, m0, _ = self.pairs(self.MODE_MATCHED, m, excl, None, edges, 1, table_range=(0, t1))
        lz0 = self._lazy[1] if getattr(self, "_lazy", None) is not None else None
        deg = self.occ_degree(pk0, m0, edges, 1)
        core = (deg.to(torch.float64) > float(threshold) * self.n).to(torch.uint8)
        lists, nc = self.core_first(core, t1)
        pk1, ps1, m1, _ = self.pairs(self.MODE_MATCHED, m, excl, None, edges, 1, lists=lists,
                                     table_range=(t1, self.t), core_count=nc)
        lz1 = self._lazy[1] if getattr(self, "_lazy", None) is not None else None
        if self.timing:  # measurement: core-core pairs left out (bench.py roofline)
            sk = torch.zeros(1, dtype=torch.int64, device=self.dev)
            nat.call("qs_lsh_core_skipped", nat.ptr(self.bsize), nat.ptr(self.btab), nat.ptr(nc),
                     self.nb, self.t, m, t1, nat.ptr(sk), nat.stream())
            self.core_skipped = sk
        del lists, nc
        pk = torch.cat([pk0, pk1])
        ps = torch.cat([ps0, ps1])
        if lz0 is not None and lz1 is not None:
            self._lazy = (pk, torch.cat([lz0, lz1]))
        return pk, ps, m0 + m1, 0

    def complete_sims(self, pk, ps, matched):
        """Exact sims for lazily counted MATCHED pairs (the tables left
        unexamined once a pair reached m are confirmed now, for the pairs that
        survived the filter only)."""
        lz = getattr(self, "_lazy", None)
        if lz is None or lz[0] is not pk:
            return
        if matched:
            nat.call("qs_lsh_complete_sims", nat.ptr(pk), nat.ptr(ps), nat.ptr(lz[1]), matched,
                     nat.ptr(self.rkeys), self.t, nat.stream())
            self.launches += 1
        self._lazy = None

    def occurrence(self, pk, ps, matched, threshold, edges, p):
        torch = self.torch
        self._mark("filter")
        emask = torch.empty(self.n, dtype=torch.uint8, device=self.dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
        ws = torch.empty(self.n, dtype=torch.int32, device=self.dev)
        nat.call("qs_lsh_occurrence_filter", nat.ptr(pk), nat.ptr(ps), matched, self.n,
                 float(threshold), nat.ptr(edges), p, nat.ptr(emask), nat.ptr(cnt), nat.ptr(ws),
                 nat.stream())
        self.launches += 4
        return emask, int(cnt.item())

    # the occurrence filter in three steps (table-sharded searches reduce the
    # degree vector with SUM and the mark vector with MAX between them)
    def occ_degree(self, pk, matched, edges, p):
        self._mark("filter")
        deg = self.torch.zeros(self.n, dtype=self.torch.int32, device=self.dev)
        nat.call("qs_lsh_occ_degree", nat.ptr(pk), matched, nat.ptr(edges), p, nat.ptr(deg),
                 nat.stream())
        self.launches += 1
        return deg

    def occ_mark(self, pk, matched, deg, threshold, edges, p):
        mark = self.torch.empty(self.n, dtype=self.torch.uint8, device=self.dev)
        nat.call("qs_lsh_occ_mark", nat.ptr(pk), matched, nat.ptr(deg), self.n, float(threshold),
                 nat.ptr(edges), p, nat.ptr(mark), nat.stream())
        self.launches += 2
        return mark

    def occ_finish(self, mark):
        cnt = self.torch.zeros(1, dtype=self.torch.int64, device=self.dev)
        nat.call("qs_lsh_occ_finish", nat.ptr(mark), self.n, nat.ptr(cnt), nat.stream())
        self.launches += 1
        return mark, int(cnt.item())

    def filter_pairs(self, pk, ps, matched, emask, edges, p):
        torch = self.torch
        opk = torch.empty(max(matched, 1), dtype=torch.int64, device=self.dev)
        ops = torch.empty(max(matched, 1), dtype=torch.int32, device=self.dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
        lz = getattr(self, "_lazy", None)
        rest = lz[1] if lz is not None and lz[0] is pk else None
        W = (self.t + 31) // 32
        orest = torch.empty(max(matched, 1) * W, dtype=torch.int32, device=self.dev) if rest is not None else None
        nat.call("qs_lsh_filter_pairs", nat.ptr(pk), nat.ptr(ps), nat.ptr(rest), W, matched,
                 nat.ptr(emask), nat.ptr(edges), p, nat.ptr(opk), nat.ptr(ops), nat.ptr(orest),
                 nat.ptr(cnt), nat.stream())
        self.launches += 1
        k = int(cnt.item())
        opk, ops = opk[:k], ops[:k]
        if rest is not None:
            self._lazy = (opk, orest[: k * W])
        return opk, ops, k

    def bucket_stats(self, emask, edges, p):
        torch = self.torch
        cached = getattr(self, "_compact_stats", None)
        if p == 1 and cached is not None and cached[0] is emask:
            _, hist, big, big_cap, out = cached
            looks, pieces, n_big, mx = (int(v) for v in out.tolist())
            if n_big > big_cap:
                raise RuntimeError("bucket size overflow list too small")
            return looks, pieces, mx, hist.cpu().numpy(), big[:n_big].cpu().numpy()
        self._mark("stats")
        hist = torch.zeros(_HIST_LEN, dtype=torch.int64, device=self.dev)
        big_cap = max(1024, self.nb // 64)
        big = torch.empty(big_cap, dtype=torch.int32, device=self.dev)
        out = torch.zeros(4, dtype=torch.int64, device=self.dev)
        nat.call("qs_lsh_bucket_stats", nat.ptr(self.sids), nat.ptr(self.bstart), nat.ptr(self.bsize),
                 self.nb, nat.ptr(emask), nat.ptr(edges), p, nat.ptr(hist), _HIST_LEN, nat.ptr(big),
                 big_cap, nat.ptr(out), nat.stream())
        self.launches += 1
        looks, pieces, n_big, mx = (int(v) for v in out.tolist())
        if n_big > big_cap:
            raise RuntimeError("bucket size overflow list too small")
        return looks, pieces, mx, hist.cpu().numpy(), big[:n_big].cpu().numpy()

    def finalize(self, pk, ps, matched):
        torch, lib = self.torch, nat.lib()
        self._mark("sort")
        trip = torch.empty(matched * 20, dtype=torch.uint8, device=self.dev)
        if matched:
            ws = self._empty(lib.qs_sort_pairs_ws_bytes(matched))
            key_bits = 32 + max(1, int(self.n).bit_length())
            nat.call("qs_lsh_finalize", nat.ptr(pk), nat.ptr(ps), matched, key_bits,
                     nat.ptr(trip), nat.ptr(ws), ws.numel(), nat.stream())
            self.launches += 3 * ((key_bits + 7) // 8) + 1
        self._mark("end")
        return trip


def _top_mass(hist, big, n_buckets, total):
    top = max(1, int(math.ceil(0.001 * n_buckets)))
    need, acc = top, 0
    for v in sorted(big.tolist(), reverse=True):
        if need == 0:
            break
        acc += v
        need -= 1
    idx = np.flatnonzero(hist)[::-1]
    for s in idx:
        if need == 0:
            break
        take = min(need, int(hist[s]))
        acc += take * int(s)
        need -= take
    return float(acc / total) if total else 0.0


def run_search(keys, rkeys, tags, n: int, t: int, cfg: SearchConfig, exclusion_windows: int,
               timing: bool = False):
    """Full search over the device search layout. Returns (triplets: uint8 CUDA
    tensor of TRIPLET_DTYPE records, SearchStats, DeviceSearch)."""
    torch = nat.torch()
    stats = SearchStats(n_fingerprints=n)
    bounds = partition_bounds(n, cfg.partitions) if n else []
    stats.partitions = bounds
    ds = DeviceSearch(keys, rkeys, tags, n, t, timing=timing)
    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device="cuda"), stats, ds
    p = len(bounds)
    edges_h = np.array([a for a, _ in bounds] + [bounds[-1][1]], dtype=np.int64)
    edges = torch.from_numpy(edges_h).to(keys.device)
    stats.peak_table_entries = int(max(b - a for a, b in bounds)) * t
    excl = int(exclusion_windows)
    if excl < 0:
        raise ParameterError("exclusion_windows must be >= 0")
    m = cfg.min_matches
    ds.buckets()
    emask, n_ex = None, 0
    if cfg.occurrence_threshold is None:
        pk, ps, matched, distinct = ds.pairs(ds.MODE_FULL, m, excl, None, edges, p)
    else:
        # pass 1: matched pairs (no exclusions yet) -> occurrence filter; with one
        # partition and _CORE_SPLIT < t <= 128 the later tables skip pairs of two
        # fingerprints the first tables already prove core (QS_CORE_SKIP=0: off)
        if p == 1 and _CORE_SPLIT < t <= 128 and os.environ.get("QS_CORE_SKIP", "1") != "0":
            pk, ps, matched, _ = ds.matched_core_skip(m, excl, edges, cfg.occurrence_threshold)
        else:
            pk, ps, matched, _ = ds.pairs(ds.MODE_MATCHED, m, excl, None, edges, p)
        emask, n_ex = ds.occurrence(pk, ps, matched, cfg.occurrence_threshold, edges, p)
        if n_ex == 0:
            emask = None
            _, _, _, distinct = ds.pairs(ds.MODE_DISTINCT, m, excl, None, edges, p)
        else:
            pk, ps, matched = ds.filter_pairs(pk, ps, matched, emask, edges, p)
            if p == 1:
                lists = ds.compact(emask)
                _, _, _, distinct = ds.pairs(ds.MODE_DISTINCT, m, excl, None, edges, p, lists=lists)
                del lists
            else:
                _, _, _, distinct = ds.pairs(ds.MODE_DISTINCT, m, excl, emask, edges, p)
    ds.complete_sims(pk, ps, matched)
    looks, pieces, mx, hist, big = ds.bucket_stats(emask, edges, p)
    trip = ds.finalize(pk, ps, matched)
    fill_stats(stats, n, t, looks, pieces, mx, hist, big, ds.heads - ds.nb, distinct, matched, n_ex)
    return trip, stats, ds


def fill_stats(stats, n, t, looks, pieces, mx, hist, big, singles, distinct, matched, n_ex):
    """SearchStats fields (lsh_search.py:295-302) from bucket-walk totals."""
    stats.lookups_total = looks
    stats.distinct_pairs = distinct
    stats.emitted_triplets = matched
    stats.filtered_fingerprints = n_ex
    stats.n_queries = n - n_ex
    stats.n_buckets = pieces + singles
    stats.max_bucket = max(mx, 1 if singles else 0)
    hist = np.array(hist, dtype=np.int64, copy=True)
    hist[1] += singles
    stats.top_bucket_mass = _top_mass(hist, big, stats.n_buckets, n * t)
    return stats


def _empty_triplets():
    return np.empty(0, dtype=TRIPLET_DTYPE)


def search_signatures(sigs, cfg: SearchConfig, exclusion_windows: int = 0):
    """Find similar pairs among an (n, t) signature matrix (lsh_search.py:222-303).

    Returns (triplets, stats); triplets is a TRIPLET_DTYPE record array sorted
    by (dt, idx1) — a host numpy array for host input, a CUDA uint8 tensor of
    packed records for CUDA tensor input."""
    cfg.validate()
    torch = nat.torch()
    on_device = nat.is_device_tensor(sigs)
    if on_device:
        if sigs.dim() != 2 or sigs.shape[1] != cfg.tables:
            raise ParameterError("signature matrix does not match cfg.tables")
        sdev = sigs.contiguous()
        if sdev.dtype != torch.int64:
            sdev = sdev.to(torch.int64)
    else:
        arr = np.ascontiguousarray(sigs, dtype=np.uint64)
        if arr.ndim != 2 or arr.shape[1] != cfg.tables:
            raise ParameterError("signature matrix does not match cfg.tables")
        sdev = None
    n = int(sdev.shape[0] if on_device else arr.shape[0])
    if n >= 2**32:
        raise ParameterError("more than 2**32 fingerprints are not supported")
    t = cfg.tables
    if n == 0:
        stats = SearchStats(n_fingerprints=0)
        return (_empty_triplets() if not on_device else
                torch.empty(0, dtype=torch.uint8, device=sigs.device)), stats
    if not on_device:
        sdev = torch.from_numpy(arr.view(np.int64)).to("cuda")
    keys, rkeys, tags = prep_signatures(sdev)
    trip, stats, _ = run_search(keys, rkeys, tags, n, t, cfg, exclusion_windows)
    if on_device:
        return trip, stats
    return trip.cpu().numpy().view(TRIPLET_DTYPE), stats


def prep_signatures(sdev):
    """Search layout (keys, rkeys, tags) of a CUDA int64 (n, t) signature matrix."""
    torch = nat.torch()
    n, t = (int(v) for v in sdev.shape)
    W = (t + 31) // 32
    keys = torch.empty((t, n), dtype=torch.int64, device=sdev.device)
    rkeys = torch.empty((n, t), dtype=torch.int64, device=sdev.device)
    tags = torch.empty((2, n, W, 8), dtype=torch.int32, device=sdev.device)
    nat.call("qs_lsh_prep", nat.ptr(sdev), n, t, nat.ptr(keys), nat.ptr(rkeys), nat.ptr(tags),
             nat.stream())
    return keys, rkeys, tags


_COPY_POOL = None


def _copy_pool():
    global _COPY_POOL
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        want = int(os.environ.get("QS_COPY_THREADS", "16"))
        _COPY_POOL = ThreadPoolExecutor(max(1, min(want, len(os.sched_getaffinity(0)))))
    return _COPY_POOL


def _to_device_staged(arr: np.ndarray, chunk_bytes: int = 256 << 20, on_chunk=None, out=None,
                      narrow_f32: bool = False):
    """Host -> device copy of a numpy array in chunks on a copy stream.
    `on_chunk(done)` is called after each chunk is ordered on the compute
    stream (work on the first `done` elements overlaps the remaining copies).
    `out`: an existing CUDA tensor of the same shape to fill.

    A page-locked array is copied by DMA from where it lies.  A pageable one
    goes through two pinned staging buffers: the host pass into one buffer is
    split over a thread pool (the C helpers and numpy release the GIL) while
    the DMA of the other runs.  `narrow_f32`: a float64 array is narrowed to
    float32 on the way (`out` is float32; qs_host_pack_f32) — returns None as
    soon as a value is not exactly representable, the caller then repeats the
    copy in float64."""
    torch = nat.torch()
    flat = arr.reshape(-1)
    if out is None:
        out = torch.empty(arr.shape, dtype=torch.from_numpy(flat[:0]).dtype, device="cuda")
    if flat.size == 0:
        return out
    dst = out.view(-1)
    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    copy.wait_stream(compute)  # dst's allocation is ordered on the compute stream
    if not narrow_f32 and _host_pinned(flat):
        per = max(1, chunk_bytes // flat.itemsize)
        cstream = nat.ctypes.c_void_p(copy.cuda_stream)
        isz = flat.itemsize
        for a in range(0, flat.size, per):
            b = min(flat.size, a + per)
            nat.call("qs_memcpy_h2d_async", nat.ctypes.c_void_p(dst.data_ptr() + a * isz),
                     nat.ctypes.c_void_p(flat.ctypes.data + a * isz), (b - a) * isz, cstream)
            ev = torch.cuda.Event()
            ev.record(copy)
            compute.wait_event(ev)
            if on_chunk is not None:
                on_chunk(b)
        out.record_stream(copy)
        return out
    per = max(1, chunk_bytes // dst.element_size())
    stage = [torch.empty(min(per, flat.size), dtype=dst.dtype, pin_memory=True) for _ in range(2)]
    done = [None, None]
    pool = _copy_pool()
    nthr = pool._max_workers
    lib = nat.lib()
    for k, a in enumerate(range(0, flat.size, per)):
        b = min(flat.size, a + per)
        s = k & 1
        if done[s] is not None:
            done[s].synchronize()
        n = b - a
        step = max(1 << 16, -(-n // nthr))
        if narrow_f32:
            hbase, sbase = stage[s].data_ptr(), flat.ctypes.data

            def pack(i, a=a, n=n, hbase=hbase):
                ok = nat.ctypes.c_int(1)
                lib.qs_host_pack_f32(nat.ctypes.c_void_p(sbase + (a + i) * 8),
                                     nat.ctypes.c_void_p(hbase + i * 4), min(n, i + step) - i,
                                     nat.ctypes.byref(ok))
                return ok.value

            if not all(pool.map(pack, range(0, n, step))):
                copy.synchronize()
                return None
        else:
            host = stage[s].numpy()
            list(pool.map(lambda i: np.copyto(host[i:min(n, i + step)], flat[a + i:a + min(n, i + step)]),
                          range(0, n, step)))
        with torch.cuda.stream(copy):
            dst[a:b].copy_(stage[s][:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        done[s] = ev
        compute.wait_event(ev)
        if on_chunk is not None:
            on_chunk(b)
    out.record_stream(copy)
    return out


def _search_layout(n: int, t: int, device, with_keys: bool = True):
    torch = nat.torch()
    W = (t + 31) // 32
    keys = torch.empty((t, n), dtype=torch.int64, device=device) if with_keys else None
    rkeys = torch.empty((n, t), dtype=torch.int64, device=device)
    tags = torch.empty((2, n, W, 8), dtype=torch.int32, device=device)
    bad = torch.zeros(1, dtype=torch.int32, device=device)
    return keys, rkeys, tags, bad


def signatures_for_search(bits, mapping: HashMapping, with_keys: bool = True):
    """Fused Min-Max kernel writing table-major keys + tags directly (no
    row-major signature round trip). bits: CUDA int32 (n, K)."""
    n, K = bits.shape
    t = mapping.t
    _, plan = mapping.device_plan()
    keys, rkeys, tags, bad = _search_layout(n, t, bits.device, with_keys)
    nat.call("qs_minmax_signatures_search", nat.ptr(bits), n, K, nat.ptr(plan), mapping.d, t,
             mapping.k_half, None, nat.ptr(keys), nat.ptr(rkeys), nat.ptr(tags), nat.ptr(bad),
             nat.stream())
    return keys, rkeys, tags, bad


LAST_H2D_BYTES = 0  # bytes the last signatures_for_search_host call sent over PCIe
LAST_H2D_SPLIT = 0.0  # narrowed share of a page-locked array's rows at the end of that call


def _host_pinned(arr: np.ndarray) -> bool:
    """True when the array's memory is page-locked (allocated or registered
    with CUDA): it is then copied by DMA from where it lies."""
    if arr.size == 0:
        return False
    return bool(nat.lib().qs_host_ptr_pinned(nat.ctypes.c_void_p(arr.ctypes.data)))


def signatures_for_search_host(arr: np.ndarray, mapping: HashMapping, chunk_bytes: int = 256 << 20):
    """Host (n, K) int32 bits -> the search layout, the host->device copy
    pipelined with the signature kernel: the kernel signs each row chunk
    (qs_minmax_signatures_search_rows) on the compute stream as soon as it has
    landed.  A page-locked array is copied by DMA straight from the caller's
    memory; a pageable one goes through two pinned staging buffers (the host
    pass into one buffer split over a thread pool while the other's DMA runs),
    narrowed on the way: to 12-bit fields when d <= 4096 (qs_host_pack_u12: 3/8
    of the staging writes and DMA bytes; a chunk holding an index above 4095
    switches the call to the uint16 route), to uint16 when d <= 65535
    (qs_host_pack_u16: half the bytes; out-of-range values saturate and are
    flagged by the kernel's range check); widened again on the device."""
    torch = nat.torch()
    n, K = arr.shape
    t = mapping.t
    _, plan = mapping.device_plan()
    keys, rkeys, tags, bad = _search_layout(n, t, "cuda")
    bdev = torch.empty((n, K), dtype=torch.int32, device="cuda")
    if n == 0:
        return keys, rkeys, tags, bad
    rows_per = max(4, (chunk_bytes // (K * 4)) & ~3)  # chunk starts stay 16-byte aligned
    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    copy.wait_stream(compute)  # bdev's allocation is ordered on the compute stream
    cstream = nat.ctypes.c_void_p(copy.cuda_stream)
    lib = nat.lib()
    global LAST_H2D_BYTES, LAST_H2D_SPLIT
    LAST_H2D_BYTES = 0

    def sign(r0, rows):
        nat.call("qs_minmax_signatures_search_rows", nat.ptr(bdev), n, r0, rows, K, nat.ptr(plan),
                 mapping.d, t, mapping.k_half, None, nat.ptr(keys), nat.ptr(rkeys), nat.ptr(tags),
                 nat.ptr(bad), nat.stream())

    # field width of the narrowed rows: 12 bits when every index fits (d <= 4096
    # and an even K, so that row ranges start on byte boundaries), else 16 bits
    # (d <= 65535), else none.  QS_H2D_NARROW = 0 / 16 / 12 caps it.
    level = os.environ.get("QS_H2D_NARROW", "12")  # "0": off, "16" (or "1"): uint16 only
    width = 0
    if mapping.d <= 0xFFFF and level != "0":
        width = 16
    if mapping.d <= 4096 and K % 2 == 0 and level not in ("0", "1", "16"):
        width = 12
    pinned_src = _host_pinned(arr)
    src_base = arr.ctypes.data if pinned_src else arr.view(np.uint32).ctypes.data
    split = 1.0
    if pinned_src:
        # DMA from the caller's memory.  With narrowing on, the first `split` of
        # every chunk's rows is narrowed by the thread pool (into pinned staging
        # buffers, for the next chunk while this one's copies run) and the rest is
        # copied as it lies: the PCIe link then moves fewer bytes while the host
        # cores stay below their own narrowing rate (QS_H2D_SPLIT, default 0.7:
        # measured on the 16-core B200 box, where the cores narrow ~67 GB/s of
        # source and the link copies ~55 GB/s).
        split = float(os.environ.get("QS_H2D_SPLIT", "0.7")) if width else 0.0
        split = min(1.0, max(0.0, split))
    # Without an explicit QS_H2D_SPLIT the share follows the measured rates of
    # the call itself: the staging pass takes a * s and the chunk's copies
    # b * (w * s + 1 - s) (w = narrowed bytes per source byte), equal at
    # s = b / (a + (1 - w) * b); a and b come from the host clock around the
    # pack and CUDA events around the copies of the chunk two steps back.  The
    # narrowing rate of the host cores and the DMA rate from the caller's pages
    # both vary from box to box (0.46-0.55 s for the same cfg1 call at a fixed
    # 0.7); every split gives identical bytes.
    adaptive = pinned_src and width and "QS_H2D_SPLIT" not in os.environ
    timing = [None, None]  # per staging slot: (split, pack seconds, start event, end event)
    pool = _copy_pool()
    nthr = pool._max_workers
    cap = min(rows_per, n)
    ncap = (cap if adaptive else int(cap * split)) if width else (0 if pinned_src else cap)
    state = {"width": width, "stage": None, "dstage": None}

    def alloc(w):
        # two pinned staging buffers (+ their device twins when the rows are narrowed)
        if ncap == 0:
            return
        row_bytes = K * 4 if w == 0 else (K * 2 if w == 16 else K * 3 // 2)
        nbytes = (ncap * row_bytes + 15) & ~15
        state["stage"] = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        state["dstage"] = ([torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
                           if w else None)
        state["width"] = w

    alloc(width)
    done = [None, None]

    def state_w():
        return {12: 0.375, 16: 0.5}.get(state["width"], 1.0)

    def pack_rows(w, r0, nrow, hbase):
        """Rows [r0, r0 + nrow) into the staging buffer at hbase, split over the
        pool; False when a 12-bit pack met a value above 4095."""
        step = max(1, (1 << 18) // K, -(-nrow // nthr))
        if w == 12 and step % 2:
            step += 1  # even row counts keep every task's start on a byte boundary for any even K
        fits = [True]

        def one(i):
            cnt = min(nrow, i + step) - i
            sp = nat.ctypes.c_void_p(src_base + (r0 + i) * K * 4)
            if w == 12:
                ok = nat.ctypes.c_int(1)
                lib.qs_host_pack_u12(sp, nat.ctypes.c_void_p(hbase + i * K * 3 // 2), cnt * K,
                                     nat.ctypes.byref(ok))
                if not ok.value:
                    fits[0] = False
            elif w == 16:
                lib.qs_host_pack_u16(sp, nat.ctypes.c_void_p(hbase + i * K * 2), cnt * K)
            else:
                nat.ctypes.memmove(hbase + i * K * 4, sp, cnt * K * 4)

        list(pool.map(one, range(0, nrow, step)))
        return fits[0]

    for k, r0 in enumerate(range(0, n, rows_per)):
        rows = min(n, r0 + rows_per) - r0
        sl = k & 1
        if done[sl] is not None:
            done[sl].synchronize()
            if adaptive and timing[sl] is not None:
                s_k, tp, e0, e1 = timing[sl]
                td = e0.elapsed_time(e1) * 1e-3
                if s_k > 0 and tp > 0 and td > 0:
                    a_ = tp / s_k
                    b_ = td / (state_w() * s_k + 1.0 - s_k)
                    split = 0.5 * split + 0.5 * min(1.0, max(0.3, b_ / (a_ + (1.0 - state_w()) * b_)))
                timing[sl] = None
        nrow = min(ncap, int(rows * split)) if pinned_src else rows
        t_pack0 = time.perf_counter()
        if nrow:
            w = state["width"]
            if not pack_rows(w, r0, nrow, state["stage"][sl].data_ptr()):
                # an index above 4095 (invalid for this d): this and the later chunks
                # take the uint16 route, whose saturated values the kernel flags
                for ev_ in done:
                    if ev_ is not None:
                        ev_.synchronize()
                alloc(16)
                w = 16
                pack_rows(16, r0, nrow, state["stage"][sl].data_ptr())
            if adaptive:
                t_pack = time.perf_counter() - t_pack0
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record(copy)  # this chunk's copies start here (or when the stream frees up)
            row_bytes = K * 4 if w == 0 else (K * 2 if w == 16 else K * 3 // 2)
            st_, dst_ = state["stage"][sl], bdev.data_ptr() + r0 * K * 4
            with torch.cuda.stream(copy):
                if w == 0:
                    nat.call("qs_memcpy_h2d_async", nat.ctypes.c_void_p(dst_),
                             nat.ctypes.c_void_p(st_.data_ptr()), nrow * row_bytes, cstream)
                else:
                    dv = state["dstage"][sl]
                    dv[:nrow * row_bytes].copy_(st_[:nrow * row_bytes], non_blocking=True)
                    nat.call("qs_bits_widen_u16" if w == 16 else "qs_bits_widen_u12", nat.ptr(dv),
                             nat.ctypes.c_void_p(dst_), nrow * K, cstream)
            LAST_H2D_BYTES += nrow * row_bytes
        if rows > nrow:  # the rest of a page-locked chunk by DMA from where it lies
            nat.call("qs_memcpy_h2d_async",
                     nat.ctypes.c_void_p(bdev.data_ptr() + (r0 + nrow) * K * 4),
                     nat.ctypes.c_void_p(src_base + (r0 + nrow) * K * 4), (rows - nrow) * K * 4,
                     cstream)
            LAST_H2D_BYTES += (rows - nrow) * K * 4
        ev = torch.cuda.Event(enable_timing=bool(adaptive))
        ev.record(copy)
        done[sl] = ev
        if adaptive and nrow and rows == rows_per:
            timing[sl] = (nrow / rows, t_pack, ev0, ev)
        compute.wait_event(ev)
        sign(r0, rows)
    LAST_H2D_SPLIT = split if pinned_src else 1.0
    bdev.record_stream(copy)
    if state["dstage"]:
        for d_ in state["dstage"]:
            d_.record_stream(copy)
    # a page-locked caller array is read until the last copy has run: the search
    # that follows synchronises (the range flag's .item()) before anything returns
    return keys, rkeys, tags, bad


def search_fingerprints(fps, cfg: SearchConfig, mapping: HashMapping | None = None,
                        workers: int = 1):
    """Signature generation plus similarity search for one channel
    (lsh_search.py:314-333). Returns (triplets, stats, mapping)."""
    cfg.validate()
    if mapping is None:
        mapping = gen_hash_mapping(fps.d, cfg.tables, cfg.hash_funcs, cfg.seed)
    if (mapping.t, mapping.k) != (cfg.tables, cfg.hash_funcs):
        raise ConsistencyError("hash mapping does not match search config")
    if mapping.d != fps.d:
        raise ConsistencyError("hash mapping dimensionality does not match fingerprints")
    torch = nat.torch()
    bits = fps.bits
    on_device = nat.is_device_tensor(bits)
    if on_device:
        bdev = bits.contiguous().to(torch.int32) if bits.dtype != torch.int32 else bits.contiguous()
        if bdev.dim() != 2:
            raise ParameterError("bits must be a 2-D (n, K) array")
    else:
        arr = np.ascontiguousarray(bits, dtype=np.uint32)
        if arr.ndim != 2:
            raise ParameterError("bits must be a 2-D (n, K) array")
        if arr.shape[1] < 1:
            raise ParameterError("fingerprints must have at least one set bit")
    n, K = bdev.shape if on_device else arr.shape
    if K < 1:
        raise ParameterError("fingerprints must have at least one set bit")
    if n >= 2**32:
        raise ParameterError("more than 2**32 fingerprints are not supported")
    excl = exclusion_windows_for(fps, cfg)
    if n == 0:
        empty = _empty_triplets() if not on_device else torch.empty(0, dtype=torch.uint8, device="cuda")
        return empty, SearchStats(n_fingerprints=0), mapping
    if on_device:
        keys, rkeys, tags, bad = signatures_for_search(bdev, mapping)
    else:
        # the range check (minmax_hash.py:107-108) runs on the device, flagged by
        # the signature kernel, instead of a host pass over the whole array
        keys, rkeys, tags, bad = signatures_for_search_host(arr.view(np.int32), mapping)
    if int(bad.item()):
        raise ParameterError("fingerprint bit index out of range for mapping")
    trip, stats, _ = run_search(keys, rkeys, tags, n, cfg.tables, cfg, excl)
    if on_device:
        return trip, stats, mapping
    return trip.cpu().numpy().view(TRIPLET_DTYPE), stats, mapping


# ---------------------------------------------------------------------------
# triplet files (lsh_search.py:336-416)

from . import container as _container  # noqa: E402
from . import hostio  # noqa: E402
from .errors import CorruptInputError  # noqa: E402

TRI_MAGIC = b"QSTR0001"
_TRI_KIND = "triplet"


def write_triplet_file(path, triplets, header: dict) -> None:
    """Binary triplet file, records sorted by (dt, idx1) as given.  Accepts the
    host record array or the packed CUDA uint8 tensor a device search returns
    (streamed to the file through pinned buffers)."""
    if nat.is_device_tensor(triplets):
        if triplets.numel() % TRIPLET_DTYPE.itemsize:
            raise ParameterError("device triplets must be packed 20-byte records")
        count = triplets.numel() // TRIPLET_DTYPE.itemsize
        with open(path, "wb") as f:
            _container.write_preamble(f, TRI_MAGIC, header, count=count)
            hostio.write_device_bytes(f, triplets)
        return
    triplets = np.asarray(triplets, dtype=TRIPLET_DTYPE)
    with open(path, "wb") as f:
        _container.write_preamble(f, TRI_MAGIC, header, count=triplets.size)
        triplets.tofile(f)


def read_triplet_file(path, device: bool = False):
    """-> (records, header); device=True returns the packed CUDA uint8 tensor."""
    with open(path, "rb") as f:
        header, count, off = _container.read_preamble(f, TRI_MAGIC, _TRI_KIND)
        size = os.fstat(f.fileno()).st_size
        _container.check_payload_size(size, off, count, TRIPLET_DTYPE.itemsize, _TRI_KIND)
        if device:
            rec = hostio.read_to_device(f, count * TRIPLET_DTYPE.itemsize)
            if count:
                torch = nat.torch()
                dt = rec.view(count, TRIPLET_DTYPE.itemsize)[:, :8].contiguous().view(torch.int64)
                if int(dt.min().item()) < 1:
                    raise CorruptInputError("triplet with non-positive dt")
            return rec, header
        rec = np.fromfile(f, dtype=TRIPLET_DTYPE, count=count)
    if rec.size and int(rec["dt"].min()) < 1:
        raise CorruptInputError("triplet with non-positive dt")
    return rec, header


def iter_triplet_batches(path, start: int = 0, stop: int | None = None, batch: int = 1 << 16):
    """Yield record batches of rows [start, stop) (lsh_search.py:360-377)."""
    with open(path, "rb") as f:
        _, count, off = _container.read_preamble(f, TRI_MAGIC, _TRI_KIND)
        size = os.fstat(f.fileno()).st_size
        _container.check_payload_size(size, off, count, TRIPLET_DTYPE.itemsize, _TRI_KIND)
        stop = count if stop is None else min(stop, count)
        pos = max(0, start)
        f.seek(off + pos * TRIPLET_DTYPE.itemsize)
        while pos < stop:
            k = min(batch, stop - pos)
            rec = np.fromfile(f, dtype=TRIPLET_DTYPE, count=k)
            if rec.size < k:
                raise CorruptInputError("triplet file truncated")
            yield rec
            pos += k


def read_triplet_header(path) -> dict:
    with open(path, "rb") as f:
        header, count, _ = _container.read_preamble(f, TRI_MAGIC, _TRI_KIND)
    header["count"] = count
    return header


def write_triplet_csv(path, triplets) -> None:
    """CSV interchange form `dt,idx1,sim` (lsh_search.py:387-393)."""
    if nat.is_device_tensor(triplets):
        triplets = triplets.cpu().numpy().view(TRIPLET_DTYPE)
    t = np.asarray(triplets, dtype=TRIPLET_DTYPE)
    body = "".join(f"{a},{b},{c}\n" for a, b, c in zip(t["dt"].tolist(), t["idx1"].tolist(),
                                                        t["sim"].tolist()))
    with open(path, "w", encoding="utf-8") as f:
        f.write("dt,idx1,sim\n")
        f.write(body)


def read_triplet_csv(path) -> np.ndarray:
    with open(path, encoding="utf-8") as f:
        head = f.readline().strip()
        if head != "dt,idx1,sim":
            raise CorruptInputError(f"unexpected triplet CSV header {head!r}")
        rows = []
        for line_no, line in enumerate(f, start=2):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) != 3:
                raise CorruptInputError(f"triplet CSV line {line_no} malformed")
            try:
                rows.append(tuple(int(v) for v in parts))
            except ValueError as exc:
                raise CorruptInputError(f"triplet CSV line {line_no}: {exc}") from exc
    return np.array(rows, dtype=TRIPLET_DTYPE) if rows else np.empty(0, dtype=TRIPLET_DTYPE)
