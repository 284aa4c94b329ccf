"""Table-sharded similarity search: one process per GPU, b/world tables each.

The reference search is single-process (lsh_search.py:222-303); its tables
are independent, so the north-star multi-GPU layout gives each rank a share
of the t tables.  Because pair enumeration counts every pair only in the
bucket of its FIRST colliding table (csrc/qs_pairs.cu), exactly one rank
owns each distinct pair: ranks never exchange per-pair counts.  The only
exchanges are the ones the algorithm itself has:

* occurrence filter (lsh_search.py:256-274): the degree vector (N x u32) is
  summed over ranks, every rank derives the same core set, marks the matched
  neighbours it owns, and the N-byte mark vector is max-reduced;
* counters (distinct pairs, lookups, bucket counts) are summed, the largest
  bucket max-reduced, the large-bucket sizes all-gathered for
  top_bucket_mass;
* the matched pairs are gathered on the root rank, which sorts them into the
  canonical (dt, idx1) triplet order — byte-identical to the 1-GPU result.

Every rank needs the row-major keys and tags of all t tables (the
first-colliding-table test looks at earlier tables).  Fingerprint rows are
block-distributed (`row_block`): each rank runs the Min-Max kernel over its
own block only, the row-major keys (8t B/row) and tags (64 B/row at t = 100)
are all-gathered over NVLink, and each rank transposes its own tables' keys
out of the gathered rows and builds buckets for those tables only.

Tables are dealt round-robin (table j -> rank j mod world): the "no earlier
collision" test reads ceil((j+1)/32) tag words, so interleaving balances the
per-rank work better than contiguous blocks.

`run_search_sharded` is written against two small interfaces so the host
protocol can be tested on CPU with gloo (tests/test_sharded_cpu.py): `comm`
(TorchComm over a torch.distributed group) and `engine` (DeviceSearch on the
GPU; a numpy stand-in in the tests).
"""

import numpy as np

from .errors import ParameterError
from .lsh_search import DeviceSearch, SearchStats, fill_stats, partition_bounds


def shard_tables(t: int, world: int, rank: int) -> list[int]:
    """Global table ids owned by `rank` (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError("bad rank/world")
    return list(range(rank, t, world))


class TorchComm:
    """Collectives of the sharded search over a torch.distributed group
    (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def sum_(self, x):
        self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group)
        return x

    def max_(self, x):
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group)
        return x

    def gather_rows(self, x):
        """All-gather a 1-D tensor of per-rank length; returns the list."""
        torch = self.torch
        n = torch.tensor([x.numel()], dtype=torch.int64, device=x.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        cap = max(1, max(sizes))
        buf = torch.zeros(cap, dtype=x.dtype, device=x.device)
        buf[: x.numel()] = x
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(outs, buf, group=self.group)
        return [o[:s] for o, s in zip(outs, sizes)]

    def gather_into(self, out, x):
        """All-gather equal-size blocks: out (world * x.numel() elements) = concat."""
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(out, x, group=self.group)
        else:
            self.dist.all_gather(list(out.view(self.world, *x.shape).unbind(0)), x, group=self.group)
        return out

    def gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


def run_search_sharded(engine, comm, n: int, t: int, cfg, exclusion_windows: int, root: int = 0):
    """One rank's part of a table-sharded search.  `engine` holds this rank's
    tables (DeviceSearch(..., tables=shard_tables(t, world, rank))).

    Returns (triplets, SearchStats, engine): triplets is the full sorted
    TRIPLET_DTYPE byte tensor on `root` and an empty tensor elsewhere; the
    stats are the global ones on every rank."""
    import torch  # CUDA tensors with DeviceSearch, CPU tensors in the gloo tests
    stats = SearchStats(n_fingerprints=n)
    bounds = partition_bounds(n, cfg.partitions) if n else []
    stats.partitions = bounds
    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device=engine.dev), stats, engine
    p = len(bounds)
    edges = torch.tensor([a for a, _ in bounds] + [bounds[-1][1]], dtype=torch.int64,
                         device=engine.dev)
    stats.peak_table_entries = int(max(b - a for a, b in bounds)) * t
    excl = int(exclusion_windows)
    if excl < 0:
        raise ParameterError("exclusion_windows must be >= 0")
    m = cfg.min_matches
    engine.buckets()
    emask, n_ex = None, 0
    if cfg.occurrence_threshold is None:
        pk, ps, matched, distinct = engine.pairs(engine.MODE_FULL, m, excl, None, edges, p)
    else:
        pk, ps, matched, _ = engine.pairs(engine.MODE_MATCHED, m, excl, None, edges, p)
        deg = comm.sum_(engine.occ_degree(pk, matched, edges, p))
        mark = comm.max_(engine.occ_mark(pk, matched, deg, cfg.occurrence_threshold, edges, p))
        del deg
        emask, n_ex = engine.occ_finish(mark)
        if n_ex == 0:
            emask = None
            _, _, _, distinct = engine.pairs(engine.MODE_DISTINCT, m, excl, None, edges, p)
        else:
            pk, ps, matched = engine.filter_pairs(pk, ps, matched, emask, edges, p)
            if p == 1:
                lists = engine.compact(emask)
                _, _, _, distinct = engine.pairs(engine.MODE_DISTINCT, m, excl, None, edges, p,
                                                 lists=lists)
                del lists
            else:
                _, _, _, distinct = engine.pairs(engine.MODE_DISTINCT, m, excl, emask, edges, p)
    engine.complete_sims(pk, ps, matched)
    looks, pieces, mx, hist, big = engine.bucket_stats(emask, edges, p)
    singles = engine.heads - engine.nb
    tot = torch.tensor([distinct, looks, pieces, singles, matched], dtype=torch.int64,
                       device=engine.dev)
    comm.sum_(tot)
    distinct, looks, pieces, singles, matched_all = (int(v) for v in tot.tolist())
    mxt = comm.max_(torch.tensor([mx], dtype=torch.int64, device=engine.dev))
    mx = int(mxt.item())
    hist_t = comm.sum_(torch.as_tensor(np.asarray(hist, dtype=np.int64), device=engine.dev))
    bigs = comm.gather_object(np.asarray(big, dtype=np.int64).tolist())
    big_all = np.array([v for b in bigs for v in b], dtype=np.int64)
    keys = comm.gather_rows(pk[:matched])
    sims = comm.gather_rows(ps[:matched])
    if comm.rank == root:
        pk_all = torch.cat(keys) if keys else pk[:0]
        ps_all = torch.cat(sims) if sims else ps[:0]
        trip = engine.finalize(pk_all, ps_all, matched_all)
    else:
        trip = torch.empty(0, dtype=torch.uint8, device=engine.dev)
    fill_stats(stats, n, t, looks, pieces, mx, hist_t.cpu().numpy(), big_all, singles, distinct,
               matched_all, n_ex)
    return trip, stats, engine


def row_block(n: int, world: int, rank: int):
    """Rows [a, b) of `rank`'s block and the common padded block length s
    (= ceil(n / world)); the gathered blocks' first n rows are rows 0..n-1."""
    s = -(-n // world) if n else 0
    a = min(n, rank * s)
    return a, min(n, a + s), s


def gather_search_layout(bits_block, n: int, mapping, comm):
    """Row-sharded Min-Max + all-gather of the search layout.

    bits_block: CUDA int32 (s, K), this rank's rows `row_block(n, world,
    rank)` padded to s rows (pad rows: any in-range bit indices).  Returns
    (rkeys (n, t), tags (2, n, W, 8), bad) for all n rows on every rank."""
    import torch
    from .lsh_search import signatures_for_search
    world = comm.world
    s = int(bits_block.shape[0])
    t = mapping.t
    W = (t + 31) // 32
    _, rk_l, tg_l, bad = signatures_for_search(bits_block, mapping, with_keys=False)
    rk = torch.empty((world * s, t), dtype=torch.int64, device=bits_block.device)
    comm.gather_into(rk, rk_l)
    tg = torch.empty((2, world * s, W, 8), dtype=torch.int32, device=bits_block.device)
    for h in range(2):
        comm.gather_into(tg[h], tg_l[h].contiguous())
    del rk_l, tg_l
    comm.max_(bad)
    rkeys = rk[:n]
    tags = tg if n == world * s else tg[:, :n].contiguous()
    return rkeys, tags, bad


def own_keys(rkeys, tables):
    """(len(tables), n) table-major keys of this rank's tables, from the rows."""
    import torch
    ids = torch.as_tensor(list(tables), dtype=torch.int64, device=rkeys.device)
    return rkeys.index_select(1, ids).t().contiguous()


def search_bits_sharded(bits_block, n: int, cfg, mapping, exclusion_windows: int = 0,
                        comm=None, root: int = 0, timing: bool = False):
    """Device-resident table-sharded search of one station's n fingerprints
    whose rows are block-distributed over the ranks (see gather_search_layout).
    Returns (triplets on root, global SearchStats, this rank's DeviceSearch)."""
    comm = comm or TorchComm()
    rkeys, tags, bad = gather_search_layout(bits_block, n, mapping, comm)
    if int(bad.item()):
        raise ParameterError("fingerprint bit index out of range for mapping")
    tables = shard_tables(mapping.t, comm.world, comm.rank)
    engine = DeviceSearch(own_keys(rkeys, tables), rkeys, tags, n, mapping.t, timing=timing,
                          tables=tables)
    return run_search_sharded(engine, comm, n, mapping.t, cfg, exclusion_windows, root=root)


def search_fingerprints_sharded(fps_block, n: int, cfg, mapping=None, group=None, root: int = 0):
    """Multi-GPU lsh_search.search_fingerprints (lsh_search.py:314-333) for one
    station: this rank holds rows row_block(n, world, rank) of the
    fingerprints (`fps_block`, host numpy or CUDA bits); the triplets come
    back on `root` (host numpy for host input), the stats on every rank."""
    import numpy as _np
    from . import _native as nat
    from .errors import ConsistencyError
    from .lsh_search import (TRIPLET_DTYPE, _to_device_staged, exclusion_windows_for)
    from .minmax_hash import gen_hash_mapping
    cfg.validate()
    comm = TorchComm(group)
    torch = nat.torch()
    if mapping is None:
        mapping = gen_hash_mapping(fps_block.d, cfg.tables, cfg.hash_funcs, cfg.seed)
    if (mapping.t, mapping.k) != (cfg.tables, cfg.hash_funcs) or mapping.d != fps_block.d:
        raise ConsistencyError("hash mapping does not match search config / fingerprints")
    a, b, s = row_block(n, comm.world, comm.rank)
    bits = fps_block.bits
    on_device = nat.is_device_tensor(bits)
    if int(bits.shape[0]) != b - a:
        raise ParameterError(f"rank {comm.rank} must hold rows [{a}, {b}) of the {n} fingerprints")
    if on_device:
        blk = bits.to(torch.int32).contiguous()
    else:
        blk = _to_device_staged(_np.ascontiguousarray(bits, dtype=_np.uint32).view(_np.int32))
    if b - a < s:  # pad the last block; pad rows repeat row 0's indices (always valid)
        pad = (blk[:1] if b > a else torch.zeros((1, blk.shape[1]), dtype=torch.int32,
                                                   device=blk.device)).expand(s - (b - a), -1)
        blk = torch.cat([blk, pad])
    trip, stats, _ = search_bits_sharded(blk, n, cfg, mapping, exclusion_windows_for(fps_block, cfg),
                                         comm=comm, root=root)
    if on_device:
        return trip, stats, mapping
    return trip.cpu().numpy().view(TRIPLET_DTYPE), stats, mapping


def search_signatures_sharded(keys, rkeys, tags, n: int, t: int, cfg, exclusion_windows: int = 0,
                              group=None, root: int = 0, timing: bool = False):
    """GPU entry: this rank's DeviceSearch over its round-robin tables, then
    the sharded protocol over `group` (NCCL)."""
    comm = TorchComm(group)
    tables = shard_tables(t, comm.world, comm.rank)
    engine = DeviceSearch(keys, rkeys, tags, n, t, timing=timing, tables=tables)
    return run_search_sharded(engine, comm, n, t, cfg, exclusion_windows, root=root)
