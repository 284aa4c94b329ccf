"""Table-sharded search with the real kernels, ranks emulated on one GPU.

Each emulated rank is a host thread driving its DeviceSearch share
(sharded.search over shard_tables); the collectives are done by a
thread-barrier stand-in for TorchComm.  No kernel waits on another rank's
kernel (all exchanges are host-side between launches), so this is safe on a
single device.  The gathered triplets and global stats must be byte-/value-
identical to the golden reference runs and to the 1-GPU search."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STAT_KEYS = ("n_queries", "lookups_total", "distinct_pairs", "emitted_triplets",
             "filtered_fingerprints", "peak_table_entries", "n_buckets", "max_bucket",
             "top_bucket_mass")


class ThreadComm:
    def __init__(self, shared, rank, world):
        self.shared, self.rank, self.world = shared, rank, world

    def _exchange(self, x):
        sh = self.shared
        sh["slots"][self.rank] = x
        sh["barrier"].wait()
        vals = list(sh["slots"])
        sh["barrier"].wait()
        return vals

    def sum_(self, x):
        import torch
        vals = self._exchange(x)
        s = torch.stack(vals).sum(0).to(x.dtype)
        self.shared["barrier"].wait()
        x.copy_(s)
        return x

    def max_(self, x):
        import torch
        vals = self._exchange(x)
        s = torch.stack(vals).amax(0)
        self.shared["barrier"].wait()
        x.copy_(s)
        return x

    def gather_rows(self, x):
        return self._exchange(x.clone())

    def gather_object(self, obj):
        return self._exchange(obj)

    def gather_into(self, out, x):
        import torch
        vals = self._exchange(x)
        out.view(-1).copy_(torch.cat([v.reshape(-1) for v in vals]))
        self.shared["barrier"].wait()  # every reader enqueued before owners reuse x
        return out


def _threads(world, body):
    shared = dict(barrier=threading.Barrier(world), slots=[None] * world)
    res, errs = [None] * world, []

    def run(r):
        try:
            res[r] = body(r, ThreadComm(shared, r, world))
        except Exception as e:  # surfaced below
            errs.append(repr(e))
            shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs
    return res


def _sharded(keys, rkeys, tags, n, t, cfg, excl, world):
    import torch
    from paper_1803_09835_b200.lsh_search import DeviceSearch
    from paper_1803_09835_b200.sharded import run_search_sharded, shard_tables

    def body(r, comm):
        eng = DeviceSearch(keys, rkeys, tags, n, t, tables=shard_tables(t, world, r))
        trip, st, _ = run_search_sharded(eng, comm, n, t, cfg, excl)
        torch.cuda.synchronize()
        return trip.cpu().numpy().tobytes(), st.to_dict()

    return _threads(world, body)


def _cfg(c):
    from paper_1803_09835_b200.lsh_search import SearchConfig
    cfg = c["cfg"]
    return SearchConfig(tables=cfg["tables"], hash_funcs=cfg.get("hash_funcs", 4),
                        min_matches=cfg["min_matches"], partitions=cfg.get("partitions", 1),
                        occurrence_threshold=cfg.get("occurrence_threshold"))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_golden(golden_search, world):
    import torch
    from paper_1803_09835_b200.lsh_search import prep_signatures
    for name, c in golden_search.items():
        sigs = c["sigs"]
        n, t = sigs.shape
        if n == 0:
            continue
        sdev = torch.from_numpy(np.ascontiguousarray(sigs).view(np.int64)).cuda()
        keys, rkeys, tags = prep_signatures(sdev)
        res = _sharded(keys, rkeys, tags, n, t, _cfg(c), int(c["cfg"].get("exclusion_windows", 0)),
                       world)
        assert res[0][0] == c["trip"].tobytes(), name
        for r in range(world):
            if r:
                assert res[r][0] == b""
            for k in STAT_KEYS:
                assert res[r][1][k] == pytest.approx(c["stats"][k], rel=1e-12), (name, r, k)


def test_sharded_cfg1_matches_single_gpu():
    import torch
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    n = 200_000
    bits, _ = workloads.cfg1_bits_torch(n=n, seed=3, device=torch.device("cuda"))
    mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
    keys, rkeys, tags, bad = ls.signatures_for_search(bits, mapping)
    assert int(bad.item()) == 0
    for occ in (None, 6e-4):
        cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=occ)
        trip, st, _ = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0)
        want = trip.cpu().numpy().tobytes()
        res = _sharded(keys, rkeys, tags, n, 100, cfg, 0, 4)
        assert res[0][0] == want
        d = st.to_dict()
        for k in STAT_KEYS:
            assert res[2][1][k] == d[k], (occ, k)
        if occ is not None:
            assert st.filtered_fingerprints > 0


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_signatures_and_search(world):
    """Block-distributed bits -> per-rank Min-Max -> gathered layout ->
    table-sharded search == the 1-GPU search_fingerprints path."""
    import torch
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.sharded import row_block, search_bits_sharded
    n = 100_003  # not a multiple of world: exercises the padded last block
    bits, _ = workloads.cfg1_bits_torch(n=n, seed=5, device=torch.device("cuda"))
    mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=1.2e-3)
    keys, rkeys, tags, _ = ls.signatures_for_search(bits, mapping)
    trip, st, _ = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0)
    want = trip.cpu().numpy().tobytes()
    del keys, rkeys, tags

    def body(r, comm):
        a, b, s = row_block(n, world, r)
        blk = bits[a:b]
        if b - a < s:
            blk = torch.cat([blk, blk[:1].expand(s - (b - a), -1)])
        tr, stt, _ = search_bits_sharded(blk.contiguous(), n, cfg, mapping, comm=comm)
        torch.cuda.synchronize()
        return tr.cpu().numpy().tobytes(), stt.to_dict()

    res = _threads(world, body)
    assert res[0][0] == want
    d = st.to_dict()
    for r in range(world):
        for k in STAT_KEYS:
            assert res[r][1][k] == d[k], (r, k)
