"""Table-sharded search protocol (paper_1803_09835_b200/sharded.py) on CPU:
world_size 2 and 3 gloo process groups, each rank a numpy stand-in for its
DeviceSearch share (tests/shard_engine_np.py).  The gathered triplets and the
global SearchStats must equal the single-process oracle search (itself
pinned to the reference's golden runs) — the same check the GPU test makes
with the real kernels."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from oracle import search as osr

STAT_KEYS = ("n_queries", "lookups_total", "distinct_pairs", "emitted_triplets",
             "filtered_fingerprints", "peak_table_entries", "n_buckets", "max_bucket")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sigs, cfg_kw, excl, q):
    import torch.distributed as dist
    from paper_1803_09835_b200.lsh_search import SearchConfig
    from paper_1803_09835_b200.sharded import TorchComm, run_search_sharded, shard_tables
    from shard_engine_np import NumpyShardEngine
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        cfg = SearchConfig(**cfg_kw)
        eng = NumpyShardEngine(sigs, shard_tables(sigs.shape[1], world, rank))
        trip, st, _ = run_search_sharded(eng, TorchComm(), sigs.shape[0], sigs.shape[1], cfg, excl)
        q.put((rank, trip.numpy().tobytes(), st.to_dict(), None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, None, None, repr(e)))


def _run(sigs, cfg_kw, excl, world):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sigs, cfg_kw, excl, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, trip, st, err = q.get(timeout=300)
        assert err is None, err
        out[r] = (trip, st)
    for p in procs:
        p.join(timeout=60)
    return out


def _check(out, sigs, cfg_kw, excl):
    want, wst = osr.search(sigs, tables=cfg_kw["tables"], min_matches=cfg_kw["min_matches"],
                           partitions=cfg_kw["partitions"],
                           occurrence_threshold=cfg_kw["occurrence_threshold"],
                           exclusion_windows=excl)
    assert out[0][0] == want.tobytes()
    for r, (trip, st) in out.items():
        if r:
            assert trip == b""
        for k in STAT_KEYS:
            assert st[k] == wst[k], (r, k, st[k], wst[k])
        assert st["top_bucket_mass"] == pytest.approx(wst["top_bucket_mass"], rel=1e-12)


def _collide_prone(n, t, seed, alphabet=3):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, alphabet, size=(n, t)).astype(np.uint64)
    # planted near-duplicates and a noisy group to drive the occurrence filter
    for i in range(0, n - 1, 7):
        j = min(n - 1, i + 1 + int(rng.integers(0, 5)))
        keep = rng.random(t) < 0.6
        base[j, keep] = base[i, keep]
    g = rng.choice(n, size=n // 5, replace=False)
    base[g[1:], : t // 2] = base[g[0], : t // 2]
    return base


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [
    dict(partitions=1, occurrence_threshold=None, excl=0),
    dict(partitions=1, occurrence_threshold=0.05, excl=0),
    dict(partitions=3, occurrence_threshold=0.05, excl=2),
    dict(partitions=2, occurrence_threshold=None, excl=1),
])
def test_sharded_protocol_matches_oracle(world, case):
    t = 10
    sigs = _collide_prone(90, t, seed=world * 10 + case["partitions"])
    cfg_kw = dict(tables=t, hash_funcs=4, min_matches=3, partitions=case["partitions"],
                  occurrence_threshold=case["occurrence_threshold"])
    out = _run(sigs, cfg_kw, case["excl"], world)
    _check(out, sigs, cfg_kw, case["excl"])


def test_sharded_golden_cases(golden_search):
    """Every golden reference run, split over two gloo ranks."""
    done = 0
    for name, c in golden_search.items():
        sigs = c["sigs"]
        if sigs.shape[0] == 0 or sigs.shape[0] > 400:
            continue
        cfg = c["cfg"]
        cfg_kw = dict(tables=sigs.shape[1], hash_funcs=cfg.get("hash_funcs", 4),
                      min_matches=cfg["min_matches"], partitions=cfg.get("partitions", 1),
                      occurrence_threshold=cfg.get("occurrence_threshold"))
        excl = int(cfg.get("exclusion_windows", 0))
        out = _run(sigs, cfg_kw, excl, 2)
        assert out[0][0] == c["trip"].tobytes(), name
        for k in STAT_KEYS:
            assert out[1][1][k] == c["stats"][k], (name, k)
        done += 1
    assert done >= 5


def test_shard_tables_partition_the_tables():
    from paper_1803_09835_b200.sharded import shard_tables
    for t in (1, 7, 100, 130):
        for world in (1, 2, 3, 8):
            got = sorted(x for r in range(world) for x in shard_tables(t, world, r))
            assert got == list(range(t))
    with pytest.raises(Exception):
        shard_tables(10, 2, 2)
