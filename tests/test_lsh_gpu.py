"""LSH search parity on the GPU: byte-identical triplets and identical
SearchStats against the reference's golden runs, plus oracle comparisons on
random and cfg1-shaped inputs (reference tests/test_lsh_search.py strategy:
brute force, partition identity, canonical/sorted output, near-repeat
exclusion, occurrence filter, stats fields)."""

import numpy as np
import pytest

from oracle import search as osr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ls():
    from paper_1803_09835_b200 import lsh_search
    return lsh_search


def _cfg(ls, c):
    c = dict(c)
    excl = c.pop("exclusion_windows", 0)
    return ls.SearchConfig(**c), excl


def _check_stats(got, want, name):
    d = got.to_dict()
    for k, v in want.items():
        if isinstance(v, float):
            assert d[k] == pytest.approx(v, rel=1e-12, abs=1e-15), (name, k, d[k], v)
        else:
            assert d[k] == v, (name, k, d[k], v)


def test_golden_search_cases(ls, golden_search):
    for name, case in golden_search.items():
        cfg, excl = _cfg(ls, case["cfg"])
        rec, st = ls.search_signatures(case["sigs"], cfg, exclusion_windows=excl)
        assert rec.dtype == ls.TRIPLET_DTYPE
        assert rec.tobytes() == case["trip"].tobytes(), name
        _check_stats(st, case["stats"], name)


def _oracle(sigs, cfg, excl):
    return osr.search(sigs, tables=cfg.tables, min_matches=cfg.min_matches,
                      partitions=cfg.partitions, occurrence_threshold=cfg.occurrence_threshold,
                      exclusion_windows=excl)


@pytest.mark.parametrize("seed", range(24))
def test_random_collide_prone_vs_oracle(ls, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 400))
    t = int(rng.choice([1, 3, 16, 32, 33, 64, 100, 128, 130]))
    sigs = rng.integers(0, int(rng.integers(2, 30)), size=(n, t)).astype(np.uint64)
    if rng.random() < 0.3:
        sigs[:, :] |= np.uint64(1) << np.uint64(63)
    m = int(rng.integers(1, t + 1))
    p = int(rng.choice([1, 2, 3, 7]))
    occ = [None, 0.05, 0.3, 1.0][int(rng.integers(0, 4))]
    excl = int(rng.integers(0, 5))
    cfg = ls.SearchConfig(tables=t, hash_funcs=2, min_matches=m, partitions=p,
                          occurrence_threshold=occ)
    rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
    want, wst = _oracle(sigs, cfg, excl)
    assert rec.tobytes() == want.tobytes()
    _check_stats(st, {k: v for k, v in wst.items() if k not in ("lookups_per_query", "selectivity")},
                 seed)
    if occ is None:
        bf = osr.brute_force_triplets(sigs, m, excl)
        assert sorted((int(a), int(b), int(c)) for a, b, c in
                      zip(rec["dt"], rec["idx1"], rec["sim"])) == bf


def test_partition_identity_and_device_output(ls):
    import torch
    rng = np.random.default_rng(6)
    sigs = rng.integers(0, 40, size=(2000, 12)).astype(np.uint64)
    base = None
    for p in (1, 2, 3, 8, 64):
        cfg = ls.SearchConfig(tables=12, hash_funcs=2, min_matches=2, partitions=p)
        rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=1)
        if base is None:
            base = rec.tobytes()
            assert rec.size > 50
        assert rec.tobytes() == base
    dev, _ = ls.search_signatures(torch.from_numpy(sigs.view(np.int64)).cuda(),
                                  ls.SearchConfig(tables=12, hash_funcs=2, min_matches=2),
                                  exclusion_windows=1)
    assert dev.is_cuda and dev.cpu().numpy().tobytes() == base


def test_cfg1_shaped_vs_oracle(ls):
    from oracle import minmax as omm
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    bits, _ = workloads.cfg1_bits(n=20000, seed=3, pair_frac=1 / 80, group_frac=1 / 1000)
    m = mh.gen_hash_mapping(4096, 100, 4, 0)
    sigs = mh.signatures(bits, m)
    assert np.array_equal(sigs[:500], omm.signatures_c(bits[:500], m.values, 100, 2))
    for occ, p, excl in [(None, 1, 0), (120 / 20000, 1, 0), (60 / 20000, 4, 3)]:
        cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, partitions=p,
                              occurrence_threshold=occ)
        rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
        want, wst = _oracle(sigs, cfg, excl)
        assert rec.tobytes() == want.tobytes(), (occ, p)
        _check_stats(st, {k: v for k, v in wst.items()}, (occ, p))


def test_search_config_validation(ls):
    from paper_1803_09835_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        ls.SearchConfig(tables=0).validate()
    with pytest.raises(ParameterError):
        ls.SearchConfig(hash_funcs=3).validate()
    with pytest.raises(ParameterError):
        ls.SearchConfig(min_matches=101).validate()
    with pytest.raises(ParameterError):
        ls.search_signatures(np.zeros((3, 4), np.uint64), ls.SearchConfig(tables=5))
    assert ls.PROFILES == {"baseline": (6, 5), "optimized": (8, 2)}


def _check_triplets_against_keys(rec_dev, rkeys, n, m):
    """Size-independent properties of an emitted triplet set: sorted by
    (dt, idx1) without duplicates, dt >= 1, both ends in range, sim >= m and
    sim == the number of tables whose keys agree (recomputed from the keys)."""
    import torch
    cnt = rec_dev.numel() // 20
    if cnt == 0:
        return
    r = rec_dev.view(cnt, 20)
    dt = r[:, 0:8].contiguous().view(torch.int64).view(-1)
    i1 = r[:, 8:16].contiguous().view(torch.int64).view(-1)
    sim = r[:, 16:20].contiguous().view(torch.int32).view(-1)
    key = dt * (1 << 32) + i1
    assert bool(torch.all(key[1:] > key[:-1]).item())
    assert int(dt.min().item()) >= 1 and int((i1 + dt).max().item()) < n
    assert int(sim.min().item()) >= m
    for a in range(0, cnt, 1 << 20):
        b = min(cnt, a + (1 << 20))
        ka = rkeys.index_select(0, i1[a:b])
        kb = rkeys.index_select(0, i1[a:b] + dt[a:b])
        assert torch.equal((ka == kb).sum(1).to(torch.int32), sim[a:b])


def test_cfg1_full_scale_properties(ls):
    """BASELINE cfg1 at full size (N = 8e6) with the filter, and N = 2e6
    without: properties checked on the GPU (the oracle cannot run there)."""
    import torch
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
    for n, occ in [(8_000_000, 1.5e-5), (2_000_000, None)]:
        bits, _ = workloads.cfg1_bits_torch(n=n, seed=11, device=torch.device("cuda"))
        keys, rkeys, tags, bad = ls.signatures_for_search(bits, mapping)
        del bits
        cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=occ)
        trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0)
        _check_triplets_against_keys(trip, rkeys, n, 5)
        assert st.emitted_triplets == trip.numel() // 20
        if occ is None:
            bs = ds.bsize[: ds.nb].to(torch.int64)
            assert st.lookups_total == int((bs * (bs - 1)).sum().item())
            assert st.distinct_pairs <= st.lookups_total // 2
            assert st.n_queries == n and st.filtered_fingerprints == 0
        else:
            assert 0 < st.filtered_fingerprints < n
        del keys, rkeys, tags, trip, ds
        torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def cfg1_1e5():
    """The cfg1 generator (BASELINE configs[1] densities) at N = 1e5, its
    Min-Max signatures from the C oracle, and the mapping."""
    from oracle import minmax as omm
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    bits, _ = workloads.cfg1_bits(n=100_000, seed=21)
    m = mh.gen_hash_mapping(4096, 100, 4, 0)
    sigs = omm.signatures_c(bits, m.values, 100, 2, threads=8)
    return bits, sigs, m


@pytest.mark.parametrize("occ_limit,p,excl", [(None, 1, 0), (120, 1, 0), (60, 3, 2)])
def test_cfg1_1e5_vs_oracle(ls, cfg1_1e5, occ_limit, p, excl):
    """cfg1 at N = 1e5 (the scale of the CPU baseline), filter off (the
    reference default) and on at limit 120 (the bench's setting, which removes
    the noise groups): signatures bit-identical, triplets byte-identical and
    every SearchStats field equal to the oracle's."""
    from paper_1803_09835_b200 import minmax_hash as mh
    bits, want_sigs, m = cfg1_1e5
    sigs = mh.signatures(bits, m)
    assert np.array_equal(sigs, want_sigs)
    n = bits.shape[0]
    occ = occ_limit / n if occ_limit else None
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, partitions=p,
                          occurrence_threshold=occ)
    rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
    want, wst = _oracle(want_sigs, cfg, excl)
    assert rec.size > 1000
    assert rec.tobytes() == want.tobytes(), (occ_limit, p)
    _check_stats(st, dict(wst), (occ_limit, p))
    if occ_limit == 120:
        assert st.filtered_fingerprints > 0.3 * n  # the filter fires (noise groups removed)


@pytest.mark.parametrize("host_memory", ["pageable", "pageable_u32", "pinned", "pinned_direct",
                                         "pinned_all_narrowed"])
def test_cfg1_1e5_host_bits_e2e(ls, cfg1_1e5, host_memory, monkeypatch):
    """The same N = 1e5 batch through search_fingerprints with host bits (the
    e2e path the bench times: row-chunk H2D pipelined with the fused signature
    kernel) from a pageable array (narrowed to uint16 while staged, or staged
    as uint32 with QS_H2D_NARROW=0) and from page-locked memory (DMA from the
    array, a share of the rows narrowed on the way: default, none, all)."""
    import torch
    from paper_1803_09835_b200.fingerprint import FingerprintSet
    bits, want_sigs, m = cfg1_1e5
    n = bits.shape[0]
    if host_memory.startswith("pinned"):
        if host_memory != "pinned":
            monkeypatch.setenv("QS_H2D_SPLIT", "0" if host_memory == "pinned_direct" else "1")
        hold = torch.empty(bits.shape, dtype=torch.int32, pin_memory=True)
        hbits = hold.numpy().view(np.uint32)
        hbits[...] = bits
        assert ls._host_pinned(hbits)
    else:
        hbits = bits
        assert not ls._host_pinned(np.ascontiguousarray(hbits))
        if host_memory == "pageable_u32":
            monkeypatch.setenv("QS_H2D_NARROW", "0")
    fps = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                         indices=np.arange(n, dtype=np.uint64),
                         epochs=np.arange(n, dtype=np.float64), bits=hbits)
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=120 / n,
                          near_repeat_exclusion_s=0.0)
    rec, st, _ = ls.search_fingerprints(fps, cfg, mapping=m)
    want, wst = _oracle(want_sigs, cfg, 0)
    assert rec.tobytes() == want.tobytes()
    _check_stats(st, dict(wst), "e2e")


@pytest.mark.parametrize("bad_value", [4096, 65535, 65536, 70000, 0xFFFFFFFF])
def test_host_bits_out_of_range(ls, bad_value):
    """An index >= d raises like the reference's range check (minmax_hash.py:
    107-108) on the narrowed staging path too: values above 65535 saturate to
    65535 >= d instead of wrapping into range."""
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.errors import ParameterError
    from paper_1803_09835_b200.fingerprint import FingerprintSet
    bits, _ = workloads.cfg1_bits(n=3000, seed=5)
    bits = np.array(bits, dtype=np.uint32)
    bits[1234, 7] = bad_value
    n = bits.shape[0]
    fps = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                         indices=np.arange(n, dtype=np.uint64),
                         epochs=np.arange(n, dtype=np.float64), bits=bits)
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, near_repeat_exclusion_s=0.0)
    with pytest.raises(ParameterError):
        ls.search_fingerprints(fps, cfg)


@pytest.mark.parametrize("n,K,d", [(1, 1, 64), (7, 3, 1000), (1001, 5, 70000), (4099, 37, 65535),
                                   (5000, 400, 4096), (1, 2, 4096), (1001, 6, 4096), (333, 10, 17),
                                   (4099, 38, 4095)])
def test_host_transfer_shapes(ls, n, K, d, monkeypatch):
    """Row widths that are not multiples of 16 bytes, one-row inputs and d
    above the uint16 range (no narrowing) give the device path's signatures on
    every host-transfer route, with chunks small enough to cycle the staging
    buffers."""
    import torch
    from paper_1803_09835_b200 import minmax_hash as mh
    rng = np.random.default_rng(n * 31 + K)
    bits = np.sort(rng.integers(0, d, size=(n, K), dtype=np.uint32), axis=1)
    m = mh.gen_hash_mapping(d, 12, 2, 3)
    want = ls.signatures_for_search(torch.from_numpy(bits.view(np.int32)).cuda(), m)
    hold = torch.empty(bits.shape, dtype=torch.int32, pin_memory=True)
    hold.numpy()[...] = bits.view(np.int32)
    for label, arr, env in (("pageable", bits.view(np.int32), {}),
                            ("pageable_u32", bits.view(np.int32), {"QS_H2D_NARROW": "0"}),
                            ("pageable_u16", bits.view(np.int32), {"QS_H2D_NARROW": "16"}),
                            ("pinned_u16", hold.numpy(), {"QS_H2D_NARROW": "16", "QS_H2D_SPLIT": "1"}),
                            ("pinned", hold.numpy(), {}),
                            ("pinned_all", hold.numpy(), {"QS_H2D_SPLIT": "1"}),
                            ("pinned_direct", hold.numpy(), {"QS_H2D_SPLIT": "0"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        got = ls.signatures_for_search_host(arr, m, chunk_bytes=max(64, n * K * 4 // 5))
        torch.cuda.synchronize()
        for k in env:
            monkeypatch.delenv(k)
        for g, w in zip(got, want):
            assert torch.equal(g, w), (label, n, K, d)


@pytest.mark.parametrize("host_memory", ["pageable", "pinned"])
def test_host_bits_12bit_fallback_mid_call(ls, host_memory, monkeypatch):
    """d = 4096 rows go up as 12-bit fields; an index above 4095 in a later chunk
    (invalid for this d) switches the call to the uint16 route, and the range
    flag is raised exactly as on the device path."""
    import torch
    from paper_1803_09835_b200 import minmax_hash as mh
    rng = np.random.default_rng(11)
    n, K, d = 3000, 8, 4096
    bits = np.sort(rng.integers(0, d, size=(n, K), dtype=np.uint32), axis=1)
    bits[2500, 3] = 5000
    m = mh.gen_hash_mapping(d, 12, 2, 3)
    want = ls.signatures_for_search(torch.from_numpy(bits.view(np.int32)).cuda(), m)
    arr = bits.view(np.int32)
    if host_memory == "pinned":
        hold = torch.empty(bits.shape, dtype=torch.int32, pin_memory=True)
        hold.numpy()[...] = arr
        arr = hold.numpy()
        monkeypatch.setenv("QS_H2D_SPLIT", "1")
    got = ls.signatures_for_search_host(arr, m, chunk_bytes=n * K * 4 // 6)
    torch.cuda.synchronize()
    assert int(got[3].item()) == int(want[3].item()) == 1  # the range flag
    ok = np.ones(n, bool)
    ok[2500] = False
    okt = torch.from_numpy(ok).cuda()
    assert torch.equal(got[1][okt], want[1][okt])  # row-major keys of the valid rows
