"""The one-call C entries qs_lsh_search / qs_lsh_search_bits, driven through
ctypes the way a non-Python caller would bind them: caller
workspace from the size query, triplets + qs_search_stats out.  Results must
equal the reference's golden runs and the oracle byte for byte."""

import ctypes

import numpy as np
import pytest

from oracle import search as osr

pytestmark = pytest.mark.gpu


def _stats_dict(c, n, partitions):
    d = {f: getattr(c, f) for f, _ in c._fields_ if f != "n_partitions"}
    d["lookups_per_query"] = d["lookups_total"] / d["n_queries"] if d["n_queries"] else 0.0
    d["selectivity"] = 2.0 * d["distinct_pairs"] / (n * n) if n else 0.0
    d["partitions"] = partitions
    return d


def capi_search(sigs, t, m, excl, occ, partitions, pair_cap=None, bits=None, K=0, d=0, seed=0,
                k_half=2):
    import torch
    from paper_1803_09835_b200 import _native as nat
    from paper_1803_09835_b200.lsh_search import TRIPLET_DTYPE, partition_bounds
    lib = nat.lib()
    n = int(sigs.shape[0]) if bits is None else int(bits.shape[0])
    cap = pair_cap if pair_cap is not None else max(1024, 4 * n)
    occ_c = -1.0 if occ is None else float(occ)
    for _ in range(2):
        if bits is None:
            wsb = lib.qs_lsh_search_ws_bytes(n, t, cap, partitions)
        else:
            wsb = lib.qs_lsh_search_bits_ws_bytes(n, d, t, k_half, cap, partitions)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        trip = torch.empty(max(1, cap) * 20, dtype=torch.uint8, device="cuda")
        needed = ctypes.c_uint64(0)
        st = nat.SearchStatsC()
        if bits is None:
            sd = torch.from_numpy(np.ascontiguousarray(sigs, np.uint64).view(np.int64)).cuda()
            rc = lib.qs_lsh_search(nat.ptr(sd), n, t, m, excl, occ_c, partitions, nat.ptr(trip), cap,
                                   ctypes.byref(needed), ctypes.byref(st), nat.ptr(ws), wsb,
                                   nat.stream())
        else:
            bd = torch.from_numpy(np.ascontiguousarray(bits, np.uint32).view(np.int32)).cuda()
            rc = lib.qs_lsh_search_bits(nat.ptr(bd), n, K, d, seed, t, k_half, m, excl, occ_c,
                                        partitions, nat.ptr(trip), cap, ctypes.byref(needed),
                                        ctypes.byref(st), nat.ptr(ws), wsb, nat.stream())
        if rc == nat.QS_ERR_CAPACITY:
            assert needed.value > cap
            cap = int(needed.value)
            continue
        nat.check(rc, "qs_lsh_search")
        break
    k = st.emitted_triplets
    rec = trip[: k * 20].cpu().numpy().view(TRIPLET_DTYPE)
    parts = [[a, b] for a, b in partition_bounds(n, partitions)] if n else []
    assert st.n_partitions == len(parts)
    return rec, _stats_dict(st, n, parts)


def _same_stats(got, want, name):
    for k, v in want.items():
        if isinstance(v, float):
            assert got[k] == pytest.approx(v, rel=1e-12, abs=1e-15), (name, k)
        else:
            assert got[k] == v, (name, k, got[k], v)


def test_capi_search_golden(golden_search):
    for name, case in golden_search.items():
        c = dict(case["cfg"])
        excl = c.pop("exclusion_windows", 0)
        rec, st = capi_search(case["sigs"], c["tables"], c.get("min_matches", 5), excl,
                              c.get("occurrence_threshold"), c.get("partitions", 1))
        assert rec.tobytes() == case["trip"].tobytes(), name
        _same_stats(st, case["stats"], name)


def test_capi_capacity_retry_and_errors():
    import torch
    from paper_1803_09835_b200 import _native as nat
    rng = np.random.default_rng(3)
    sigs = rng.integers(0, 6, size=(500, 8)).astype(np.uint64)
    want, wst = osr.search(sigs, tables=8, min_matches=2, partitions=1,
                           occurrence_threshold=None, exclusion_windows=0)
    assert want.size > 100
    rec, st = capi_search(sigs, 8, 2, 0, None, 1, pair_cap=16)  # forces QS_ERR_CAPACITY first
    assert rec.tobytes() == want.tobytes()
    lib = nat.lib()
    st_c = nat.SearchStatsC()
    needed = ctypes.c_uint64(0)
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    rc = lib.qs_lsh_search(None, 500, 8, 2, 0, -1.0, 1, None, 1024, ctypes.byref(needed),
                           ctypes.byref(st_c), nat.ptr(ws), 16, nat.stream())
    assert rc == nat.QS_ERR_ARG and b"workspace" in lib.qs_last_error()
    rc = lib.qs_lsh_search(None, 500, 8, 9, 0, -1.0, 1, None, 1024, ctypes.byref(needed),
                           ctypes.byref(st_c), nat.ptr(ws), 16, nat.stream())
    assert rc == nat.QS_ERR_ARG  # min_matches > tables


def test_capi_search_bits_cfg1_vs_oracle():
    from oracle import minmax as omm
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.minmax_hash import gen_hash_mapping
    bits, _ = workloads.cfg1_bits(n=20_000, seed=8, pair_frac=1 / 80, group_frac=1 / 1000)
    m = gen_hash_mapping(4096, 100, 4, 0)
    sigs = omm.signatures_c(bits, m.values, 100, 2, threads=8)
    for occ, p, excl in [(None, 1, 0), (120 / 20000, 1, 3), (60 / 20000, 3, 0)]:
        want, wst = osr.search(sigs, tables=100, min_matches=5, partitions=p,
                               occurrence_threshold=occ, exclusion_windows=excl)
        rec, st = capi_search(None, 100, 5, excl, occ, p, bits=bits, K=400, d=4096, seed=0)
        assert rec.tobytes() == want.tobytes(), (occ, p)
        _same_stats(st, wst, (occ, p))
        rec2, st2 = capi_search(sigs, 100, 5, excl, occ, p)
        assert rec2.tobytes() == want.tobytes()
