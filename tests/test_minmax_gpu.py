"""Min-Max signature kernel parity on the GPU (bit-exact vs oracle + golden).

Mirrors the reference's tests/test_minmax_hash.py strategy: frozen KATs,
mapping definition, min/max semantics, bit-order invariance, identical rows,
backend equality (here: CUDA kernel == reference compiled kernel == oracle).
"""

import numpy as np
import pytest

from oracle import minmax as omm

pytestmark = pytest.mark.gpu

SIG_FROZEN = [0xEC797BCAD18E750C, 0x168878915D63A8D2, 0x684B9C6319F40596]


@pytest.fixture(scope="module")
def mh():
    from paper_1803_09835_b200 import minmax_hash
    return minmax_hash


def rand_bits(rng, n, d, K):
    return np.stack([np.sort(rng.choice(d, K, replace=False)) for _ in range(n)]).astype(np.uint32)


def test_frozen_signature(mh):
    m = mh.gen_hash_mapping(d=64, t=3, k=4, seed=42)
    sig = mh.signatures(np.array([[0, 5, 17, 63]], np.uint32), m)[0]
    assert [int(x) for x in sig] == SIG_FROZEN


def test_mapping_matches_oracle(mh):
    for d, t, k, seed in [(128, 4, 6, 991), (4096, 100, 4, 0), (97, 5, 2, 2**64 - 3)]:
        m = mh.gen_hash_mapping(d, t, k, seed)
        assert np.array_equal(m.values, omm.gen_mapping(d, t, k, seed))


def test_golden_cases(mh, golden_minmax):
    from paper_1803_09835_b200 import _sigcore_cuda
    for name, case in golden_minmax.items():
        d, t, k = (int(v) for v in case["meta"])
        m = mh.gen_hash_mapping(d, t, k, int(case["seed"][0]))
        got = mh.signatures(case["bits"], m)
        assert np.array_equal(got, case["sigs"]), name
        out = np.zeros_like(case["sigs"])
        _sigcore_cuda.gen_signatures_range(case["bits"], m.values, t, k // 2, out, 0,
                                           case["bits"].shape[0])
        assert np.array_equal(out, case["sigs"]), name


def test_random_vs_oracle_and_reference_kernel(mh):
    rng = np.random.default_rng(3)
    for n, d, K, t, k in [(3000, 4096, 400, 100, 4), (2000, 8192, 100, 50, 6),
                          (500, 1000, 1, 7, 2), (700, 16384, 3000, 3, 10)]:
        bits = rand_bits(rng, n, d, K)
        m = mh.gen_hash_mapping(d, t, k, int(rng.integers(0, 2**63)))
        want = omm.signatures_c(bits, m.values, t, k // 2, threads=4)
        assert np.array_equal(mh.signatures(bits, m), want)
        ref = omm.signatures_reference_kernel(bits, m.values, t, k // 2, threads=4)
        if ref is not None:
            assert np.array_equal(ref, want)


def test_partial_row_range_plugin(mh):
    from paper_1803_09835_b200 import _sigcore_cuda
    rng = np.random.default_rng(4)
    bits = rand_bits(rng, 101, 1024, 25)
    m = mh.gen_hash_mapping(1024, 8, 4, 10)
    want = omm.signatures_c(bits, m.values, 8, 2)
    out = np.zeros((101, 8), np.uint64)
    _sigcore_cuda.gen_signatures_range(bits, m.values, 8, 2, out, 17, 64)
    assert np.array_equal(out[17:64], want[17:64])
    assert not out[:17].any() and not out[64:].any()


def test_min_max_semantics(mh):
    m = mh.gen_hash_mapping(d=512, t=1, k=2, seed=77)
    rng = np.random.default_rng(0)
    bits = rand_bits(rng, 20, 512, 30)
    sigs = mh.signatures(bits, m)
    col = m.values[:, 0]
    for row, sig in zip(bits, sigs[:, 0]):
        assert int(sig) == omm.combine([int(col[row].min()), int(col[row].max())])


def test_bit_order_duplicates_and_identical_rows(mh):
    rng = np.random.default_rng(12)
    m = mh.gen_hash_mapping(d=2048, t=16, k=6, seed=2)
    row = rng.choice(2048, 100, replace=False).astype(np.uint32)
    a = mh.signatures(np.sort(row)[None, :], m)
    b = mh.signatures(rng.permutation(row)[None, :], m)
    dup = np.concatenate([row, row[:7]])
    c = mh.signatures(dup[None, :], m)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    two = mh.signatures(np.vstack([np.sort(row), np.sort(row)]), m)
    assert np.array_equal(two[0], two[1])


def test_device_tensor_path(mh):
    import torch
    rng = np.random.default_rng(5)
    bits = rand_bits(rng, 1000, 4096, 200)
    m = mh.gen_hash_mapping(4096, 100, 4, 0)
    dev = mh.signatures(torch.from_numpy(bits.view(np.int32)).cuda(), m)
    assert dev.is_cuda and dev.shape == (1000, 100)
    assert np.array_equal(dev.cpu().numpy().view(np.uint64), mh.signatures(bits, m))


def test_errors(mh):
    from paper_1803_09835_b200.errors import ParameterError
    m = mh.gen_hash_mapping(64, 2, 2, 0)
    with pytest.raises(ParameterError):
        mh.signatures(np.array([[1, 64]], np.uint32), m)
    with pytest.raises(ParameterError):
        mh.signatures(np.zeros((3, 0), np.uint32), m)
    with pytest.raises(ParameterError):
        mh.signatures(np.zeros(3, np.uint32), m)
    with pytest.raises(ParameterError):
        mh.gen_hash_mapping(8, 1, 3, 0)
    assert mh.signatures(np.zeros((0, 5), np.uint32), m).shape == (0, 2)


def test_host_pipelined_search_layout_matches_device(mh):
    """search_fingerprints' host path (row chunks staged and signed as they
    land, qs_minmax_signatures_search_rows) == the device-resident path."""
    import torch
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import workloads
    bits, _ = workloads.cfg1_bits(n=5000, seed=3, pair_frac=1 / 50, group_frac=1 / 1000)
    m = mh.gen_hash_mapping(4096, 100, 4, 0)
    arr = np.ascontiguousarray(bits, dtype=np.uint32).view(np.int32)
    want = ls.signatures_for_search(torch.from_numpy(arr).cuda(), m)
    got = ls.signatures_for_search_host(arr, m, chunk_bytes=1777 * bits.shape[1] * 4)  # 3 ragged chunks
    torch.cuda.synchronize()
    for g, w in zip(got, want):
        assert torch.equal(g, w)
    bad = arr.copy()
    bad[4321, 7] = 4096
    got = ls.signatures_for_search_host(bad, m, chunk_bytes=1000 * bits.shape[1] * 4)
    assert int(got[3].item()) == 1


def test_large_d_plan_free_path():
    """d > 16384 (e.g. freq_bins=64, time_bins=256 -> d = 32768) takes the
    plan-free kernel (the reference's elementwise min/max loop): bit-identical
    to the C oracle, directly and through the search layout."""
    from oracle import minmax as omm
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import minmax_hash as mh
    rng = np.random.default_rng(12)
    d, K, n = 32768, 120, 300
    bits = np.stack([np.sort(rng.choice(d, K, replace=False)) for _ in range(n)]).astype(np.uint32)
    bits[150] = bits[3]  # a duplicate row -> one pair with sim = t
    m = mh.gen_hash_mapping(d, 40, 4, 9)
    sigs = mh.signatures(bits, m)
    assert np.array_equal(sigs, omm.signatures_c(bits, m.values, 40, 2))
    cfg = ls.SearchConfig(tables=40, hash_funcs=4, min_matches=2)
    from paper_1803_09835_b200.fingerprint import FingerprintSet
    fps = FingerprintSet(d=d, top_k=K, window_len_s=1.0, window_lag_s=1.0,
                         indices=np.arange(n, dtype=np.uint64), epochs=np.arange(n, dtype=np.float64),
                         bits=bits)
    rec, st, _ = ls.search_fingerprints(fps, ls.SearchConfig(tables=40, hash_funcs=4, min_matches=2,
                                                             near_repeat_exclusion_s=0.0), mapping=m)
    want, _ = ls.search_signatures(sigs, cfg)
    assert rec.tobytes() == want.tobytes() and rec.size >= 1
