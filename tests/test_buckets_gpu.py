"""Bucket construction parity (lsh_search.py:157-172): qs_lsh_build_bucket_flags
against a numpy stable argsort of each table column.  Member ids must follow
the reference's stable order (key, then position) and the head/tail flags
must mark exactly the run boundaries; the flag listing must reproduce the
key-based listing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mix(x):
    x = x.astype(np.uint64) ^ np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xFF51AFD7ED558CCD)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xC4CEB9FE1A85EC53)
        x ^= x >> np.uint64(33)
    return x


def _expected(keys):
    t, n = keys.shape
    ids = np.empty((t, n), np.uint32)
    flags = np.empty((t, n), np.uint8)
    for i in range(t):
        o = np.argsort(keys[i], kind="stable")
        ids[i] = o
        s = keys[i][o]
        head = np.ones(n, bool)
        head[1:] = s[1:] != s[:-1]
        tail = np.ones(n, bool)
        tail[:-1] = s[1:] != s[:-1]
        flags[i] = head.astype(np.uint8) | (tail.astype(np.uint8) << 1)
    return ids, flags


def _build(keys):
    import torch
    from paper_1803_09835_b200 import _native as nat
    lib = nat.lib()
    t, n = keys.shape
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    ids = torch.empty((t, n), dtype=torch.int32, device="cuda")
    flags = torch.empty((t, n), dtype=torch.uint8, device="cuda")
    ws = torch.empty(lib.qs_lsh_bucket_flags_ws_bytes(n, t), dtype=torch.uint8, device="cuda")
    nat.call("qs_lsh_build_bucket_flags", nat.ptr(kd), n, t, nat.ptr(ids), nat.ptr(flags),
             nat.ptr(ws), ws.numel(), nat.stream())
    torch.cuda.synchronize()
    return ids.cpu().numpy().view(np.uint32), flags.cpu().numpy()


CASES = {
    # name: (n, t, alphabet or None for uniform 64-bit)
    "tiny": (1, 3, None),
    "small_uniform": (2500, 5, None),
    "one_bin_dups": (3000, 4, 40),
    "multi_bin_uniform": (200_000, 3, None),
    "multi_bin_dups": (200_000, 3, 50_000),
    "ragged": (12_345, 7, 3000),
    "mid_buckets": (100_000, 2, 500),
    "big_buckets": (100_000, 2, 60),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_binned_matches_stable_argsort(name):
    n, t, alpha = CASES[name]
    rng = np.random.default_rng(sum(map(ord, name)))
    if alpha is None:
        keys = rng.integers(0, 2**63, size=(t, n), dtype=np.int64).astype(np.uint64) * np.uint64(2)
        keys ^= rng.integers(0, 2, size=(t, n)).astype(np.uint64)
    else:
        keys = _mix(rng.integers(0, alpha, size=(t, n)).astype(np.uint64))
    want_ids, want_flags = _expected(keys)
    ids, flags = _build(keys)
    assert np.array_equal(ids, want_ids), name
    assert np.array_equal(flags, want_flags), name


def test_prefix_collisions_keep_full_key_order():
    # keys agreeing on their top 40 bits (beyond the radix digits) but not below
    rng = np.random.default_rng(5)
    n, t = 50_000, 2
    hi = rng.integers(0, 64, size=(t, n)).astype(np.uint64) << np.uint64(40)
    lo = rng.integers(0, 4, size=(t, n)).astype(np.uint64)
    keys = _mix(rng.integers(0, 2**20, size=(t, 1)).astype(np.uint64)) & ~np.uint64(2**46 - 1)
    keys = keys + hi + lo
    want_ids, want_flags = _expected(keys)
    ids, flags = _build(keys)
    assert np.array_equal(ids, want_ids)
    assert np.array_equal(flags, want_flags)


@pytest.mark.parametrize("big", [6_000, 15_000, 40_000])
def test_bins_with_one_huge_bucket(big):
    """A bucket bigger than the shared-memory bin sort (mid: 4k-16k members,
    giant: > 16k) next to ordinary keys, plus 32-bit prefix collisions."""
    rng = np.random.default_rng(big)
    n, t = 300_000, 2
    keys = _mix(rng.integers(0, 2**40, size=(t, n)).astype(np.uint64))
    pos = rng.choice(n, big, replace=False)
    keys[0, pos] = keys[0, 0]
    keys[1, pos[: big // 2]] = keys[1, 7]
    # same top 32 bits as the huge bucket's key, different low bits
    keys[0, rng.choice(n, 50, replace=False)] = (keys[0, 0] & ~np.uint64(0xFFFFFFFF)) | np.uint64(5)
    want_ids, want_flags = _expected(keys)
    ids, flags = _build(keys)
    assert np.array_equal(ids, want_ids)
    assert np.array_equal(flags, want_flags)


def test_large_table_many_bins():
    rng = np.random.default_rng(9)
    n, t = 3_000_000, 2
    keys = _mix(rng.integers(0, 400_000, size=(t, n)).astype(np.uint64))
    want_ids, want_flags = _expected(keys)
    ids, flags = _build(keys)
    assert np.array_equal(ids, want_ids)
    assert np.array_equal(flags, want_flags)


def test_all_identical_keys():
    n, t = 20_000, 2
    keys = np.full((t, n), 12345, np.uint64)
    keys[1, ::3] = 7
    want_ids, want_flags = _expected(keys)
    ids, flags = _build(keys)
    assert np.array_equal(ids, want_ids)
    assert np.array_equal(flags, want_flags)
