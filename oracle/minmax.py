"""ORACLE — test infrastructure only. Min-Max hash restatement.

numpy restatement of reference pkg/src/quakescan/_sigcore_py.py:20-62 and
minmax_hash.py:73-90, plus a ctypes front-end to the C restatement in
minmax_oracle.c (which follows _sigcore.pyx:32-85).
"""

import numpy as np

from . import c_lib, ref_sigcore

GOLDEN64 = 0x9E3779B97F4A7C15
_M1 = np.uint64(0xFF51AFD7ED558CCD)
_M2 = np.uint64(0xC4CEB9FE1A85EC53)


def fmix64(x):
    """Murmur3 finalizer over uint64 arrays (_sigcore_py.py:34-42)."""
    x = np.array(x, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= _M1
        x ^= x >> np.uint64(33)
        x *= _M2
        x ^= x >> np.uint64(33)
    return x


def hash_values(x, salt):
    """H(x, s) = fmix64(((x+1) * GOLDEN64) ^ s) (_sigcore_py.py:45-48)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return fmix64(((x + np.uint64(1)) * np.uint64(GOLDEN64)) ^ np.uint64(salt))


def combine(words) -> int:
    """Boost-style fold (_sigcore_py.py:51-62), pure-int arithmetic."""
    mask = (1 << 64) - 1
    acc = 0
    for w in np.asarray(words, dtype=np.uint64).tolist():
        acc ^= (int(fmix64(np.uint64(w))) + GOLDEN64 + ((acc << 6) & mask) + (acc >> 2)) & mask
    return acc


def gen_mapping(d: int, t: int, k: int, seed: int) -> np.ndarray:
    """(d, t*k/2) uint64 mapping values (minmax_hash.py:86-89)."""
    n_funcs = t * (k // 2)
    base = np.arange(d, dtype=np.uint64)
    out = np.empty((d, n_funcs), dtype=np.uint64)
    for j in range(n_funcs):
        out[:, j] = hash_values(base, (seed + j) % 2**64)
    return out


def signatures_c(bits, values, t: int, k_half: int, threads: int = 1) -> np.ndarray:
    """C restatement (minmax_oracle.c), row ranges over pthreads."""
    bits = np.ascontiguousarray(bits, dtype=np.uint32)
    values = np.ascontiguousarray(values, dtype=np.uint64)
    n, K = bits.shape
    out = np.empty((n, t), dtype=np.uint64)
    if n == 0:
        return out
    rc = c_lib().qso_signatures(bits.ctypes.data, n, K, values.ctypes.data,
                                values.shape[1], t, k_half, out.ctypes.data,
                                int(threads))
    if rc:
        raise ValueError(f"oracle signatures failed rc={rc}")
    return out


def signatures_function_major(bits, values, t: int, k_half: int) -> np.ndarray:
    """Column-at-a-time numpy restatement (the reference's own slow oracle,
    bench.py:51-73): min/max per hash column over all rows, then fold."""
    bits = np.asarray(bits, dtype=np.uint32)
    n = bits.shape[0]
    F = values.shape[1]
    mins = np.empty((n, F), np.uint64)
    maxs = np.empty((n, F), np.uint64)
    for f in range(F):
        v = values[:, f][bits]
        mins[:, f] = v.min(axis=1)
        maxs[:, f] = v.max(axis=1)
    acc = np.zeros((n, t), np.uint64)
    g = np.uint64(GOLDEN64)
    with np.errstate(over="ignore"):
        for j in range(k_half):
            w = mins.reshape(n, t, k_half)[:, :, j]
            acc ^= fmix64(w) + g + (acc << np.uint64(6)) + (acc >> np.uint64(2))
        for j in range(k_half):
            w = maxs.reshape(n, t, k_half)[:, :, j]
            acc ^= fmix64(w) + g + (acc << np.uint64(6)) + (acc >> np.uint64(2))
    return acc


def signatures_reference_kernel(bits, values, t: int, k_half: int, threads: int = 1):
    """The reference's compiled `_sigcore.gen_signatures_range` (oracle/_ref),
    row-split over a thread pool exactly like minmax_hash.py:113-128.
    Returns None if the reference kernel was not built."""
    core = ref_sigcore()
    if core is None:
        return None
    bits = np.ascontiguousarray(bits, dtype=np.uint32)
    values = np.ascontiguousarray(values, dtype=np.uint64)
    n = bits.shape[0]
    out = np.empty((n, t), dtype=np.uint64)
    if n == 0:
        return out
    threads = max(1, int(threads))
    if threads == 1 or n < 2 * threads:
        core.gen_signatures_range(bits, values, t, k_half, out, 0, n)
        return out
    from concurrent.futures import ThreadPoolExecutor
    bounds = np.linspace(0, n, threads + 1, dtype=int)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        futs = [pool.submit(core.gen_signatures_range, bits, values, t, k_half,
                            out, int(lo), int(hi))
                for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
        for f in futs:
            f.result()
    return out
