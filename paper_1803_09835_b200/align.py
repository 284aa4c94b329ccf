"""Channel combination and triplet sort on the GPU (reference align.py:45-140).

`combine_channel_triplets` and `sort_triplet_file` keep the reference's
signatures, error taxonomy and output bytes; the merge runs as one device
sort + reduce-by-key (csrc/qs_align.cu) over all channels' records instead
of a k-way heap merge in Python.  Clustering / association (the rest of the
reference module) stay out of scope.
"""

import numpy as np

from . import _native as nat
from .errors import ConsistencyError, ParameterError
from .lsh_search import TRIPLET_DTYPE, read_triplet_file, write_triplet_file


def _keys(rec):
    """(dt << 32 | idx1) of packed CUDA records, int64 view."""
    torch = nat.torch()
    r = rec.view(-1, TRIPLET_DTYPE.itemsize)
    dt = r[:, 0:8].contiguous().view(torch.int64).view(-1)
    i1 = r[:, 8:16].contiguous().view(torch.int64).view(-1)
    return dt, i1


def _check_sorted(path, rec) -> None:
    n = rec.numel() // TRIPLET_DTYPE.itemsize
    if n < 2:
        return
    torch = nat.torch()
    dt, i1 = _keys(rec)
    ddt = dt[1:] - dt[:-1]
    bad = (ddt < 0) | ((ddt == 0) & (i1[1:] < i1[:-1]))
    if bool(torch.any(bad).item()):
        raise ConsistencyError(f"{path}: triplets not sorted by (dt, idx1)")


def combine_records(records, threshold: int):
    """Device combine of packed CUDA triplet records (one tensor per channel,
    or one concatenation): sort by (dt, idx1), sum sims of equal pairs, keep
    sums >= threshold (threshold 0: sort only).  Returns packed records."""
    torch = nat.torch()
    rec = torch.cat([r.view(-1) for r in records]) if isinstance(records, (list, tuple)) else records
    n = rec.numel() // TRIPLET_DTYPE.itemsize
    out = torch.empty(max(n, 1) * TRIPLET_DTYPE.itemsize, dtype=torch.uint8, device=rec.device)
    if n == 0:
        return out[:0]
    dt, i1 = _keys(rec)
    hi = int(torch.max(dt).item())
    key_bits = 32 + max(1, hi.bit_length()) if hi < (1 << 32) else 64
    lib = nat.lib()
    ws = torch.empty(lib.qs_triplets_combine_ws_bytes(n), dtype=torch.uint8, device=rec.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=rec.device)
    nat.call("qs_triplets_combine", nat.ptr(rec), n, int(threshold), key_bits, nat.ptr(out),
             nat.ptr(cnt), nat.ptr(ws), ws.numel(), nat.stream())
    return out[: int(cnt.item()) * TRIPLET_DTYPE.itemsize]


def combine_channel_triplets(paths, dst, threshold: int, header: dict) -> int:
    """Merge per-channel triplet files of one station (align.py:113-140):
    window pairs matched on several channels get their counts summed, sums
    below `threshold` are dropped; inputs and output sorted by (dt, idx1).
    Returns the number of records written."""
    if not paths:
        raise ParameterError("no triplet files to combine")
    if threshold < 1:
        raise ParameterError("threshold must be >= 1")
    recs = []
    for p in paths:
        rec, _ = read_triplet_file(p, device=True)
        _check_sorted(p, rec)
        recs.append(rec)
    out = combine_records(recs, threshold)
    write_triplet_file(dst, out, header)
    return out.numel() // TRIPLET_DTYPE.itemsize


def sort_triplet_file(src, dst, header: dict, chunk_records: int = 2_000_000) -> int:
    """Sort a triplet file by (dt, idx1) (align.py:87-110).  The whole file is
    sorted in HBM; `chunk_records` is validated for API parity only."""
    if chunk_records < 1:
        raise ParameterError("chunk_records must be >= 1")
    rec, _ = read_triplet_file(src, device=True)
    out = combine_records(rec, 0)
    write_triplet_file(dst, out, header)
    return out.numel() // TRIPLET_DTYPE.itemsize


def combine_host(records: list, threshold: int) -> np.ndarray:
    """Host-array convenience wrapper of combine_records."""
    torch = nat.torch()
    devs = [torch.from_numpy(np.ascontiguousarray(r, dtype=TRIPLET_DTYPE).view(np.uint8)).cuda()
            for r in records]
    return combine_records(devs, threshold).cpu().numpy().view(TRIPLET_DTYPE)
