"""Plugin module with the reference's native-kernel contract.

The reference picks its signature kernel at import as `_core`
(minmax_hash.py:24-30) and calls
`_core.gen_signatures_range(bits, values, t, k_half, out, start, stop)`
(_sigcore.pyx:32-36) on host numpy buffers.  This module has exactly that
interface (plus BACKEND_NAME) and forwards to the C-ABI host entry
`qs_gen_signatures_range`, so a reference maintainer can bind it with one
line:  `from paper_1803_09835_b200 import _sigcore_cuda as _core`.
"""

import numpy as np

from . import _native as nat

BACKEND_NAME = "cuda"


def gen_signatures_range(bits, values, t, k_half, out, start, stop):
    """Fill out[start:stop] with t-word Min-Max signatures of bits[start:stop]."""
    bits = np.asarray(bits)
    values = np.asarray(values)
    if bits.dtype != np.uint32 or not bits.flags.c_contiguous or bits.ndim != 2:
        raise ValueError("bits must be a C-contiguous (n, K) uint32 array")
    if values.dtype != np.uint64 or not values.flags.c_contiguous or values.ndim != 2:
        raise ValueError("values must be a C-contiguous (d, F) uint64 array")
    if out.dtype != np.uint64 or not out.flags.c_contiguous or out.shape != (bits.shape[0], t):
        raise ValueError("out must be a C-contiguous (n, t) uint64 array")
    nat.call("qs_gen_signatures_range", bits.ctypes.data, bits.shape[0], bits.shape[1],
             values.ctypes.data, values.shape[0], values.shape[1], int(t), int(k_half),
             out.ctypes.data, int(start), int(stop))
