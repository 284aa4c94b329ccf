"""Min-Max hash signatures on the B200 — drop-in for reference minmax_hash.py.

Same public surface as the reference module (minmax_hash.py:1-128): the hash
family (`GOLDEN64`, `fmix64`, `hash_values`, `combine`, host-side helpers on
numpy scalars/arrays exactly as the reference exposes them), `HashMapping`,
`gen_hash_mapping`, `signatures`, `backend_name`, `BACKEND`.  The signature
computation itself runs only in the sm_100a kernel (csrc/qs_minmax.cu) —
there is no CPU fallback.

`signatures()` accepts a host numpy array (returns numpy, like the
reference) or a CUDA torch tensor (returns a CUDA tensor, no host copies).
`workers` is accepted for API compatibility and ignored: rows are spread
over all SMs by the kernel.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ParameterError

BACKEND = "cuda"
GOLDEN64 = 0x9E3779B97F4A7C15

_M1 = np.uint64(0xFF51AFD7ED558CCD)
_M2 = np.uint64(0xC4CEB9FE1A85EC53)


def backend_name(pure_python: bool | None = None) -> str:
    """Name of the signature kernel in use (always 'cuda'; the reference's
    'cython'/'python' backends are replaced, minmax_hash.py:43-47)."""
    return BACKEND


def fmix64(x):
    """Murmur3 64-bit finalizer over a uint64 array (host helper, reference
    _sigcore_py.py:34-42)."""
    x = np.array(x, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= _M1
        x ^= x >> np.uint64(33)
        x *= _M2
        x ^= x >> np.uint64(33)
    return x


def hash_values(x, seed):
    """H(x, seed) = fmix64(((x + 1) * GOLDEN64) ^ seed) (host helper)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return fmix64(((x + np.uint64(1)) * np.uint64(GOLDEN64)) ^ np.uint64(seed))


def combine_step(acc, w):
    with np.errstate(over="ignore"):
        acc ^= fmix64(w) + np.uint64(GOLDEN64) + (acc << np.uint64(6)) + (acc >> np.uint64(2))
    return acc


def combine(words):
    """Fold a 1-D sequence of uint64 words into one signature word (host helper)."""
    acc = np.zeros(1, dtype=np.uint64)
    for w in np.asarray(words, dtype=np.uint64):
        combine_step(acc, w)
    return int(acc[0])


@dataclass
class HashMapping:
    """t * k/2 random mappings from element index to uint64 (minmax_hash.py:50-70).

    values[x, j] = H(x, seed + j).  The device copy and the probe plan are
    cached on first use."""

    d: int
    t: int
    k: int
    seed: int
    values: np.ndarray = field(repr=False)
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def k_half(self) -> int:
        return self.k // 2

    @property
    def n_funcs(self) -> int:
        return self.t * self.k_half

    def device_plan(self):
        """(values_dev, plan_dev) CUDA tensors for the current device."""
        torch = nat.torch()
        dev = torch.cuda.current_device()
        hit = self._dev.get(dev)
        if hit is not None and hit[2] is self.values:
            return hit[0], hit[1]
        vals = np.ascontiguousarray(self.values, dtype=np.uint64)
        if vals.shape != (self.d, self.n_funcs):
            raise ParameterError("mapping values shape does not match (d, t*k/2)")
        vdev = torch.from_numpy(vals.view(np.int64)).to(f"cuda:{dev}")
        plan = torch.empty(int(nat.lib().qs_minmax_plan_bytes(self.d, self.n_funcs)),
                           dtype=torch.uint8, device=f"cuda:{dev}")
        nat.call("qs_minmax_plan", nat.ptr(vdev), self.d, self.n_funcs, nat.ptr(plan), nat.stream())
        self._dev[dev] = (vdev, plan, self.values)
        return vdev, plan


def gen_hash_mapping(d: int, t: int, k: int, seed: int) -> HashMapping:
    """Generate the hash mapping table for (d, t, k) (minmax_hash.py:73-90);
    the table is computed on the GPU and mirrored to the host `values`."""
    if d < 1:
        raise ParameterError(f"d must be >= 1, got {d}")
    if t < 1:
        raise ParameterError(f"t must be >= 1, got {t}")
    if k < 2 or k % 2 != 0:
        raise ParameterError(f"k must be a positive even number, got {k}")
    if not 0 <= seed < 2**64:
        raise ParameterError("seed must fit in uint64")
    torch = nat.torch()
    n_funcs = t * (k // 2)
    vdev = torch.empty((d, n_funcs), dtype=torch.int64, device="cuda")
    nat.call("qs_gen_hash_mapping", nat.ptr(vdev), d, n_funcs, int(seed), nat.stream())
    values = vdev.cpu().numpy().view(np.uint64)
    m = HashMapping(d=d, t=t, k=k, seed=seed, values=values)
    return m


def _device_bits(bits):
    """Validate and return (bits_dev int32 (n, K) CUDA tensor, is_host)."""
    torch = nat.torch()
    if nat.is_device_tensor(bits):
        if bits.dim() != 2:
            raise ParameterError("bits must be a 2-D (n, K) array")
        if bits.dtype not in (torch.int32, torch.uint32):
            bits = bits.to(torch.int32)
        return bits.contiguous(), False
    arr = np.ascontiguousarray(bits, dtype=np.uint32)
    if arr.ndim != 2:
        raise ParameterError("bits must be a 2-D (n, K) array")
    return arr, True


def signatures(bits, mapping: HashMapping, workers: int = 1):
    """Min-Max signatures (n, t) uint64 of an (n, K) set-bit array
    (minmax_hash.py:93-128; kernel _sigcore.pyx:32-85)."""
    torch = nat.torch()
    b, host = _device_bits(bits)
    n, K = b.shape
    if K < 1:
        raise ParameterError("fingerprints must have at least one set bit")
    if host:
        if n and int(b.max()) >= mapping.d:
            raise ParameterError("fingerprint bit index out of range for mapping")
        out = np.empty((n, mapping.t), dtype=np.uint64)
        if n == 0:
            return out
        bdev = torch.from_numpy(b.view(np.int32)).to("cuda")
    else:
        bdev = b
        if n == 0:
            return torch.empty((0, mapping.t), dtype=torch.int64, device=b.device)
    _, plan = mapping.device_plan()
    sig = torch.empty((n, mapping.t), dtype=torch.int64, device=bdev.device)
    bad = torch.zeros(1, dtype=torch.int32, device=bdev.device)
    nat.call("qs_minmax_signatures", nat.ptr(bdev), n, K, nat.ptr(plan), mapping.d, mapping.t,
             mapping.k_half, nat.ptr(sig), nat.ptr(bad), nat.stream())
    if int(bad.item()):
        raise ParameterError("fingerprint bit index out of range for mapping")
    if host:
        return sig.cpu().numpy().view(np.uint64)
    return sig
