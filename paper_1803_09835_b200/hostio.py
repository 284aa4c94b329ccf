"""Device <-> file streaming through pinned double buffers.

Artifacts computed on the GPU (packed .fp records, .tri triplet records) are
written without materialising a pageable host copy: chunk i+1's D2H copy runs
while chunk i is written to the file, and reads overlap file I/O with the H2D
copy the same way.
"""

import numpy as np

from . import _native as nat

CHUNK = 64 << 20


def write_device_bytes(f, dev, chunk: int = CHUNK) -> None:
    """Append the bytes of a contiguous CUDA tensor to the open binary file f."""
    torch = nat.torch()
    flat = dev.contiguous().view(torch.uint8).view(-1)
    n = flat.numel()
    if n == 0:
        return
    per = min(chunk, n)
    bufs = [torch.empty(per, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    spans = [(a, min(n, a + per)) for a in range(0, n, per)]
    for k, (a, b) in enumerate(spans[:2]):
        bufs[k][: b - a].copy_(flat[a:b], non_blocking=True)
        evs[k].record()
    for k, (a, b) in enumerate(spans):
        s = k & 1
        evs[s].synchronize()
        f.write(memoryview(bufs[s].numpy()[: b - a]))
        if k + 2 < len(spans):
            a2, b2 = spans[k + 2]
            bufs[s][: b2 - a2].copy_(flat[a2:b2], non_blocking=True)
            evs[s].record()


def read_to_device(f, nbytes: int, chunk: int = CHUNK):
    """Read nbytes from the open binary file f into a new CUDA uint8 tensor."""
    torch = nat.torch()
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    if nbytes == 0:
        return out
    per = min(chunk, nbytes)
    bufs = [torch.empty(per, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    evs = [None, None]
    for k, a in enumerate(range(0, nbytes, per)):
        b = min(nbytes, a + per)
        s = k & 1
        if evs[s] is not None:
            evs[s].synchronize()
        view = bufs[s].numpy()[: b - a]
        got = f.readinto(memoryview(view))
        if got != b - a:
            from .errors import CorruptInputError
            raise CorruptInputError("file truncated")
        out[a:b].copy_(bufs[s][: b - a], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        evs[s] = ev
    return out


def as_host_u8(x) -> np.ndarray:
    return np.ascontiguousarray(x).view(np.uint8).reshape(-1)
