"""Host -> device copy strategies for the e2e path (12.8 GB of fingerprint bits)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
nbytes = int(float(sys.argv[1])) if len(sys.argv) > 1 else 12_800_000_000
a = np.ones(nbytes // 4, dtype=np.int32)
print("cores", len(os.sched_getaffinity(0)), flush=True)

def staged(arr, chunk=256 << 20, threads=1, nbuf=2):
    flat = arr.reshape(-1)
    out = torch.empty(flat.size, dtype=torch.int32, device="cuda")
    per = chunk // 4
    stage = [torch.empty(per, dtype=torch.int32).pin_memory() for _ in range(nbuf)]
    done = [None] * nbuf
    pool = ThreadPoolExecutor(threads) if threads > 1 else None
    for k, s0 in enumerate(range(0, flat.size, per)):
        e0 = min(flat.size, s0 + per)
        b = k % nbuf
        if done[b] is not None:
            done[b].synchronize()
        dst = stage[b].numpy()
        if pool:
            n = e0 - s0
            step = -(-n // threads)
            list(pool.map(lambda i: np.copyto(dst[i:min(n, i + step)], flat[s0 + i:s0 + min(n, i + step)]),
                          range(0, n, step)))
        else:
            dst[: e0 - s0] = flat[s0:e0]
        out[s0:e0].copy_(stage[b][: e0 - s0], non_blocking=True)
        ev = torch.cuda.Event(); ev.record(); done[b] = ev
    torch.cuda.synchronize()
    return out

def registered(arr):
    cr = torch.cuda.cudart()
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    t1 = time.perf_counter()
    src = torch.from_numpy(arr)
    out = torch.empty_like(src, device="cuda")
    out.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(arr.ctypes.data)
    t3 = time.perf_counter()
    print("  register %.3f copy %.3f unregister %.3f rc %s" % (t1 - t0, t2 - t1, t3 - t2, rc), flush=True)
    return out

for name, fn in [("staged1", lambda: staged(a)), ("staged8", lambda: staged(a, threads=8)),
                 ("staged16x512", lambda: staged(a, chunk=512 << 20, threads=16, nbuf=3)),
                 ("registered", lambda: registered(a))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); o = fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(name, "%.3f s  %.1f GB/s" % (dt, nbytes / dt / 1e9), flush=True)
    del o
