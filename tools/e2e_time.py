"""search_fingerprints e2e (host bits in, host triplets out) at cfg1 N = 8e6
for the host-transfer settings: pinned direct DMA, pinned with a narrowed
share (QS_H2D_SPLIT), pageable narrowed / plain.  Prints seconds per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1803_09835_b200 import lsh_search as ls, workloads
from paper_1803_09835_b200.fingerprint import FingerprintSet
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
pin = torch.empty(tuple(bits.shape), dtype=torch.int32, pin_memory=True)
pin.copy_(bits)
del bits
torch.cuda.empty_cache()
cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0, occurrence_threshold=1.5e-5,
                      near_repeat_exclusion_s=0.0)


def run(host_bits, label, env):
    for k, v in env.items():
        os.environ[k] = v
    fps = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                         indices=np.arange(n, dtype=np.uint64), epochs=np.arange(n, dtype=np.float64),
                         bits=host_bits)
    ls.search_fingerprints(fps, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rec, st, _ = ls.search_fingerprints(fps, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:34s} min {min(ts):.4f} median {sorted(ts)[len(ts) // 2]:.4f} s  h2d {ls.LAST_H2D_BYTES / 1e9:.2f} GB "
          f"triplets {len(rec)} split {ls.LAST_H2D_SPLIT:.3f}", flush=True)
    for k in env:
        os.environ.pop(k, None)


hp = pin.numpy().view(np.uint32)
for sp in os.environ.get("QS_E2E_SPLITS", "0,0.5,0.7,0.8,0.9,1").split(","):
    run(hp, f"pinned split={sp}", {} if sp == "auto" else {"QS_H2D_SPLIT": sp})
pg = np.array(hp)
for thr_env in ({}, {"QS_H2D_NARROW": "0"}):
    run(pg, f"pageable {thr_env or 'narrowed'}", thr_env)
