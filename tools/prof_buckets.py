"""One bucket build (+ listing) at cfg1 scale, for per-kernel timing under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
for _ in range(2):
    ds = ls.DeviceSearch(keys, rkeys, tags, n, 100, timing=True)
    ds.buckets()
    torch.cuda.synchronize()
print({k: round(v, 2) for k, v in ds.stage_times_ms().items()}, ds.nb, ds.heads)
