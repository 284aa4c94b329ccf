"""One pair pass (mode, bucket-size window) at cfg1 after a warm-up, for ncu
launch lists of the small-bucket and tile kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads
mode_name, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 8_000_000
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
del bits
ds = ls.DeviceSearch(keys, rkeys, tags, n, 100)
ds.buckets()
edges = torch.tensor([0, n], dtype=torch.int64, device="cuda")
mode = {"matched": ds.MODE_MATCHED, "distinct": ds.MODE_DISTINCT, "full": ds.MODE_FULL}[mode_name]
os.environ["QS_PAIRS_SMIN"], os.environ["QS_PAIRS_SMAX"] = lo, hi
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pk, ps, matched, distinct = ds.pairs(mode, 5, 0, None, edges, 1)
    e1.record()
    torch.cuda.synchronize()
    print(mode_name, lo, hi, "ms", round(e0.elapsed_time(e1), 2), "matched", matched, "distinct", distinct, flush=True)
