"""Bucket-size distribution of the cfg1 workload (design aid for the pair kernels)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
ds = ls.DeviceSearch(keys, rkeys, tags, n, 100)
ds.buckets()
bs = ds.bsize[: ds.nb].to(torch.int64).cpu().numpy()
pairs = bs * (bs - 1) // 2
out = {"n": n, "nonsingle": int(ds.nb), "heads": int(ds.heads), "members_nonsingle": int(bs.sum()),
       "pairs": int(pairs.sum())}
edges = [2, 3, 5, 9, 17, 33, 65, 129, 257, 513, 1025, 2049, 4097, 1 << 40]
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = (bs >= lo) & (bs < hi)
    out[f"{lo}-{hi-1}"] = dict(buckets=int(sel.sum()), members=int(bs[sel].sum()), pairs=int(pairs[sel].sum()))
print(json.dumps(out, indent=1))
