"""Key-bin occupancy of the cfg1 workload (design aid for the binned bucket build)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
del rkeys, tags, bits
out = {"n": n}
for bb in (11, 12, 13):
    mx, over, overm = [], 0, 0
    for t in range(keys.shape[0]):
        b = (keys[t].view(torch.int64) >> (64 - bb)) & ((1 << bb) - 1)
        c = torch.bincount(b, minlength=1 << bb)
        mx.append(int(c.max()))
        over += int((c > 6144).sum()); overm += int(c[c > 6144].sum())
    out[f"bb{bb}"] = dict(max=max(mx), median_table_max=int(np.median(mx)), bins_over_6144=over, members_over=overm)
# largest buckets per table
big = []
for t in range(0, keys.shape[0], 10):
    u, c = torch.unique(keys[t], return_counts=True)
    big.append(sorted(c.tolist())[-5:])
out["top_buckets_every_10th_table"] = big
print(json.dumps(out))
