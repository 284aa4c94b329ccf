"""One cfg1 search at N = 8e6 after one warm-up (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=1.5e-5)
for _ in range(2):
    keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
    trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0)
    torch.cuda.synchronize()
print(st.emitted_triplets, st.distinct_pairs)
