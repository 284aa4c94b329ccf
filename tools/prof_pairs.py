"""Producer/consumer cycle breakdown of k_pairs_pc (needs a -DQS_PROF build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads, _native as nat
n = int(sys.argv[1]); occ = float(sys.argv[2]); gf = float(sys.argv[3])
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda", group_frac=gf)
m = mh.gen_hash_mapping(4096, 100, 4, 0)
cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=occ if occ > 0 else None)
lib = nat.lib(); fn = lib.qs_prof_read; fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = (ctypes.c_ulonglong * 8)()
for rep in range(2):
    keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
    fn(out, 1)
    trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0, timing=True)
    torch.cuda.synchronize()
    fn(out, 1)
v = list(out)
print("stages", {k: round(x, 1) for k, x in ds.stage_times_ms().items()})
print("producer wait_empty %.3g build %.3g | consumer wait_full %.3g compute %.3g drain %.3g (cycles summed over warps)" % (v[0], v[1], v[4], v[5], v[6]))
