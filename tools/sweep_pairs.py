"""Time the pair-enumeration stages for each library variant given on the
command line (built with different QS_* kernel configurations)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_1803_09835_b200 import lsh_search as ls, minmax_hash as mh, workloads
n = int(sys.argv[1])
bits, _ = workloads.cfg1_bits_torch(n=n, seed=1, device="cuda")
m = mh.gen_hash_mapping(4096, 100, 4, 0)
cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=1.5e-5)
res = []
for rep in range(3):
    keys, rkeys, tags, bad = ls.signatures_for_search(bits, m)
    trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0, timing=True)
    torch.cuda.synchronize()
    res.append(ds.stage_times_ms())
print(json.dumps({"stages": res[-1], "triplets": st.emitted_triplets, "distinct": st.distinct_pairs}))
''' % ROOT
n = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, QS_LIB_PATH=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code, n], env=env, capture_output=True, text=True)
    line = (out.stdout.strip().splitlines() or ["{}"])[-1]
    try:
        d = json.loads(line)
        s = d["stages"]
        print(os.path.basename(lib), "matched %.1f distinct %.1f" % (s.get("pairs_matched", 0), s.get("pairs_distinct", 0)),
              d["triplets"], d["distinct"], flush=True)
    except Exception:
        print(os.path.basename(lib), "FAILED", out.stderr[-600:], flush=True)
