"""North-star comparison: time the
HBM open-addressed pair-count table the north star names (one atomic insert
per candidate (pair, table) hit) on this B200, then project it to cfg1
(H = 2.8e10 hits over 2.55e10 distinct pairs at N = 8e6) and compare with the
first-colliding-table enumeration's measured pair stage.

    python tools/pair_table_bench.py [slots_log2=30] [inserts=4e9]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_09835_b200 import _native as nat  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 4_000_000_000
slots = 1 << lg
table = torch.zeros(slots * 12, dtype=torch.uint8, device="cuda")
probes = torch.zeros(1, dtype=torch.int64, device="cuda")
for load, hits_per_key in [(0.5, 1.1), (0.7, 1.1), (0.5, 4.0)]:
    distinct = int(slots * load)
    nn = min(n, int(distinct * hits_per_key))
    table.zero_()
    probes.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    nat.call("qs_bench_pair_table", nn, distinct, nat.ptr(table), slots, nat.ptr(probes), nat.stream())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    rate = nn / (ms / 1e3)
    cfg1_s = 2.8e10 / rate
    print(f"table {slots:.3g} slots ({slots * 12 / 1e9:.1f} GB), load {load}, {nn:.3g} inserts of "
          f"{distinct:.3g} keys: {ms:.1f} ms = {rate / 1e9:.2f} G inserts/s, "
          f"{int(probes.item()) / nn:.2f} probes/insert -> cfg1 (2.8e10 hits) {cfg1_s * 1e3:.0f} ms "
          f"(+ a 2.55e10-slot table: {2.55e10 / load * 12 / 1e9:.0f} GB, > one B200)", flush=True)
