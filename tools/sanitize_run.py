"""Small run of every asynchronous kernel family for compute-sanitizer
(racecheck / synccheck / memcheck): the pair kernel in all modes
(FULL / MATCHED with lazy counts / DISTINCT on compacted and masked lists,
big-bucket segments via a collide-prone set), the bucket radix build, the
Min-Max signature kernel, the fingerprint window kernel (images, coeffs,
MAD columns, top-K), the band-pass scan and the triplet combine."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import lsh_search as ls  # noqa: E402
from paper_1803_09835_b200 import minmax_hash as mh  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import BandpassSpec, TimeSeries, bandpass  # noqa: E402

n = int(os.environ.get("QS_SAN_N", "2000"))
bits, _ = workloads.cfg1_bits(n=n, seed=7, pair_frac=1 / 40, group_frac=1 / 200, group_size=100)
m = mh.gen_hash_mapping(4096, 100, 4, 0)
sigs = mh.signatures(bits, m)
for occ, p, excl in [(None, 1, 0), (40 / n, 1, 0), (40 / n, 3, 2)]:
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, partitions=p,
                          occurrence_threshold=occ)
    rec, st = ls.search_signatures(sigs, cfg, exclusion_windows=excl)
    print("search", occ, p, rec.size, st.distinct_pairs, flush=True)
# collide-prone: big buckets -> segment items, t = 40 (W = 2)
rng = np.random.default_rng(1)
s2 = rng.integers(0, 3, size=(1500, 40)).astype(np.uint64)
for occ in (None, 0.3):
    rec, st = ls.search_signatures(s2, ls.SearchConfig(tables=40, hash_funcs=2, min_matches=3,
                                                       occurrence_threshold=occ))
    print("prone", occ, rec.size, st.distinct_pairs, flush=True)
# fingerprint chain (windows kernel: MAD columns + top-K) and coefficient batches
x, _ = workloads.cfg0_trace(n_samples=30_000, seed=3, copies=2)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("S", "C", 100.0, 0.0, x)
fps, mad = fp.fingerprint_series(ts, params)
list(fp.iter_coeff_batches(ts, params, batch=64))
list(fp.iter_image_batches(ts, params, indices=[0, 5, 9], batch=64))
bandpass(ts, BandpassSpec(4.0, 10.0, 4))
print("fingerprints", fps.bits.shape, flush=True)
torch.cuda.synchronize()
print("SANITIZE_RUN_OK")
