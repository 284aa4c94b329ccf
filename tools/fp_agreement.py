import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_09835_b200 import fingerprint as fp, workloads
from paper_1803_09835_b200.ingest import TimeSeries
from oracle import fingerprint as ofp
x, _ = workloads.cfg0_trace(n_samples=400_000, seed=5, copies=4)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"], freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"], band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"], stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
fps, _ = fp.fingerprint_series(TimeSeries("S", "C", 100.0, 0.0, x), params)
want = ofp.fingerprint(x, 100.0, p)
eq = fps.bits == want["bits"]
print("agreement", eq.mean(), "rows differing", int((~eq.all(axis=1)).sum()), "of", len(eq))
