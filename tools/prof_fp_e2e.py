"""Host-side profile of fingerprint_series with a host trace (e2e path)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_09835_b200 import fingerprint as fp, workloads
from paper_1803_09835_b200.ingest import TimeSeries
x, _ = workloads.cfg0_trace(n_samples=8_640_000, seed=0)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x)
fp.fingerprint_series(ts, params, mad_rate=0.1); torch.cuda.synchronize()
t0 = time.perf_counter(); fp.fingerprint_series(ts, params, mad_rate=0.1); torch.cuda.synchronize()
print("e2e s", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); fp.fingerprint_series(ts, params, mad_rate=0.1); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
