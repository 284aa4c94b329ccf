"""Device-resident fingerprint_series on cfg0 (one warm-up, one measured call) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09835_b200 import fingerprint as fp, workloads
from paper_1803_09835_b200.ingest import TimeSeries
x, _ = workloads.cfg0_trace(n_samples=8_640_000, seed=0)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, torch.from_numpy(x).cuda())
for _ in range(2):
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
    torch.cuda.synchronize()
print(fps.bits.shape)
