"""Device-resident fingerprint_series on cfg2 (7.95e8 samples): one warm-up,
one measured call (for ncu launch lists / captures), plus a CUDA-event stage
split of the measured call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import TimeSeries  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 795_000_000
x, _ = workloads.cfg2_trace_torch(n_samples=n)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x)
for _ in range(2):
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
    torch.cuda.synchronize()
print(fps.bits.shape)
