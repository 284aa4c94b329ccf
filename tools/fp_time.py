"""cfg2 fingerprint_series timing as bench.py's fingerprint leg does it
(device trace, CUDA events over K calls), without the rest of the bench."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import TimeSeries  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 795_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x, _ = workloads.cfg2_trace_torch(n_samples=n)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x)
fps, _ = fp.fingerprint_series(ts, params, mad_rate=0.1)
del fps
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
t0 = time.perf_counter()
for _ in range(steps):
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
print(f"cfg2 fingerprint_series: {ms:.1f} ms/step, {n / ms / 1e3:.0f} Msamples/s "
      f"(host wall {1e3 * (time.perf_counter() - t0) / steps:.1f} ms)")
