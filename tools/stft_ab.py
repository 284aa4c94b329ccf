"""A/B of the band STFT kernels (QS_STFT_KERNEL=fma: FMA chain per column;
default: DMMA tensor-core kernel).  Writes the band rows of the cfg0 day to
/tmp/stft_<tag>.npy and times the band STFT of the cfg2 trace.

    QS_STFT_KERNEL=fma python tools/stft_ab.py fma; python tools/stft_ab.py mma
    python tools/stft_ab.py cmp          # ulp comparison of the two files
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

tag = sys.argv[1]
out = "/tmp"
if tag == "cmp":
    a = np.load(os.path.join(out, "stft_fma.npy"))
    b = np.load(os.path.join(out, "stft_mma.npy"))
    ai, bi = a.view(np.int32).astype(np.int64), b.view(np.int32).astype(np.int64)
    u = np.abs(ai - bi)
    print(f"band values {a.size}: identical {np.mean(u == 0):.7f}, max ulp {u.max()}, "
          f"values off by 1 ulp {(u == 1).sum()}, >1 ulp {(u > 1).sum()}")
    sys.exit(0)

import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import TimeSeries  # noqa: E402

p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
x, _ = workloads.cfg0_trace(n_samples=8_640_000, seed=0)
ch = fp._Chain(TimeSeries("S", "C", 100.0, 0.0, x), params)
torch.cuda.synchronize()
np.save(os.path.join(out, f"stft_{tag}.npy"), ch.band.cpu().numpy())
xd, _ = workloads.cfg2_trace_torch(n_samples=795_000_000)
ts = TimeSeries("S", "C", 100.0, 0.0, xd)
fp._Chain(ts, params)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    fp._Chain(ts, params)
b.record()
torch.cuda.synchronize()
print(f"{tag}: cfg2 band STFT {a.elapsed_time(b) / 3:.2f} ms")
