"""cfg2-scale fingerprinting (BASELINE configs[2]: 7.95e8 samples, ~7.9e6
fingerprints) on a device-resident trace: throughput and memory check."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09835_b200 import fingerprint as fp, workloads
from paper_1803_09835_b200.ingest import TimeSeries, BandpassSpec, bandpass
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 795_000_000
g = torch.Generator(device="cuda").manual_seed(2)
x = torch.randn(n, generator=g, device="cuda", dtype=torch.float32)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", 100.0, 0.0, x)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("fingerprints", len(fps), "s %.3f" % dt, "Msamples/s %.1f" % (n / dt / 1e6),
          "peak GB %.1f" % (torch.cuda.max_memory_allocated() / 1e9), flush=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
y = bandpass(ts, BandpassSpec(4.0, 10.0, 4))
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("bandpass s %.3f Msamples/s %.1f" % (dt, n / dt / 1e6), flush=True)
