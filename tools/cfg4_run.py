"""BASELINE configs[4] on one B200: 10 stations x 1 year at 100 Hz, shared
events with station-specific delays (0-8 s) and gains (0.3-3x), independent
noise per station.  Each station runs the whole path on its own trace
(fingerprint_series -> search_fingerprints, t=100, k=4, m=5, occurrence
filter 1 %, exclusion windows from the fingerprint geometry), one station after another on one GPU (on
N GPUs the stations are dealt to ranks: bench.py --shard stations).  Prints
one JSON line per station and a total.

    python tools/cfg4_run.py [stations=10] [n_samples=3.15e9]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import lsh_search as ls  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import TimeSeries  # noqa: E402

stations = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 3_150_000_000
ev = workloads.cfg4_events(n_samples=n, stations=stations)
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
cfg = ls.SearchConfig(**workloads.CFG0_SEARCH)
tot_fp_ms = tot_se_ms = 0.0
tot_fps = 0
t_all = time.time()
for s in range(stations):
    x = workloads.cfg4_station_torch(s, ev, n_samples=n)
    torch.cuda.synchronize()
    ts = TimeSeries(f"ST{s}", "HHZ", workloads.SR_HZ, 0.0, x)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
    e[1].record()
    torch.cuda.synchronize()
    del ts, x
    torch.cuda.empty_cache()
    e[1].record()
    trip, st, mapping = ls.search_fingerprints(fps, cfg)
    e[2].record()
    torch.cuda.synchronize()
    fp_ms, se_ms = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    nfp = int(fps.bits.shape[0])
    tot_fp_ms += fp_ms
    tot_se_ms += se_ms
    tot_fps += nfp
    print(json.dumps({"station": s, "gain": float(ev["gains"][s]), "n_fingerprints": nfp,
                      "fingerprint_ms": fp_ms, "search_ms": se_ms,
                      "emitted_triplets": st.emitted_triplets,
                      "distinct_pairs": st.distinct_pairs,
                      "filtered_fingerprints": st.filtered_fingerprints,
                      "max_bucket": st.max_bucket}), flush=True)
    del fps, trip, mapping
    torch.cuda.empty_cache()
print(json.dumps({"workload": "cfg4 (BASELINE.json configs[4]): 10 stations x 1 year at 100 Hz, "
                              "device-generated, stations run one after another on 1 GPU",
                  "stations": stations, "n_samples_per_station": n,
                  "n_fingerprints": tot_fps, "fingerprint_ms": tot_fp_ms, "search_ms": tot_se_ms,
                  "device_s": (tot_fp_ms + tot_se_ms) / 1e3,
                  "fp_per_s_end_to_end": tot_fps / ((tot_fp_ms + tot_se_ms) / 1e3),
                  "wall_s_incl_generation": time.time() - t_all}), flush=True)
