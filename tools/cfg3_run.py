"""BASELINE configs[3] on one B200, end to end: one year at 100 Hz (3.15e9
samples, ~3.15e7 fingerprints at 1 s lag) -> fingerprint_series (STFT,
MAD sample, top-K bits) -> search_fingerprints (Min-Max, t=100 tables,
k=4, m=5, occurrence filter 1 %, near-repeat exclusion 10 windows).  The
trace is generated on the device (workloads.cfg3_trace_torch: the 50
periodic templates bounded, see its docstring).  Log -> profiles/.

    python tools/cfg3_run.py [n_samples=3.15e9]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_09835_b200 import fingerprint as fp  # noqa: E402
from paper_1803_09835_b200 import lsh_search as ls  # noqa: E402
from paper_1803_09835_b200 import workloads  # noqa: E402
from paper_1803_09835_b200.ingest import TimeSeries  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 3_150_000_000
t0 = time.time()
x, truth = workloads.cfg3_trace_torch(n_samples=n)
torch.cuda.synchronize()
t_gen = time.time() - t0
p = workloads.CFG0_PARAMS
params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                              freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                              band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                              stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
ev[1].record()
torch.cuda.synchronize()
del ts, x
torch.cuda.empty_cache()
cfg = ls.SearchConfig(**workloads.CFG0_SEARCH)
torch.cuda.reset_peak_memory_stats()
ev[1].record()
trip, st, mapping = ls.search_fingerprints(fps, cfg)
ev[2].record()
torch.cuda.synchronize()
fp_ms = ev[0].elapsed_time(ev[1])
se_ms = ev[1].elapsed_time(ev[2])
nfp = int(fps.bits.shape[0])
out = {"workload": "cfg3 (BASELINE.json configs[3]): 1 year at 100 Hz, device-generated",
       "n_samples": n, "n_fingerprints": nfp, "generator_s": t_gen,
       "fingerprint_ms": fp_ms, "fingerprint_msamples_per_s": n / fp_ms / 1e3,
       "search_ms": se_ms, "search_fp_per_s": nfp / (se_ms / 1e3),
       "end_to_end_s": (fp_ms + se_ms) / 1e3,
       "emitted_triplets": st.emitted_triplets, "distinct_pairs": st.distinct_pairs,
       "filtered_fingerprints": st.filtered_fingerprints, "lookups_total": st.lookups_total,
       "n_buckets": st.n_buckets, "max_bucket": st.max_bucket,
       "search_peak_mem_gb": torch.cuda.max_memory_allocated() / 2**30,
       "planted": {"events": len(truth["events"]), "periodic": truth["periodic"],
                   "cells": truth["cells"]}}
print(json.dumps(out), flush=True)
