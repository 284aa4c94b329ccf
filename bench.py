"""Benchmark of the hot path (BASELINE.json metric) — one JSON line on rank 0.

Headline workload (BASELINE.json configs[1]): N = 8e6 sparse
4096-bit fingerprints with exactly 400 set bits, 1e5 planted near-duplicate
pairs, 2e4 noise groups x 200 rows (Jaccard 0.7 to the group template);
b=100 tables, r=4 (k=4 Min-Max hash functions), m=5, occurrence filter
1.5e-5 (limit 120 matches: the value that makes the filter fire on this
generator).  A step = one pass of the hot path over that
batch, the same work `search_fingerprints(fps_on_device, cfg)` does: hash
mapping + probe plan -> Min-Max signatures (fused with the search layout) ->
per-table buckets -> first-colliding-table pair enumeration with exact
collision counts -> occurrence filter (+ second enumeration) -> bucket stats
-> (dt, idx1)-sorted triplets.  Inputs (12.8 GB of bits, larger than L2)
are resident in HBM when the timed region starts.

Sub-lines of the same JSON object:
  full_mode     the same step without the occurrence filter (the reference's
                default, SearchConfig.occurrence_threshold=None);
  same_n        the GPU at the CPU baseline's sample size (a measured
                like-for-like ratio against cpu_baseline);
  fingerprint   the second BASELINE metric, fingerprint Msamples/s, on
                configs[2] (7.95e8 samples of 1/f noise + 500 planted repeats,
                device-resident; e2e from a host trace), with its own
                cpu_baseline (the reference's fingerprint_series on a 1-day
                slice).

Multi-GPU: `--gpus N` (N > 1) runs N ranks over NCCL — launched by torchrun
(WORLD_SIZE set), or spawned here (torch.multiprocessing) when WORLD_SIZE is
unset.  Default `--shard tables`: ONE station's cfg1 batch table-sharded over
the ranks (rows block-distributed for Min-Max + NCCL all-gather, tables dealt
round-robin, degree/mark all-reduces for the filter; "scaling": "strong").
`--shard stations`: every rank searches its own station (weak scaling).
Time = max over ranks of CUDA-event time.

`--impl reference` times the reference's own CPU implementation
(baseline/_ref: the unmodified quakescan package — compiled _sigcore
signatures on all host cores + its numpy search_signatures) on a bounded
sample of the same workload (N = --ref-n rows of the cfg1 generator, the
same limit-120 filter), rank 0 only.
"""

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
METRIC = "LSH search fingerprints/sec (MinHash+bucket+pair-count)"
N_FULL = 8_000_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fingerprints", dest="n", type=int, default=N_FULL)
    ap.add_argument("--occ", type=float, default=1.5e-5, help="occurrence threshold (<=0: off)")
    ap.add_argument("--ref-n", type=int, default=50_000, help="CPU sample rows (cfg1 generator)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--full-steps", type=int, default=2, help="FULL-mode sub-line steps (0: off)")
    ap.add_argument("--group-frac", type=float, default=1 / 400, help="noise-group density")
    ap.add_argument("--no-fingerprint", action="store_true")
    ap.add_argument("--fp-config", default="cfg2", choices=["cfg0", "cfg2"])
    ap.add_argument("--fp-samples", type=int, default=0, help="override the fingerprint trace length")
    ap.add_argument("--shard", default="tables", choices=["tables", "stations"],
                    help="N>1: one station's search table-sharded over the ranks (strong scaling, "
                         "north star) or one independent station per rank (weak scaling)")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def cuda_core_peaks():
    """Measured CUDA-core peaks (not in MEASURED_PEAKS.json):
    FP64 / FP32 FMA (GFLOP/s, 2 flops per FMA) and 64-bit min/max
    compare-selects (G/s), each the best of 3 timed launches of
    qs_peak_launch over 148 x 32 CTAs."""
    import ctypes
    import torch
    from paper_1803_09835_b200 import _native as nat
    blocks = 148 * 32
    scratch = torch.empty(blocks * 256 * 8, dtype=torch.uint8, device="cuda")
    out = {}
    for kind, name, iters, per_op in ((0, "fp64_gflops", 4096, 2.0), (1, "fp32_gflops", 16384, 2.0),
                                      (2, "u64_minmax_gops", 8192, 1.0)):
        ops = ctypes.c_double(0.0)
        best = None
        for rep in range(4):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            nat.call("qs_peak_launch", kind, blocks, iters, nat.ptr(scratch), ctypes.byref(ops),
                     nat.stream())
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            if rep and (best is None or ms < best):  # first launch: warm-up
                best = ms
        out[name] = ops.value * per_op / (best / 1e3) / 1e9
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def headline_config(args, world, tables_mode):
    occ = args.occ if args.occ > 0 else None
    return {"workload": "cfg1 (BASELINE.json configs[1])",
            ("n_total" if tables_mode else "n_per_gpu"): args.n,
            "d": 4096, "set_bits": 400, "tables": 100, "hash_funcs": 4, "min_matches": 5,
            "occurrence_threshold": occ,
            "occurrence_limit_matches": (occ * args.n if occ else None), "partitions": 1,
            "l2": f"inputs ({args.n * 400 * 4 / 1e9:.1f} GB bits) larger than L2 (126 MB); no flush",
            "parallelism": (f"table-sharded x{world} (round-robin tables, row-sharded Min-Max + "
                            "NCCL all-gather)" if tables_mode else f"station-sharded x{world}")}


# ----------------------------------------------------------- reference (CPU)

def reference_package():
    """The unmodified reference (baseline/_ref/quakescan), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "quakescan")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from quakescan import fingerprint as rfp
    from quakescan import lsh_search as rls
    from quakescan import minmax_hash as rmh
    from quakescan.ingest import TimeSeries as RTS
    return dict(fp=rfp, ls=rls, mh=rmh, TS=RTS)


_REF_BITS = {}


def cpu_search_step(n, occ_limit, threads, seed=0):
    """One bounded sample of the cfg1 workload through the reference CPU path:
    the reference's own signatures(workers=threads) and search_signatures
    (baseline/_ref), else the oracle port (oracle/)."""
    from paper_1803_09835_b200 import workloads
    key = (n, seed)
    if key not in _REF_BITS:
        _REF_BITS.clear()
        _REF_BITS[key] = workloads.cfg1_bits(n=n, seed=seed)[0]
    bits = _REF_BITS[key]
    occ = occ_limit / n if occ_limit else None
    ref = reference_package()
    if ref is not None:
        mapping = ref["mh"].gen_hash_mapping(4096, 100, 4, 0)
        t0 = time.perf_counter()
        sigs = ref["mh"].signatures(bits, mapping, workers=threads)
        t1 = time.perf_counter()
        trip, st = ref["ls"].search_signatures(
            sigs, ref["ls"].SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0,
                                         partitions=1, occurrence_threshold=occ))
        t2 = time.perf_counter()
        return dict(seconds=t2 - t0, sig_s=t1 - t0, search_s=t2 - t1, kind="reference",
                    triplets=int(trip.size), filtered=int(st.filtered_fingerprints),
                    backend=ref["mh"].BACKEND)
    from oracle import minmax as omm
    from oracle import search as osr
    values = omm.gen_mapping(4096, 100, 4, 0)
    t0 = time.perf_counter()
    sigs = omm.signatures_c(bits, values, 100, 2, threads=threads)
    t1 = time.perf_counter()
    trip, st = osr.search(sigs, tables=100, min_matches=5, partitions=1,
                          occurrence_threshold=occ, exclusion_windows=0)
    t2 = time.perf_counter()
    return dict(seconds=t2 - t0, sig_s=t1 - t0, search_s=t2 - t1, kind="port",
                triplets=int(trip.size), filtered=int(st["filtered_fingerprints"]), backend="c")


def fp_params(mod, p):
    return mod.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                                 freq_bins=p["freq_bins"], time_bins=p["time_bins"],
                                 top_k=p["top_k"], band_low_hz=p["band_low_hz"],
                                 band_high_hz=p["band_high_hz"],
                                 stft=mod.StftParams(p["frame_len_s"], p["hop_s"]))


def cpu_fingerprint_baseline(x_slice, threads):
    """The reference's fingerprint_series (baseline/_ref) on a host slice of
    the fingerprint workload; Msamples/s (per-sample cost is constant in the
    trace length, so the slice rate is the full-trace rate)."""
    from paper_1803_09835_b200 import workloads
    ref = reference_package()
    if ref is None:
        return None
    params = fp_params(ref["fp"], workloads.CFG0_PARAMS)
    ts = ref["TS"]("ST0", "HHZ", workloads.SR_HZ, 0.0, x_slice)
    t0 = time.perf_counter()
    fps, _ = ref["fp"].fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
    s = time.perf_counter() - t0
    return {"value": x_slice.size / s / 1e6, "unit": "Msamples/s", "cores": threads,
            "kind": "reference", "seconds": s,
            "sample": (f"reference quakescan.fingerprint.fingerprint_series (baseline/_ref) on "
                       f"{x_slice.size} samples ({x_slice.size / 8.64e6:.2f} days) of the same "
                       f"trace, mad_rate 0.1; numpy FFT/median/partition single-threaded, the "
                       f"einsum's GEMM on OpenBLAS threads ({threads} cores visible)"),
            "n_fingerprints": int(fps.bits.shape[0])}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    occ_limit = args.occ * args.n if args.occ > 0 else None
    for _ in range(args.warmup):   # warm caches/imports on a small sample
        cpu_search_step(10_000, occ_limit, threads, seed=99)
    times, kinds, sig_s, search_s = [], set(), [], []
    for i in range(args.steps):
        r = cpu_search_step(args.ref_n, occ_limit, threads, seed=0)
        times.append(r["seconds"])
        sig_s.append(r["sig_s"])
        search_s.append(r["search_s"])
        kinds.add(r["kind"])
    t = float(np.mean(times))
    value = args.ref_n / t
    kind = "reference" if kinds == {"reference"} else "port"
    sample = (f"cfg1 generator at N={args.ref_n} rows (same densities and the same limit-"
              f"{occ_limit:.0f} occurrence filter as the N={args.n} headline), through the "
              f"reference's own quakescan.minmax_hash.signatures(workers={threads}) "
              f"({np.mean(sig_s):.2f} s) and quakescan.lsh_search.search_signatures "
              f"(single-threaded numpy, {np.mean(search_s):.2f} s); search cost grows ~N^2, so "
              f"fp/s at N={args.n} is far lower (profiles/r02_cpu_scaling.log)")
    line = {"metric": METRIC, "value": value, "unit": "fingerprints/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": headline_config(args, 1, False),
            "cpu_baseline": {"value": value, "unit": "fingerprints/s", "cores": threads,
                             "kind": kind, "sample": sample, "sample_n": args.ref_n},
            "e2e": {"value": value, "unit": "fingerprints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if not args.no_fingerprint:
        from paper_1803_09835_b200 import workloads
        x, _ = workloads.cfg0_trace()  # one day of the fingerprint workload's geometry
        line["fingerprint"] = cpu_fingerprint_baseline(x, threads)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- fingerprinting

def fingerprint_bench(args, steps, device, threads, cpu=True):
    """Second BASELINE metric: fingerprint Msamples/s = samples / time of
    fingerprint_series (STFT + MAD sample pass + main pass) on a
    device-resident trace; e2e from a host float32 trace (TimeSeries coerces
    it to float64 like the reference; H2D of the float64 samples, D2H of the
    bits, both inside the timed call)."""
    import torch
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.ingest import TimeSeries
    torch.cuda.empty_cache()
    if args.fp_config == "cfg2":
        n = args.fp_samples or 795_000_000
        xd, _ = workloads.cfg2_trace_torch(n_samples=n, seed=2, device=device)
        workload = ("cfg2 (BASELINE.json configs[2]): 7.95e8 samples at 100 Hz of seeded 1/f "
                    "noise (torch RNG, rfft-shaped) + 500 planted chirp repeats; window 10 s / lag "
                    "1 s, 32x64 images, top-K 200, MAD rate 0.1")
    else:
        n = args.fp_samples or 8_640_000
        x, _ = workloads.cfg0_trace(n_samples=n, seed=0)
        xd = torch.from_numpy(x).to(device)
        workload = ("cfg0 (BASELINE.json configs[0]): 1 day at 100 Hz, 5 chirp templates x 20, "
                    "window 10 s / lag 1 s, 32x64 images, top-K 200, MAD rate 0.1")
    params = fp_params(fp, workloads.CFG0_PARAMS)
    ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, xd)
    fps, _ = fp.fingerprint_series(ts, params, mad_rate=0.1)
    del fps
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index or 0) as fclk:  # the FP64-heavy chain has its own clocks line
        a.record()
        for _ in range(steps):
            fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    n_fp = int(fps.bits.shape[0])
    del fps
    # e2e: a host float32 trace through the public call (host bits out)
    x_host = xd.cpu().numpy()
    del xd, ts
    torch.cuda.empty_cache()
    tsh = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x_host)  # coerced to float64 (reference)
    w0, _ = fp.fingerprint_series(tsh, params, mad_rate=0.1)
    del w0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fph, _ = fp.fingerprint_series(tsh, params, mad_rate=0.1)
    e2e_s = time.perf_counter() - t0
    d2h = int(fph.bits.nbytes)
    del fph, tsh
    out = {"metric": "fingerprint Msamples/s", "value": n / ms / 1e3, "unit": "Msamples/s",
           "ms_per_step": ms, "steps": steps, "n_samples": n, "n_fingerprints": n_fp,
           "workload": workload, "dtype": "f64 (STFT/resize/Haar/normalise), f32 stores",
           "clocks": fclk.summary(),
           "e2e": {"value": n / e2e_s / 1e6, "unit": "Msamples/s", "seconds": e2e_s,
                   "h2d_bytes_per_step": int(n * 4), "d2h_bytes_per_step": d2h,
                   "host_memory": ("pageable float64 (TimeSeries coerces the float32 recording like "
                                   "the reference); every sample is exactly a float32, so the staging "
                                   "pass narrows it (qs_host_pack_f32) and 4 bytes per sample cross "
                                   "PCIe; the chain widens them exactly"),
                   "path": "fingerprint.fingerprint_series(TimeSeries(host float32 -> float64))"}}
    # the step before fingerprinting in the reference CLI (cli.py:152-153): zero-phase
    # band-pass of a device-resident day
    from paper_1803_09835_b200.ingest import BandpassSpec, bandpass
    day = torch.from_numpy(x_host[:8_640_000]).to(device)
    tsd = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, day)
    spec = BandpassSpec(4.0, 10.0, 4)
    bandpass(tsd, spec)
    torch.cuda.synchronize()
    a.record()
    for _ in range(max(1, steps)):
        bandpass(tsd, spec)
    b.record()
    torch.cuda.synchronize()
    bp_ms = a.elapsed_time(b) / max(1, steps)
    out["bandpass"] = {"value": day.numel() / bp_ms / 1e3, "unit": "Msamples/s", "ms": bp_ms,
                       "n_samples": day.numel(),
                       "filter": "Butterworth order 4, 4-10 Hz, forward-backward (sosfiltfilt)"}
    if cpu:
        out["cpu_baseline"] = cpu_fingerprint_baseline(x_host[:8_640_000], threads)
    return out


# ---------------------------------------------------------------------- ours

def pair_roofline(ds, stages, n_trip, m, t, hbm, peak_kind, filt):
    """SURVEY §8d accounting of the pair stage, per pass: 16 B per candidate
    (pair, table) hit + 4 B per member of the walked buckets, + 20 B per
    emitted triplet (charged to the emitting pass).  MATCHED walks the buckets
    of tables <= t - m; DISTINCT walks the compacted buckets (excluded members
    removed); FULL walks every bucket."""
    import torch
    bs = ds.bsize[: ds.nb].to(torch.int64)
    bt = ds.btab[: ds.nb]  # global table ids (a sharded rank's listing maps them)
    passes = {}

    def acc(sizes):
        sizes = sizes.to(torch.int64)
        return int((sizes * (sizes - 1) // 2).sum().item()), int(sizes.sum().item())

    skipped = None
    if filt:
        h1, m1 = acc(bs[bt <= t - m])
        sk = getattr(ds, "core_skipped", None)
        if sk is not None:  # pairs of two proven-core fingerprints are never compared
            skipped = int(sk.item())
            h1 -= skipped
        cs = getattr(ds, "compact_sizes", None)
        h2, m2 = acc(cs) if cs is not None else acc(bs)
        passes["matched"] = (h1, m1, 20 * n_trip, stages.get("pairs_matched", 0.0))
        passes["distinct"] = (h2, m2, 0, stages.get("pairs_distinct", 0.0))
    else:
        h, mm = acc(bs)
        passes["full"] = (h, mm, 20 * n_trip, stages.get("pairs_full", 0.0))
    per = {}
    tot_b, tot_ms = 0, 0.0
    for name, (h, mm, tb, ms) in passes.items():
        nbytes = 16 * h + 4 * mm + tb
        tot_b += nbytes
        tot_ms += ms
        gbs = nbytes / (ms / 1e3) / 1e9 if ms else None
        per[name] = {"hits": h, "members": mm, "algorithmic_bytes": nbytes, "ms": ms,
                     "achieved_gbs": gbs, "frac": gbs / hbm if gbs else None}
        if name == "matched" and skipped is not None:
            per[name]["core_core_pairs_skipped"] = skipped
            per[name]["hits_note"] = ("hits = pairs compared: the buckets' pairs minus the "
                                      "core-core pairs the core skip leaves out")
    achieved = tot_b / (tot_ms / 1e3) / 1e9 if tot_ms else 0.0
    return {"bound": "hbm", "kernel": "k_pairs_pc (first-colliding-table pair enumeration), all passes",
            "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / hbm, "algorithmic_bytes": tot_b, "ms": tot_ms, "passes": per,
            "accounting": "16 B/hit + 4 B/member of walked buckets + 20 B/triplet (SURVEY 8d)",
            "traffic": _ncu_traffic(int(ds.n) if hasattr(ds, "n") else None, filt)}


def _ncu_traffic(n, filt):
    """DRAM bytes (read + write) of every pair-stage launch of one step, from the
    committed ncu capture (profiles/traffic.json, written by tools/launch_summary.py
    from a run of tools/one_search.py at the same n with the filter on); None when
    no capture matches this run."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    if not filt or "pair_stage_dram_bytes_total" not in t or (n is not None and t.get("n") != n):
        return None
    return t["pair_stage_dram_bytes_total"]


def _stage_avg(timed):
    stages = {}
    for evs, ev in timed:
        for (k, ea), (_, eb) in zip(evs[:-1], evs[1:]):
            stages[k] = stages.get(k, 0.0) + ea.elapsed_time(eb) / len(timed)
        stages["minhash"] = stages.get("minhash", 0.0) + ev[0].elapsed_time(ev[1]) / len(timed)
        stages["mapping"] = stages.get("mapping", 0.0) + ev[2].elapsed_time(ev[0]) / len(timed)
    return stages


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    # QS_BENCH_BACKEND=gloo lets a 1-GPU box run the N>1 control flow (ranks
    # share the device; no kernel waits on another rank's kernel)
    backend = os.environ.get("QS_BENCH_BACKEND", "nccl")
    ndev = max(1, torch.cuda.device_count())
    if world > 1 and backend == "nccl" and ndev < world:
        raise SystemExit(f"bench.py --gpus {world}: only {ndev} CUDA device(s) visible")
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    dev = torch.device(f"cuda:{local}")
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.fingerprint import FingerprintSet

    n = args.n
    occ = args.occ if args.occ > 0 else None
    tables_mode = world > 1 and args.shard == "tables"
    threads = len(os.sched_getaffinity(0))
    # tables mode: every rank generates the same station (seed 1) and keeps only
    # its block of rows; stations mode: rank r searches its own station
    bits, _ = workloads.cfg1_bits_torch(n=n, seed=1 if tables_mode else 1 + rank, device=dev,
                                        group_frac=args.group_frac)
    comm = None
    if tables_mode:
        from paper_1803_09835_b200 import sharded as sh
        comm = sh.TorchComm()
        a, b, s_rows = sh.row_block(n, world, rank)
        blk = bits[a:b]
        if b - a < s_rows:
            blk = torch.cat([blk, blk[:1].expand(s_rows - (b - a), -1)])
        bits = blk.contiguous()
        host_rows = (a, b)
    torch.cuda.synchronize()

    def make_cfg(o):
        return ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0, partitions=1,
                               occurrence_threshold=o)

    last = {}

    def step(cfg, timing=False):
        # the hash mapping + probe plan are part of the step (search_fingerprints
        # with mapping=None, lsh_search.py:314-333)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timing else None
        if ev:
            ev[2].record()
        mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
        mapping.device_plan()
        if tables_mode:
            trip, st, ds = sh.search_bits_sharded(bits, n, cfg, mapping, 0, comm=comm, timing=timing)
            ev = None
        else:
            if ev:
                ev[0].record()
            keys, rkeys, tags, bad = ls.signatures_for_search(bits, mapping)
            if ev:
                ev[1].record()
            trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0, timing=timing)
        last.update(trip=trip, stats=st, ds=ds, sig_ev=ev)
        return ds

    def timed_loop(cfg, steps, warm):
        for _ in range(warm):
            step(cfg)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        launches, timed = 0, []
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            start.record()
            for _ in range(steps):
                ds = step(cfg, timing=not tables_mode)
                launches += ds.launches + 3  # + mapping kernel, plan kernel, signature kernel
                if not tables_mode:
                    timed.append((list(ds.events), last["sig_ev"]))
            end.record()
            torch.cuda.synchronize()
        ms = start.elapsed_time(end) / steps
        if world > 1:
            tmax = torch.tensor([ms], device=dev)
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            ms = float(tmax.item())
        return ms, launches, timed, clk.summary()

    cfg = make_cfg(occ)
    ms, launches, timed, clocks = timed_loop(cfg, args.steps, max(3, args.warmup))
    value = (n if tables_mode else world * n) / (ms / 1e3)
    hbm, peak_kind = peaks()

    if tables_mode:
        # per-stage split from one more (event-timed) search after the timed region
        st = last["stats"]
        step(cfg, timing=True)
        torch.cuda.synchronize()
        ds = last["ds"]
        stages = ds.stage_times_ms()
    else:
        stages = _stage_avg(timed)
        ds, st = last["ds"], last["stats"]
    roof = pair_roofline(ds, stages, st.emitted_triplets if rank == 0 else 0, 5, 100, hbm,
                         peak_kind, occ is not None)
    kt = len(ds.table_ids) if ds.table_ids is not None else 100
    other = {}
    if stages.get("buckets"):
        sms = stages["buckets"] + stages.get("list", 0.0)
        nbytes = 12 * n * kt
        other["buckets"] = {"scope": "bucket build + listing", "algorithmic_bytes": nbytes,
                            "ms": sms, "achieved_gbs": nbytes / (sms / 1e3) / 1e9,
                            "frac": nbytes / (sms / 1e3) / 1e9 / hbm}
    if stages.get("minhash"):
        nbytes = (4 * 400 + 8 * 100) * n
        other["minhash"] = {"algorithmic_bytes": nbytes, "ms": stages["minhash"],
                            "achieved_gbs": nbytes / (stages["minhash"] / 1e3) / 1e9,
                            "frac": nbytes / (stages["minhash"] / 1e3) / 1e9 / hbm}
    roof["other_stages"] = other
    emitted, filtered, distinct = st.emitted_triplets, st.filtered_fingerprints, st.distinct_pairs
    del last["trip"], last["ds"], ds
    torch.cuda.empty_cache()

    # the reference's default: no occurrence filter (FULL mode)
    full = None
    if args.full_steps > 0 and not tables_mode:
        fms, _, ftimed, _ = timed_loop(make_cfg(None), args.full_steps, 1)
        fstages = _stage_avg(ftimed)
        froof = pair_roofline(last["ds"], fstages, last["stats"].emitted_triplets, 5, 100, hbm,
                              peak_kind, False)
        full = {"value": n / (fms / 1e3), "unit": "fingerprints/s", "ms_per_step": fms,
                "steps": args.full_steps, "occurrence_threshold": None,
                "emitted_triplets": last["stats"].emitted_triplets,
                "distinct_pairs": last["stats"].distinct_pairs, "stages_ms": fstages,
                "roofline": {k: froof[k] for k in ("achieved", "frac", "algorithmic_bytes", "ms",
                                                     "passes")}}
        del last["trip"], last["ds"]
        torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        # the step's inputs in PINNED host memory (the bench contract): the library
        # detects page-locked arrays and copies them by DMA from where they lie; the
        # same call with a pageable numpy array (staged through pinned buffers,
        # narrowed to 12-bit fields on the way) is reported as `pageable`
        src = bits[: host_rows[1] - host_rows[0]] if tables_mode else bits
        pinned_t = torch.empty(tuple(src.shape), dtype=torch.int32, pin_memory=True)
        pinned_t.copy_(src)
        torch.cuda.synchronize()
        cfg_e = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0,
                                occurrence_threshold=occ, near_repeat_exclusion_s=0.0)

        def time_e2e(host_bits):
            rows = host_bits.shape[0]
            fps = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                                 indices=np.arange(rows, dtype=np.uint64),
                                 epochs=np.arange(rows, dtype=np.float64), bits=host_bits)

            def e2e_call():
                if tables_mode:
                    return sh.search_fingerprints_sharded(fps, n, cfg_e)
                return ls.search_fingerprints(fps, cfg_e)  # mapping generated inside, like the reference

            e2e_call()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            out_bytes = 0
            for _ in range(args.e2e_steps):
                rec, est, _ = e2e_call()
                out_bytes = rec.nbytes
            torch.cuda.synchronize()
            e_s = (time.perf_counter() - t0) / args.e2e_steps
            if world > 1:
                et = torch.tensor([e_s], dtype=torch.float64, device=dev)
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
                e_s = float(et.item())
            return e_s, out_bytes, int(ls.LAST_H2D_BYTES)

        e_units = n if tables_mode else world * n
        e_s, out_bytes, h2d = time_e2e(pinned_t.numpy().view(np.uint32))
        e2e = {"value": e_units / e_s, "unit": "fingerprints/s",
               "h2d_bytes_per_step": h2d or int(e_units * 400 * 4),
               "d2h_bytes_per_step": int(out_bytes), "input_bytes_per_step": int(e_units * 400 * 4),
               "seconds_per_step": e_s,
               "host_memory": ("pinned: DMA from the caller's array, a share of every chunk's rows "
                               "(balanced during the call against the measured pack and copy "
                               "rates, narrowed_share) narrowed to 12-bit fields (d = 4096) by the "
                               "host cores on the way (h2d_bytes_per_step = the bytes that crossed "
                               "PCIe)"),
               "narrowed_share": round(float(ls.LAST_H2D_SPLIT), 3),
               "path": ("sharded.search_fingerprints_sharded (host row block per rank)" if tables_mode
                        else "lsh_search.search_fingerprints(FingerprintSet with host numpy bits)")}
        if not tables_mode:
            pageable = np.array(pinned_t.numpy().view(np.uint32))  # an ordinary numpy array
            del pinned_t
            p_s, _, ph2d = time_e2e(pageable)
            e2e["pageable"] = {"value": e_units / p_s, "seconds_per_step": p_s,
                               "h2d_bytes_per_step": ph2d,
                               "host_memory": ("pageable numpy array: staged through two pinned "
                                               "buffers by a thread pool, narrowed to 12-bit fields "
                                               "on the way (qs_host_pack_u12), widened on the device")}
            del pageable
        else:
            del pinned_t
    del bits
    torch.cuda.empty_cache()

    cpu, same_n = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        occ_limit = occ * n if occ else None
        r = cpu_search_step(args.ref_n, occ_limit, threads, seed=0)
        cpu = {"value": args.ref_n / r["seconds"], "unit": "fingerprints/s", "cores": threads,
               "kind": r["kind"], "sample_n": args.ref_n,
               "sample": (f"cfg1 generator at N={args.ref_n} rows, limit-{occ_limit:.0f} filter: "
                          f"the reference's own signatures (backend {r['backend']}, "
                          f"workers={threads}, {r['sig_s']:.2f} s) + search_signatures "
                          f"(single-threaded numpy, {r['search_s']:.2f} s); the search grows "
                          f"~N^2, so at N={n} its fp/s is far lower")}
        # the GPU on the very same sample (host bits of the same generator call):
        # a measured like-for-like ratio against cpu_baseline
        sb = _REF_BITS[(args.ref_n, 0)]
        fps_s = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                               indices=np.arange(args.ref_n, dtype=np.uint64),
                               epochs=np.arange(args.ref_n, dtype=np.float64), bits=sb)
        cfg_s = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0,
                                occurrence_threshold=(occ_limit / args.ref_n if occ else None),
                                near_repeat_exclusion_s=0.0)
        bd = torch.from_numpy(sb.view(np.int32)).to(dev)
        fps_d = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                               indices=fps_s.indices, epochs=fps_s.epochs, bits=bd)
        for _ in range(3):
            ls.search_fingerprints(fps_d, cfg_s)
        torch.cuda.synchronize()
        a_ev = torch.cuda.Event(enable_timing=True)
        b_ev = torch.cuda.Event(enable_timing=True)
        a_ev.record()
        for _ in range(5):
            ls.search_fingerprints(fps_d, cfg_s)
        b_ev.record()
        torch.cuda.synchronize()
        dms = a_ev.elapsed_time(b_ev) / 5
        t0 = time.perf_counter()
        for _ in range(3):
            ls.search_fingerprints(fps_s, cfg_s)
        es = (time.perf_counter() - t0) / 3
        same_n = {"n": args.ref_n, "value": args.ref_n / (dms / 1e3), "ms_per_step": dms,
                  "e2e": {"value": args.ref_n / es, "seconds_per_step": es},
                  "unit": "fingerprints/s",
                  "vs_cpu_baseline": (args.ref_n / (dms / 1e3)) / cpu["value"],
                  "e2e_vs_cpu_baseline": (args.ref_n / es) / cpu["value"]}
        del bd

    fpb = None
    if rank == 0 and not args.no_fingerprint:
        fpb = fingerprint_bench(args, max(1, min(args.steps, 3)), dev, threads,
                                cpu=not args.no_cpu_baseline)
        # the chain against the measured FP64 peak (F_win = 74,100 flops
        # per window + the MAD pass's rate x 68,000)
        cpk = cuda_core_peaks()
        fp_flops = fpb["n_fingerprints"] * (74_100 + 0.1 * 68_000)
        fp_gf = fp_flops / (fpb["ms_per_step"] / 1e3) / 1e9
        fpb["roofline"] = {"bound": "fp64", "achieved": fp_gf, "peak": cpk["fp64_gflops"],
                           "peak_kind": "measured (qs_peak_launch, FP64 FMA)", "unit": "GFLOP/s",
                           "frac": fp_gf / cpk["fp64_gflops"], "flops_per_call": fp_flops}
        fpb["cuda_core_peaks"] = cpk

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "fingerprints/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong" if tables_mode else "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": headline_config(args, world, tables_mode),
                "stages_ms": stages, "emitted_triplets": emitted,
                "filtered_fingerprints": filtered, "distinct_pairs": distinct,
                "roofline": roof, "cpu_baseline": cpu, "same_n": same_n, "full_mode": full,
                "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "fingerprint": fpb}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn_entry(rank, args, port):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(args.gpus),
                      LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    run_ours(args)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1:
        # communicator init lines (rank count) on stderr for the scaling record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if "WORLD_SIZE" not in os.environ:
            import torch.multiprocessing as mp
            mp.spawn(_spawn_entry, args=(args, _free_port()), nprocs=args.gpus, join=True)
            return
    run_ours(args)


if __name__ == "__main__":
    main()
