"""Benchmark of the hot path (BASELINE.json metric) — one JSON line on rank 0.

Workload (BASELINE.json configs[1]): N = 8e6 sparse 4096-bit
fingerprints with exactly 400 set bits, 1e5 planted near-duplicate pairs,
2e4 noise groups x 200 rows (Jaccard 0.7 to the group template); b=100
tables, r=4 (k=4 Min-Max hash functions), m=5, occurrence filter 1.5e-5
(limit 120 matches, the value that makes the filter fire on this generator,
SURVEY.md §8d).  A step = one pass of the hot path over that batch:
Min-Max signatures (fused with the table-major key/tag layout) -> per-table
bucket construction -> first-colliding-table pair enumeration with exact
collision counts -> occurrence filter (+ second enumeration) -> bucket stats
-> (dt, idx1)-sorted triplets.  Inputs are resident in HBM (12.8 GB, larger
than L2) when the timed region starts.

Multi-GPU (torchrun): every rank searches its own station-sized cfg1 batch
(seed = rank), no data-path collective ("scaling": "weak"); the reported
time is the max over ranks.

`--impl reference` times the reference CPU path on the host cores: the
reference's own compiled Min-Max kernel (oracle/_ref/_sigcore, all cores) and
the numpy port of its search (single-threaded, as the reference), on a
bounded sample of the same workload (N = --ref-n rows).
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fingerprints", dest="n", type=int, default=8_000_000)
    ap.add_argument("--occ", type=float, default=1.5e-5, help="occurrence threshold (<=0: off)")
    ap.add_argument("--ref-n", type=int, default=100_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--group-frac", type=float, default=1 / 400, help="noise-group density (design experiments)")
    ap.add_argument("--no-fingerprint", action="store_true")
    ap.add_argument("--shard", default="tables", choices=["tables", "stations"],
                    help="N>1: one station's search table-sharded over the ranks (strong scaling, "
                         "north star) or one independent station per rank (weak scaling)")
    ap.add_argument("--fp-samples", type=int, default=8_640_000)
    return ap.parse_args()


TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")


def measured_traffic(n):
    """DRAM bytes (read + write) of the pair stage per step, from the committed
    `ncu --set full` capture summary (profiles/traffic.json), or None."""
    try:
        with open(TRAFFIC_PATH) as f:
            t = json.load(f)
        if int(t["n"]) != n:
            return None
        return float(sum(t["pair_stage_dram_bytes"].values())), t["source"]
    except Exception:
        return None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


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


# ---------------------------------------------------------------- reference arm

def cpu_reference_step(n, occ_limit, threads, seed=0):
    """One bounded sample of the cfg1 workload through the reference CPU path."""
    from oracle import minmax as omm
    from oracle import search as osr
    from paper_1803_09835_b200 import workloads
    bits, _ = workloads.cfg1_bits(n=n, seed=seed)
    values = omm.gen_mapping(4096, 100, 4, 0)
    t0 = time.perf_counter()
    sigs = omm.signatures_reference_kernel(bits, values, 100, 2, threads=threads)
    kind = "reference"
    if sigs is None:
        sigs = omm.signatures_c(bits, values, 100, 2, threads=threads)
        kind = "port"
    t1 = time.perf_counter()
    occ = occ_limit / n if occ_limit else None
    trip, st = osr.search(sigs, tables=100, min_matches=5, partitions=1,
                          occurrence_threshold=occ, exclusion_windows=0)
    t2 = time.perf_counter()
    return dict(seconds=t2 - t0, sig_s=t1 - t0, search_s=t2 - t1, kind=kind,
                triplets=int(trip.size), filtered=st["filtered_fingerprints"])


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    occ_limit = args.occ * args.n if args.occ > 0 else None
    for _ in range(args.warmup):
        cpu_reference_step(args.ref_n, occ_limit, threads)
    times, kinds = [], set()
    for i in range(args.steps):
        r = cpu_reference_step(args.ref_n, occ_limit, threads, seed=i)
        times.append(r["seconds"])
        kinds.add(r["kind"])
    t = float(np.mean(times))
    value = args.ref_n / t
    kind = "reference" if kinds == {"reference"} else "port"
    sample = (f"cfg1 generator at N={args.ref_n} rows (same densities as N=8e6; search is "
              f"O(N^2) so fp/s at 8e6 is far lower), signatures by the reference's compiled "
              f"_sigcore on {threads} threads + numpy port of lsh_search.search_signatures "
              f"(single-threaded like the reference), occurrence limit {occ_limit}")
    line = {"metric": "LSH search fingerprints/sec (MinHash+bucket+pair-count)", "value": value,
            "unit": "fingerprints/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": "cfg1 (BASELINE.json configs[1]) sample",
                                            "n": args.ref_n, "tables": 100, "hash_funcs": 4,
                                            "min_matches": 5},
            "cpu_baseline": {"value": value, "unit": "fingerprints/s", "cores": threads,
                             "kind": kind, "sample": sample,
                             "extrapolated_to_n": {"n": 8_000_000,
                                                   "value": value * args.ref_n / 8_000_000,
                                                   "law": "search time ~ N^2 (SURVEY 6.2)"}},
            "e2e": {"value": value, "unit": "fingerprints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- fingerprinting

def fingerprint_bench(n_samples, steps, device):
    """Second BASELINE metric: fingerprint Msamples/s (fingerprint_series on a
    device-resident cfg0-style trace: STFT + MAD sample + main pass)."""
    import torch
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200 import workloads
    from paper_1803_09835_b200.ingest import TimeSeries
    # a separate workload: release the search's cached device blocks first so its
    # allocations do not run into the caching allocator's free-and-retry path
    torch.cuda.empty_cache()
    x, _ = workloads.cfg0_trace(n_samples=n_samples, seed=0)
    xd = torch.from_numpy(x).to(device)
    p = workloads.CFG0_PARAMS
    params = fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                                  freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
                                  band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
                                  stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))
    ts = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, xd)
    fp.fingerprint_series(ts, params, mad_rate=0.1)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    # e2e: host float32 numpy trace in, host bits out
    tsh = TimeSeries("ST0", "HHZ", workloads.SR_HZ, 0.0, x)
    # warm-up to steady state: two calls with the first result still held (a
    # caller keeps its last result alive, so the pinned result buffers rotate)
    w0, _ = fp.fingerprint_series(tsh, params, mad_rate=0.1)
    w1, _ = fp.fingerprint_series(tsh, params, mad_rate=0.1)
    del w0, w1
    t0 = time.perf_counter()
    for _ in range(steps):
        fph, _ = fp.fingerprint_series(tsh, params, mad_rate=0.1)
    e2e_s = (time.perf_counter() - t0) / steps
    # the step before fingerprinting in the reference CLI (cli.py:152-153):
    # zero-phase band-pass of the device-resident trace
    from paper_1803_09835_b200.ingest import BandpassSpec, bandpass
    spec = BandpassSpec(p["band_low_hz"], p["band_high_hz"], 4)
    bandpass(ts, spec)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        bandpass(ts, spec)
    b.record()
    torch.cuda.synchronize()
    bp_ms = a.elapsed_time(b) / steps
    return {"metric": "fingerprint Msamples/s", "value": n_samples / ms / 1e3, "unit": "Msamples/s",
            "bandpass": {"value": n_samples / bp_ms / 1e3, "unit": "Msamples/s", "ms": bp_ms,
                         "filter": "Butterworth order 4, 4-10 Hz, forward-backward (sosfiltfilt)"},
            "ms_per_step": ms, "n_samples": n_samples, "n_fingerprints": int(len(fps)),
            "workload": "cfg0 (BASELINE.json configs[0]): 1 day at 100 Hz, 5 chirp templates x 20, "
                        "window 10 s / lag 1 s, 32x64 images, top-K 200, MAD rate 0.1",
            "e2e": {"value": n_samples / e2e_s / 1e6, "unit": "Msamples/s",
                    "h2d_bytes_per_step": int(x.nbytes), "d2h_bytes_per_step": int(fph.bits.nbytes)}}


# ---------------------------------------------------------------------- ours

def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # QS_BENCH_BACKEND=gloo lets a 1-GPU box run the N>1 control flow (ranks
    # share the device; no kernel waits on another rank's kernel)
    backend = os.environ.get("QS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
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
    # tables mode: every rank generates the same station (seed 1) and keeps only
    # its block of rows; stations mode: rank r searches its own station
    bits, _ = workloads.cfg1_bits_torch(n=n, seed=1 if tables_mode else 1 + rank, device=dev,
                                        group_frac=args.group_frac)
    mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
    mapping.device_plan()
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0, partitions=1,
                          occurrence_threshold=occ)
    comm = None
    if tables_mode:
        from paper_1803_09835_b200 import sharded as sh
        comm = sh.TorchComm()
        a, b, s_rows = sh.row_block(n, world, rank)
        blk = bits[a:b]
        if b - a < s_rows:
            blk = torch.cat([blk, blk[:1].expand(s_rows - (b - a), -1)])
        blk = blk.contiguous()
        host_rows = (a, b)
        del bits
        bits = blk
    torch.cuda.synchronize()

    last = {}

    def step(timing=False):
        if tables_mode:
            trip, st, ds = sh.search_bits_sharded(bits, n, cfg, mapping, 0, comm=comm, timing=timing)
            ev = None
        else:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timing else None
            if ev:
                ev[0].record()
            keys, rkeys, tags, bad = ls.signatures_for_search(bits, mapping)
            if ev:
                ev[1].record()
            trip, st, ds = ls.run_search(keys, rkeys, tags, n, 100, cfg, 0, timing=timing)
        last.update(trip=trip, stats=st, ds=ds, sig_ev=ev)
        return ds

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    launches = 0
    timed = []  # 1 GPU: per-stage CUDA events recorded inside the timed steps
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            ds = step(timing=not tables_mode)
            launches += ds.launches + 1
            if not tables_mode:  # events only: the step's buffers are released
                timed.append((list(ds.events), last["sig_ev"]))
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        tmax = torch.tensor([ms], device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        ms = float(tmax.item())
    value = (n if tables_mode else world * n) / (ms / 1e3)

    # per-stage split + roofline of the dominant kernel (pair enumeration)
    if tables_mode:
        # N > 1: one extra timed-stage search after the timed region
        sig_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        sig_ev[0].record()
        rkeys, tags, bad = sh.gather_search_layout(bits, n, mapping, comm)
        sig_ev[1].record()
        own = sh.shard_tables(100, world, rank)
        ds = ls.DeviceSearch(sh.own_keys(rkeys, own), rkeys, tags, n, 100, timing=True, tables=own)
        trip, st, ds = sh.run_search_sharded(ds, comm, n, 100, cfg, 0)
        torch.cuda.synchronize()
        stages = ds.stage_times_ms()
        stages["minhash+gather"] = sig_ev[0].elapsed_time(sig_ev[1])
    else:
        # 1 GPU: the stages of the K timed steps themselves (events on the
        # launching stream), averaged
        stages = {}
        for evs, ev in timed:
            for (k, ea), (_, eb) in zip(evs[:-1], evs[1:]):
                stages[k] = stages.get(k, 0.0) + ea.elapsed_time(eb) / len(timed)
            stages["minhash"] = stages.get("minhash", 0.0) + ev[0].elapsed_time(ev[1]) / len(timed)
        ds, st = last["ds"], last["stats"]
    bs = ds.bsize[: ds.nb].to(torch.int64)
    hits = int((bs * (bs - 1) // 2).sum().item())
    m2 = int(bs.sum().item())
    passes = 2 if occ is not None else 1
    pair_bytes = passes * (16 * hits + 4 * m2) + 20 * (st.emitted_triplets if not tables_mode else 0)
    pair_ms = sum(v for k, v in stages.items() if k.startswith("pairs"))
    hbm, peak_kind = peaks()
    achieved = pair_bytes / (pair_ms / 1e3) / 1e9
    traffic = measured_traffic(n) if not tables_mode else None
    roof = {"bound": "hbm", "kernel": "k_pairs_pc (first-colliding-table pair enumeration)",
            "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic[0] if traffic else None,
            "traffic_source": traffic[1] if traffic else None,
            "scope": ("all pair-enumeration launches of one step (matched + distinct pass)"
                      + (f", rank 0's {len(ds.table_ids) if ds.table_ids is not None else 100}"
                         " tables" if tables_mode else "")),
            "algorithmic_bytes": pair_bytes, "hits": hits, "passes": passes,
            "ms": pair_ms}
    # the other stages against the same accounting, for transparency
    kt = len(ds.table_ids) if ds.table_ids is not None else 100
    stage_roofs = {}
    for name, nbytes in [("buckets", 12 * n * kt), ("minhash" + ("+gather" if tables_mode else ""),
                                                     (4 * 400 + 8 * 100) * (n if not tables_mode
                                                                            else -(-n // world)))]:
        if stages.get(name):
            sms = stages[name] + (stages.get("list", 0.0) if name == "buckets" else 0.0)
            gbs = nbytes / (sms / 1e3) / 1e9
            stage_roofs[name] = {"algorithmic_bytes": nbytes, "ms": sms,
                                 "achieved_gbs": gbs, "frac": gbs / hbm}
            if name == "buckets":
                # bytes the build really moves per (fp, table): 4 radix histogram
                # reads (4 x 8) + scatter passes (8 + 12 | 3 x (12 + 12)) + flag
                # sweep (8 + 1) + listing (~2): DESIGN.md section 5.2
                moved = 143 * n * kt
                stage_roofs[name].update({"scope": "bucket build + listing",
                                          "moved_bytes": moved,
                                          "moved_gbs": moved / (sms / 1e3) / 1e9,
                                          "moved_frac": moved / (sms / 1e3) / 1e9 / hbm})
    roof["other_stages"] = stage_roofs

    e2e = None
    if not args.no_e2e:
        if tables_mode:
            a, b = host_rows
            host_bits = bits[: b - a].cpu().numpy().view(np.uint32)
        else:
            host_bits = bits.cpu().numpy().view(np.uint32)
        rows = host_bits.shape[0]
        fps = FingerprintSet(d=4096, top_k=400, window_len_s=1.0, window_lag_s=1.0,
                             indices=np.arange(rows, dtype=np.uint64),
                             epochs=np.arange(rows, dtype=np.float64), bits=host_bits)
        cfg_e = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0,
                                occurrence_threshold=occ, near_repeat_exclusion_s=0.0)

        def e2e_call():
            if tables_mode:
                return sh.search_fingerprints_sharded(fps, n, cfg_e, mapping=mapping)
            return ls.search_fingerprints(fps, cfg_e, mapping=mapping)

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
        e_units = n if tables_mode else world * n
        e2e = {"value": e_units / e_s, "unit": "fingerprints/s",
               "h2d_bytes_per_step": int(e_units * 400 * 4), "d2h_bytes_per_step": int(out_bytes),
               "seconds_per_step": e_s,
               "path": ("sharded.search_fingerprints_sharded (host row block per rank)" if tables_mode
                        else "lsh_search.search_fingerprints(FingerprintSet with host numpy bits)")}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        r = cpu_reference_step(args.ref_n, args.occ * n if occ else None, threads)
        cpu = {"value": args.ref_n / r["seconds"], "unit": "fingerprints/s", "cores": threads,
               "kind": r["kind"],
               "sample": (f"cfg1 generator at N={args.ref_n} (search is O(N^2); fp/s at N=8e6 "
                          f"would be ~{(8e6 / args.ref_n):.0f}x lower): reference compiled _sigcore on "
                          f"{threads} threads ({r['sig_s']:.2f} s) + numpy port of search_signatures "
                          f"single-threaded ({r['search_s']:.2f} s)")}

    fpb = None
    if rank == 0 and not args.no_fingerprint:
        fpb = fingerprint_bench(args.fp_samples, max(1, args.steps), dev)
        # the fingerprint chain against the measured FP64 peak (F_win
        # = 74,100 flops per window + the MAD pass's rate x 68,000)
        cpk = cuda_core_peaks()
        fp_flops = fpb["n_fingerprints"] * (74_100 + 0.1 * 68_000)
        fp_gf = fp_flops / (fpb["ms_per_step"] / 1e3) / 1e9
        fpb["roofline"] = {"bound": "fp64", "achieved": fp_gf, "peak": cpk["fp64_gflops"],
                           "peak_kind": "measured (qs_peak_launch, FP64 FMA)", "unit": "GFLOP/s",
                           "frac": fp_gf / cpk["fp64_gflops"],
                           "flops_per_call": fp_flops}
        fpb["cuda_core_peaks"] = cpk
        mh_roof = roof["other_stages"].get("minhash")
        if mh_roof and not tables_mode:
            # the reference kernel's work (K x t x k 64-bit compare-selects per
            # fingerprint, _sigcore.pyx:60-75) per second of the probe kernel
            ref_ops = 400 * 100 * 4 * n
            rate = ref_ops / (mh_roof["ms"] / 1e3) / 1e9
            mh_roof.update({"reference_equivalent_minmax_gops": rate,
                            "u64_minmax_peak_gops": cpk["u64_minmax_gops"],
                            "reference_equivalent_frac": rate / cpk["u64_minmax_gops"]})

    if rank == 0:
        line = {"metric": "LSH search fingerprints/sec (MinHash+bucket+pair-count)",
                "value": value, "unit": "fingerprints/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if tables_mode else "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic",
                "config": {"workload": "cfg1 (BASELINE.json configs[1])",
                           ("n_total" if tables_mode else "n_per_gpu"): n,
                           "d": 4096, "set_bits": 400, "tables": 100, "hash_funcs": 4,
                           "min_matches": 5, "occurrence_threshold": occ, "partitions": 1,
                           "l2": f"inputs ({n * 400 * 4 / 1e9:.1f} GB bits) larger than L2 "
                                 "(126 MB); no flush",
                           "parallelism": (f"table-sharded x{world} (round-robin tables, "
                                           "row-sharded Min-Max + NCCL all-gather)" if tables_mode
                                           else f"station-sharded x{world}")},
                "stages_ms": stages, "emitted_triplets": st.emitted_triplets,
                "filtered_fingerprints": st.filtered_fingerprints,
                "distinct_pairs": st.distinct_pairs, "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
                "fingerprint": fpb}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
