"""Generate tests/golden/* by running the REFERENCE implementation.

Runs only in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the reference package `quakescan` from /root/reference/pkg/src
(the reference's compiled `_sigcore`, built into oracle/_ref by
`make -C oracle ref`, is registered as `quakescan._sigcore` when present;
otherwise the reference's own bit-identical numpy backend is used) and records
inputs and outputs of the hot-path functions as small fixtures. Nothing on
the GPU box reads /root/reference; the fixtures travel instead.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import oracle  # noqa: E402

core = oracle.ref_sigcore()
if core is not None:
    sys.modules["quakescan._sigcore"] = core

from quakescan import fingerprint as rfp  # noqa: E402
from quakescan import lsh_search as rls  # noqa: E402
from quakescan import minmax_hash as rmh  # noqa: E402
from quakescan.ingest import TimeSeries  # noqa: E402

from paper_1803_09835_b200 import workloads  # noqa: E402


def kat():
    xs = [0, 1, 2, 0xDEADBEEF, 2**63, 2**64 - 1, 0x0123456789ABCDEF, 12345]
    fm = {hex(x): hex(int(rmh.fmix64(np.array([x], np.uint64))[0])) for x in xs}
    hv = {}
    for x, s in [(0, 0), (1, 0), (0, 1), (12345, 67890), (8191, 2**63), (4095, 2**64 - 1)]:
        hv[f"{x},{s}"] = hex(int(rmh.hash_values(np.array([x], np.uint64), s)[0]))
    cb = {}
    for ws in [(0,), (1, 2), (5, 9, 3), (2**64 - 1, 0, 7, 2**63)]:
        cb[",".join(str(w) for w in ws)] = hex(rmh.combine(np.array(ws, np.uint64)))
    m = rmh.gen_hash_mapping(d=64, t=3, k=4, seed=42)
    sig = rmh.signatures(np.array([[0, 5, 17, 63]], np.uint32), m)[0]
    # detection_probability (lsh_search.py:112-136) at the reference's DP_FROZEN
    # points (tests/test_lsh_search.py:13-22) plus a grid, evaluated by the reference
    pts = [(0.5, 6, 5, 100), (0.5, 4, 2, 100), (0.8, 6, 5, 100), (0.2, 6, 5, 100),
           (0.3, 8, 2, 100), (0.7, 8, 2, 100), (0.95, 2, 90, 100), (0.1, 2, 1, 10)]
    pts += [(s, k, m, t) for s in (0.0, 0.05, 0.4, 0.65, 0.9, 1.0) for k in (2, 4, 8)
            for m, t in ((1, 1), (5, 100), (20, 50))]
    dp = [[s, k, m, t, rls.detection_probability(s, k, m, t)] for s, k, m, t in pts]
    return dict(fmix64=fm, hash=hv, combine=cb, dp_frozen=dp,
                sig_d64_t3_k4_s42_bits_0_5_17_63=[hex(int(v)) for v in sig],
                backend=rmh.BACKEND)


def minmax_cases():
    rng = np.random.default_rng(31)
    cases = {}
    for name, (n, d, K, t, k, seed) in {
        "small": (64, 1024, 50, 10, 6, 3),
        "cfg0shape": (256, 4096, 200, 100, 4, 0),
        "cfg1shape": (512, 4096, 400, 100, 4, 0),
        "odd": (33, 97, 7, 5, 2, 2**64 - 3),
        "k8": (40, 8192, 100, 13, 8, 12345),
    }.items():
        bits = np.stack([np.sort(rng.choice(d, K, replace=False)) for _ in range(n)]).astype(np.uint32)
        m = rmh.gen_hash_mapping(d, t, k, seed)
        sigs = rmh.signatures(bits, m)
        cases[name] = dict(bits=bits, sigs=sigs, meta=np.array([d, t, k], np.int64),
                           seed=np.array([seed], np.uint64))
    return cases


def search_case(sigs, **cfg):
    excl = cfg.pop("exclusion_windows", 0)
    rec, st = rls.search_signatures(sigs, rls.SearchConfig(**cfg), exclusion_windows=excl)
    return rec, st.to_dict()


def burst_corpus(rng, n=400, burst=60, k_bits=60, d=2048):
    bits = np.stack([np.sort(rng.choice(d, k_bits, replace=False)) for _ in range(n)]).astype(np.uint32)
    rows = rng.permutation(n)
    burst_rows = np.sort(rows[:burst])
    pair_rows = np.sort(rows[burst:burst + 2])
    template = np.sort(rng.choice(d, k_bits, replace=False))
    pool = np.setdiff1d(np.arange(d), template)
    for r in burst_rows:
        churn = rng.integers(0, 4)
        keep = rng.choice(k_bits, k_bits - churn, replace=False)
        bits[r] = np.sort(np.concatenate([template[keep], rng.choice(pool, churn, replace=False)]))
    event = np.sort(rng.choice(d, k_bits, replace=False))
    bits[pair_rows[0]] = event
    bits[pair_rows[1]] = event
    return bits


def search_cases():
    rng = np.random.default_rng(5)
    out = {}
    prone = rng.integers(0, 40, size=(300, 16)).astype(np.uint64)
    for p in (1, 2, 3, 8):
        out[f"prone_p{p}"] = (prone, dict(tables=16, hash_funcs=2, min_matches=3,
                                          partitions=p, exclusion_windows=2))
    tiny = rng.integers(0, 5, size=(150, 10)).astype(np.uint64)
    out["tiny_alpha_excl0"] = (tiny, dict(tables=10, hash_funcs=2, min_matches=2))
    out["tiny_alpha_excl5_p3"] = (tiny, dict(tables=10, hash_funcs=2, min_matches=2,
                                             partitions=3, exclusion_windows=5))
    out["tiny_alpha_occ"] = (tiny, dict(tables=10, hash_funcs=2, min_matches=2,
                                        occurrence_threshold=0.2, exclusion_windows=1))
    out["tiny_alpha_occ_p4"] = (tiny, dict(tables=10, hash_funcs=2, min_matches=2,
                                           occurrence_threshold=0.2, partitions=4))
    bits = burst_corpus(np.random.default_rng(9))
    m = rmh.gen_hash_mapping(2048, 32, 4, 1)
    bs = rmh.signatures(bits, m)
    out["burst_off"] = (bs, dict(tables=32, hash_funcs=4, min_matches=2))
    out["burst_on"] = (bs, dict(tables=32, hash_funcs=4, min_matches=2, occurrence_threshold=0.05))
    out["burst_on_p4"] = (bs, dict(tables=32, hash_funcs=4, min_matches=2,
                                   occurrence_threshold=0.05, partitions=4))
    out["empty"] = (np.zeros((0, 4), np.uint64), dict(tables=4, hash_funcs=2, min_matches=1))
    out["single"] = (np.zeros((1, 4), np.uint64), dict(tables=4, hash_funcs=2, min_matches=1))
    out["all_same"] = (np.full((64, 6), 7, np.uint64), dict(tables=6, hash_funcs=2, min_matches=6,
                                                           exclusion_windows=3))
    out["all_same_occ"] = (np.full((64, 6), 7, np.uint64),
                           dict(tables=6, hash_funcs=2, min_matches=6, occurrence_threshold=0.5,
                                partitions=2))
    # cfg1-shaped: 400-of-4096, t=100, k=4, m=5, planted pairs and noise groups
    cbits, _ = workloads.cfg1_bits(n=3000, seed=11, pair_frac=1 / 60, group_frac=1 / 1000)
    cm = rmh.gen_hash_mapping(4096, 100, 4, 0)
    csig = rmh.signatures(cbits, cm)
    out["cfg1_small"] = (csig, dict(tables=100, hash_funcs=4, min_matches=5))
    out["cfg1_small_occ"] = (csig, dict(tables=100, hash_funcs=4, min_matches=5,
                                        occurrence_threshold=120 / 3000))
    out["cfg1_small_occ_p3"] = (csig, dict(tables=100, hash_funcs=4, min_matches=5,
                                           occurrence_threshold=60 / 3000, partitions=3,
                                           exclusion_windows=7))
    res = {}
    for name, (sigs, cfg) in out.items():
        rec, st = search_case(sigs, **dict(cfg))
        res[name] = (sigs, cfg, rec, st)
    return res


def fingerprint_cases():
    cases = {}
    x, _ = workloads.cfg0_trace(n_samples=60 * 60 * 100 // 2, seed=3, copies=4)
    p = workloads.CFG0_PARAMS
    params = rfp.FingerprintParams(
        window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
        freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
        band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
        stft=rfp.StftParams(frame_len_s=p["frame_len_s"], hop_s=p["hop_s"]))
    ts = TimeSeries("ST0", "HHZ", 100.0, 1000.0, x)
    fps, mad = rfp.fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
    freqs, times, logpow = rfp.spectrogram(ts, params)
    r0, r1 = rfp._band_rows(freqs, params)
    sel = np.array([0, 1, 7, 100, 555, fps.bits.shape[0] - 1])
    _, _, coeffs = next(rfp.iter_coeff_batches(ts, params, indices=sel))
    _, _, imgs = next(rfp.iter_image_batches(ts, params, indices=sel))
    cases["cfg0_half_hour"] = dict(
        samples=x, bits=fps.bits, median=mad.median, mad=mad.mad,
        band=np.ascontiguousarray(logpow[r0:r1].T), band_rows=np.array([r0, r1]),
        sel=sel, coeffs=coeffs, images=imgs,
        meta=np.array([mad.n_sampled, mad.n_total]))
    # small reference-test geometry with a non-power-of-two image side
    rng = np.random.default_rng(4)
    y = rng.standard_normal(30_000).astype(np.float32)
    small = rfp.FingerprintParams(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12,
                                  top_k=24, stft=rfp.StftParams(frame_len_s=0.5, hop_s=0.05))
    ts2 = TimeSeries("ST1", "HHZ", 100.0, 0.0, y)
    fps2, mad2 = rfp.fingerprint_series(ts2, small, mad_rate=1.0)
    cases["small_full_band"] = dict(samples=y, bits=fps2.bits, median=mad2.median, mad=mad2.mad,
                                    meta=np.array([mad2.n_sampled, mad2.n_total]))
    return cases


def bandpass_cases():
    """Reference ingest.bandpass (scipy sosfiltfilt) on seeded traces."""
    from quakescan import ingest as ring
    rng = np.random.default_rng(21)
    out = {}
    for name, (n, lo, hi, order, sr) in {
        "cfg0_band": (60_000, 4.0, 10.0, 4, 100.0),
        "wide_o2": (50_000, 1.0, 20.0, 2, 100.0),
        "o8_short": (5_000, 2.0, 8.0, 8, 50.0),
        "o1_min": (40, 5.0, 15.0, 1, 100.0),
    }.items():
        x = rng.standard_normal(n).astype(np.float32).astype(np.float64)
        x += np.sin(np.arange(n) * 0.3) * 3.0
        ts = TimeSeries("ST0", "HHZ", sr, 0.0, x)
        y = ring.bandpass(ts, ring.BandpassSpec(lo, hi, order)).samples
        out[name] = dict(x=x, y=y, spec=np.array([lo, hi, order, sr]))
    return out


def files():
    """Artifacts written by the reference's own writers (lsh_search.py:339-393,
    fingerprint.py:392-404, 529-551) -> tests/golden/files/."""
    out = os.path.join(HERE, "files")
    os.makedirs(out, exist_ok=True)
    rng = np.random.default_rng(4)
    y = rng.standard_normal(30_000).astype(np.float32)
    small = rfp.FingerprintParams(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12,
                                  top_k=24, stft=rfp.StftParams(frame_len_s=0.5, hop_s=0.05))
    ts2 = TimeSeries("ST1", "HHZ", 100.0, 12.5, y)
    fps2, mad2 = rfp.fingerprint_series(ts2, small, mad_rate=1.0)
    rfp.write_fingerprint_file(os.path.join(out, "ref.fp"), fps2,
                               extra={"config_hash": "abc123", "mad_seed": 0, "mad_rate": 1.0})
    rfp.write_mad_file(os.path.join(out, "ref.mad"), mad2, extra={"station": "ST1"})
    sigs = np.load(os.path.join(HERE, "search.npz"))["sigs7"]
    cfg = rls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=0.04)
    rec, _ = rls.search_signatures(sigs, cfg)
    header = {"config_hash": "abc123", "station": "ST1", "channel": "HHZ", "window_len_s": 3.0,
              "window_lag_s": 0.5, "start_epoch_s": 12.5, "sorted": True}
    rls.write_triplet_file(os.path.join(out, "ref.tri"), rec, header)
    rls.write_triplet_csv(os.path.join(out, "ref.csv"), rec)
    # channel combine + external sort (align.py:87-140) on three channels
    from quakescan import align as ral
    rng2 = np.random.default_rng(9)
    pairs = rng2.integers(1, 40, size=(600, 2))
    chans = []
    for c in range(3):
        sel = pairs[rng2.random(len(pairs)) < 0.5]
        recc = np.zeros(len(sel), dtype=rls.TRIPLET_DTYPE)
        recc["dt"], recc["idx1"] = sel[:, 0], sel[:, 1]
        recc["sim"] = rng2.integers(1, 9, size=len(sel))
        recc = recc[np.lexsort((recc["idx1"], recc["dt"]))]
        # unique (dt, idx1) per channel, as a search emits
        keep = np.ones(len(recc), bool)
        keep[1:] = (recc["dt"][1:] != recc["dt"][:-1]) | (recc["idx1"][1:] != recc["idx1"][:-1])
        recc = recc[keep]
        pth = os.path.join(out, f"ch{c}.tri")
        rls.write_triplet_file(pth, recc, {"channel": f"C{c}", "sorted": True})
        chans.append(pth)
    ral.combine_channel_triplets(chans, os.path.join(out, "combined.tri"), 6,
                                 {"station": "ST1", "combined": True})
    shuffled = np.fromfile(chans[0], dtype=np.uint8)
    rec0, _ = rls.read_triplet_file(chans[0])
    rls.write_triplet_file(os.path.join(out, "unsorted.tri"), rec0[rng2.permutation(len(rec0))],
                           {"channel": "C0"})
    ral.sort_triplet_file(os.path.join(out, "unsorted.tri"), os.path.join(out, "sorted.tri"),
                          {"channel": "C0", "sorted": True}, chunk_records=50)
    del shuffled
    with open(os.path.join(out, "ref_inputs.json"), "w") as f:
        json.dump({"tri_header": header, "n_triplets": int(rec.size)}, f, sort_keys=True)
    for fn in sorted(os.listdir(out)):
        print(fn, os.path.getsize(os.path.join(out, fn)))


def row_hashes(a) -> np.ndarray:
    """8-byte blake2b digest of every row of a 2-D array (little-endian bytes)."""
    import hashlib
    a = np.ascontiguousarray(a)
    out = np.empty(a.shape[0], np.uint64)
    for i in range(a.shape[0]):
        out[i] = int.from_bytes(hashlib.blake2b(a[i].tobytes(), digest_size=8).digest(), "little")
    return out


def fingerprint_day():
    """The full cfg0 day (BASELINE configs[0]: 8.64e6 samples, 86,391 windows)
    through the reference: per-window digests of the float32 coefficient rows
    and of the bit rows, the band-row spectrogram digest per 4096-column block,
    and the MAD statistics.  Digests keep the fixture small (the arrays are
    707 MB of coefficients); the GPU test recomputes the values with the
    oracle on the box for ulp-level comparisons and uses these digests to pin
    that oracle run to the reference's."""
    x, _ = workloads.cfg0_trace()
    p = workloads.CFG0_PARAMS
    params = rfp.FingerprintParams(
        window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
        freq_bins=p["freq_bins"], time_bins=p["time_bins"], top_k=p["top_k"],
        band_low_hz=p["band_low_hz"], band_high_hz=p["band_high_hz"],
        stft=rfp.StftParams(frame_len_s=p["frame_len_s"], hop_s=p["hop_s"]))
    ts = TimeSeries("ST0", "HHZ", 100.0, 0.0, x)
    fps, mad = rfp.fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
    freqs, times, logpow = rfp.spectrogram(ts, params)
    r0, r1 = rfp._band_rows(freqs, params)
    band = np.ascontiguousarray(logpow[r0:r1].T)
    nblk = -(-band.shape[0] // 4096)
    band_blk = np.zeros((nblk, 4096 * band.shape[1]), np.float32)
    for k in range(nblk):
        blk = band[k * 4096:(k + 1) * 4096].reshape(-1)
        band_blk[k, :blk.size] = blk
    chash = np.empty(fps.bits.shape[0], np.uint64)
    for idx, _, c in rfp.iter_coeff_batches(ts, params):
        chash[idx] = row_hashes(c)
    return dict(bits_hash=row_hashes(fps.bits), coeff_hash=chash, band_hash=row_hashes(band_blk),
                band_rows=np.array([r0, r1]), median=mad.median, mad=mad.mad,
                meta=np.array([mad.n_sampled, mad.n_total, fps.bits.shape[0], fps.bits.shape[1]]))


def demo_golden():
    """The reference's frozen demo report (pkg/tests/data/demo_golden.json),
    re-derived here with the reference's serial in-memory harness
    (pkg/tests/test_cli.py:54-100, reference stages throughout) and copied
    only if the two agree byte for byte."""
    import tempfile
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, ROOT)
    from quakescan import config as rcfg
    from quakescan import ingest as ring
    from test_demo_golden_gpu import detection_report
    from quakescan import align as ral
    from importlib import resources
    ref = dict(align=ral, ingest=ring, lsh_search=rls, config=rcfg)
    with tempfile.TemporaryDirectory() as tmp:
        dst = os.path.join(tmp, "demo.toml")
        with open(dst, "w") as f:
            f.write(resources.files("quakescan").joinpath("data/demo.toml").read_text())
        cfg = rcfg.load_config(dst)
        blob = detection_report(ref, cfg, ring.bandpass, rfp.fingerprint_series,
                                rls.search_fingerprints)
    with open("/root/reference/pkg/tests/data/demo_golden.json", "rb") as f:
        frozen = f.read()
    assert blob == frozen, "reference harness does not reproduce its own golden"
    with open(os.path.join(HERE, "demo_golden.json"), "wb") as f:
        f.write(blob)


def main():
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat(), f, indent=1, sort_keys=True)
    mm = minmax_cases()
    np.savez_compressed(os.path.join(HERE, "minmax.npz"),
                        **{f"{c}__{k}": v for c, d in mm.items() for k, v in d.items()})
    sc = search_cases()
    arrays, meta, seen = {}, {}, {}
    for name, (sigs, cfg, rec, st) in sc.items():
        key = seen.setdefault(id(sigs), f"sigs{len(seen)}")
        arrays[key] = sigs
        arrays[f"{name}__trip"] = rec
        meta[name] = dict(cfg=cfg, stats=st, sigs=key)
    np.savez_compressed(os.path.join(HERE, "search.npz"), **arrays)
    with open(os.path.join(HERE, "search.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    fc = fingerprint_cases()
    np.savez_compressed(os.path.join(HERE, "fingerprint.npz"),
                        **{f"{c}__{k}": v for c, d in fc.items() for k, v in d.items()})
    for fn in sorted(os.listdir(HERE)):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))


if __name__ == "__main__":
    if "--kat" in sys.argv:
        with open(os.path.join(HERE, "kat.json"), "w") as f:
            json.dump(kat(), f, indent=1, sort_keys=True)
    elif "--files" in sys.argv:
        files()
    elif "--day" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "fingerprint_day.npz"), **fingerprint_day())
    elif "--demo" in sys.argv:
        demo_golden()
    elif "--bandpass" in sys.argv:
        bp = bandpass_cases()
        np.savez_compressed(os.path.join(HERE, "bandpass.npz"),
                            **{f"{c}__{k}": v for c, d in bp.items() for k, v in d.items()})
    else:
        main()
        files()
