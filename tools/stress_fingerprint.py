"""Randomised fingerprint-chain parity sweep against the oracle (geometry,
band, image size and top-K drawn at random; run on a GPU box).  Bar: MAD
median within 1e-5 relative and >= 99.9 % of the fingerprint bits equal."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fingerprint as ofp
from paper_1803_09835_b200 import fingerprint as fp
from paper_1803_09835_b200.errors import ParameterError, DataError
from paper_1803_09835_b200.ingest import TimeSeries

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
t0 = time.time()
done = bad = 0
worst = 1.0
for seed in range(n_cases):
    rng = np.random.default_rng(500 + seed)
    F = int(rng.choice([4, 6, 8, 16, 32]))
    T = int(rng.choice([8, 10, 16, 32, 64]))
    frame = float(rng.choice([0.32, 0.5, 0.64, 1.0, 2.0]))
    hop = float(rng.choice([0.03, 0.05, 0.1, 0.13]))
    win = float(rng.uniform(max(2.0, frame * 1.5), 12.0))
    lag = float(rng.uniform(0.3, 2.0))
    lo = float(rng.uniform(0.5, 10.0)) if rng.random() < 0.7 else None
    hi = (lo + float(rng.uniform(3.0, 30.0))) if lo is not None else None
    k = int(rng.integers(4, max(5, F * T // 6)))
    p = dict(window_len_s=win, window_lag_s=lag, freq_bins=F, time_bins=T, top_k=k,
             band_low_hz=lo, band_high_hz=hi, frame_len_s=frame, hop_s=hop)
    n = int(rng.integers(20_000, 120_000))
    x = rng.standard_normal(n)
    try:
        params = fp.FingerprintParams(window_len_s=win, window_lag_s=lag, freq_bins=F, time_bins=T,
                                      top_k=k, band_low_hz=lo, band_high_hz=hi,
                                      stft=fp.StftParams(frame, hop))
        fps, mad = fp.fingerprint_series(TimeSeries("S", "C", 100.0, 0.0, x), params,
                                         mad_rate=0.3, mad_seed=seed)
    except (ParameterError, DataError) as e:
        try:
            ofp.fingerprint(x, 100.0, p, mad_rate=0.3, mad_seed=seed)
            print("GPU rejected, oracle accepted", seed, p, e, flush=True)
            bad += 1
        except Exception:
            pass
        continue
    res = ofp.fingerprint(x, 100.0, p, mad_rate=0.3, mad_seed=seed)
    done += 1
    agree = float(np.mean(fps.bits == res["bits"]))
    med_ok = np.allclose(mad.median, res["median"], rtol=1e-5, atol=1e-7)
    worst = min(worst, agree)
    if agree < 0.999 or not med_ok:
        bad += 1
        print("MISMATCH", seed, p, "agree", agree, "median ok", med_ok, flush=True)
print(f"{done - bad}/{done} valid cases within the bar, worst bit agreement {worst:.6f} "
      f"({time.time() - t0:.0f} s)")
