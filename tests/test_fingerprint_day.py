"""The full cfg0 day (BASELINE configs[0]: 8.64e6 samples, 86,391 windows).

Pins (tests/golden/fingerprint_day.npz, made by make_golden.py --day from the
reference itself): per-window digests of the reference's float32 Haar
coefficient rows and bit rows, band-row spectrogram digests, MAD statistics.

* CPU: the oracle restatement reproduces every digest (so it is the
  reference's output, bit for bit, at full scale on this machine).
* GPU: the device chain against that oracle run on the same samples, with
  tolerances sized to the f64 design: spectrogram band values
  within 1 float32 ulp; coefficients within COEFF_ULP ulps of their window's
  largest coefficient; bits identical on every window except where the
  K-th and (K+1)-th |v'| are a near-tie the ulp-level coefficient difference
  can reorder.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import fingerprint as ofp

# Measured on the B200 (profiles/r02_pytest_gpu.log): band rows max 1 ulp
# (>99.9999 % identical: a direct f64 DFT vs pocketfft rounding), coefficients
# and bits identical on every window.  Limits sit at what the design delivers.
SPEC_ULP = 1          # float32 ulps, band rows of the spectrogram
SPEC_EXACT = 0.9999   # fraction of band values bit-identical
COEFF_ULP = 1         # float32 ulps of max|coefficient| of the window
COEFF_EXACT = 0.99999  # fraction of coefficients bit-identical
TIE_REL = 1e-6        # relative gap between the K-th and (K+1)-th |v'| below which
                      # a bit difference counts as a tie reordering
MAX_TIE_WINDOWS = 2   # windows allowed to differ (only at such near-ties)


def _row_hashes(a):
    import hashlib
    a = np.ascontiguousarray(a)
    out = np.empty(a.shape[0], np.uint64)
    for i in range(a.shape[0]):
        out[i] = int.from_bytes(hashlib.blake2b(a[i].tobytes(), digest_size=8).digest(), "little")
    return out


@pytest.fixture(scope="module")
def golden_day():
    z = np.load(os.path.join(GOLDEN, "fingerprint_day.npz"))
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def oracle_day():
    """The oracle chain over the whole day (~40 s on one core)."""
    from paper_1803_09835_b200 import workloads
    x, _ = workloads.cfg0_trace()
    p = workloads.CFG0_PARAMS
    xf = x.astype(np.float64)
    g = ofp.geometry(100.0, xf.size, p["window_len_s"], p["window_lag_s"], p["frame_len_s"],
                     p["hop_s"])
    spec = ofp.stft_logpow(xf, g["frame"], g["hop"])
    freqs = np.fft.rfftfreq(g["frame"], 1.0 / 100.0)
    r0, r1 = ofp.band_rows(freqs, p["band_low_hz"], p["band_high_hz"])
    band = np.ascontiguousarray(spec[:, r0:r1])
    del spec
    F, T = p["freq_bins"], p["time_bins"]
    coeffs = ofp.coeffs(band, np.arange(g["n_win"]), g, F, T, batch=512)
    sample = ofp.mad_sample(g["n_win"], 0.1, 0)
    med, mad = ofp.mad_stats(coeffs[sample])
    bits = np.empty((g["n_win"], p["top_k"]), np.uint32)
    for a in range(0, g["n_win"], 4096):
        bits[a:a + 4096] = ofp.topk_bits(coeffs[a:a + 4096], med, mad, p["top_k"])
    return dict(x=x, band=band, band_rows=(r0, r1), coeffs=coeffs, med=med, mad=mad, bits=bits,
                params=p)


def test_oracle_day_pinned_to_reference(oracle_day, golden_day):
    o, gd = oracle_day, golden_day
    assert tuple(o["band_rows"]) == tuple(gd["band_rows"])
    band = o["band"]
    nblk = -(-band.shape[0] // 4096)
    blk = np.zeros((nblk, 4096 * band.shape[1]), np.float32)
    for k in range(nblk):
        v = band[k * 4096:(k + 1) * 4096].reshape(-1)
        blk[k, :v.size] = v
    assert np.array_equal(_row_hashes(blk), gd["band_hash"])
    assert np.array_equal(_row_hashes(o["coeffs"]), gd["coeff_hash"])
    assert np.array_equal(o["med"], gd["median"]) and np.array_equal(o["mad"], gd["mad"])
    assert np.array_equal(_row_hashes(o["bits"]), gd["bits_hash"])


def _params(fp, p):
    return fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                                freq_bins=p["freq_bins"], time_bins=p["time_bins"],
                                top_k=p["top_k"], band_low_hz=p["band_low_hz"],
                                band_high_hz=p["band_high_hz"],
                                stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))


def _ulps(got, want):
    """float32 ulp distance (same-sign values; sign changes count large)."""
    a = np.ascontiguousarray(got, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(want, np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7FFFFFFF), a)
    b = np.where(b < 0, -(b & 0x7FFFFFFF), b)
    return np.abs(a - b)


@pytest.mark.gpu
def test_day_spectrogram_and_coefficients(oracle_day):
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200.ingest import TimeSeries
    o = oracle_day
    params = _params(fp, o["params"])
    ts = TimeSeries("ST0", "HHZ", 100.0, 0.0, o["x"])
    _, _, logpow = fp.spectrogram(ts, params)
    r0, r1 = o["band_rows"]
    u = _ulps(logpow[r0:r1].T, o["band"])
    print(f"\nspectrogram band rows: max {int(u.max())} ulp, {float(np.mean(u == 0)):.6f} exact")
    assert int(u.max()) <= SPEC_ULP and float(np.mean(u == 0)) >= SPEC_EXACT
    worst, exact = 0.0, 0
    for idx, _, c in fp.iter_coeff_batches(ts, params, batch=8192):
        want = o["coeffs"][idx]
        scale = np.abs(want).max(axis=1, keepdims=True).astype(np.float32)
        ulp = np.spacing(scale)
        err = np.abs(c.astype(np.float64) - want) / ulp
        worst = max(worst, float(err.max()))
        exact += int(np.sum(c == want))
    print(f"coefficients: max {worst:.2f} ulp of the window max, "
          f"{exact / o['coeffs'].size:.6f} exact")
    assert worst <= COEFF_ULP and exact / o["coeffs"].size >= COEFF_EXACT


@pytest.mark.gpu
def test_day_bits_and_mad(oracle_day, golden_day):
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200.ingest import TimeSeries
    o = oracle_day
    params = _params(fp, o["params"])
    fps, mad = fp.fingerprint_series(TimeSeries("ST0", "HHZ", 100.0, 0.0, o["x"]), params,
                                     mad_rate=0.1, mad_seed=0)
    # medians/MADs of float32 coefficients, averaged in f64 like np.median:
    # identical coefficients give identical statistics
    np.testing.assert_allclose(mad.median, golden_day["median"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(mad.mad, golden_day["mad"], rtol=1e-12, atol=0)
    assert np.array_equal(mad.mad > 0, golden_day["mad"] > 0)
    same = _row_hashes(fps.bits) == golden_day["bits_hash"]
    diff = np.flatnonzero(~same)
    print(f"\nbits: {same.size - diff.size}/{same.size} windows identical to the reference")
    K = o["params"]["top_k"]
    ok = golden_day["mad"] > 0
    for i in diff:
        c = o["coeffs"][i].astype(np.float64)
        v = np.where(ok, (c - golden_day["median"]) / np.where(ok, golden_day["mad"], 1.0), 0.0)
        mag = np.sort(np.abs(v[ok]))[::-1]
        gap = (mag[K - 1] - mag[K]) / max(mag[K - 1], 1e-300)
        assert gap <= TIE_REL, (int(i), gap)
    assert diff.size <= MAX_TIE_WINDOWS
