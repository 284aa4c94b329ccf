"""Fingerprint chain parity on the GPU.

Tolerances are set at what the f64 design delivers (measured, see
tests/test_fingerprint_day.py), far inside the north star's 1e-4 relative /
99.9 % of bits: spectrogram and image values within 1 float32 ulp,
coefficients within 1 ulp of their window's largest magnitude, MAD
statistics to 1e-12 relative, fingerprint bits identical.  Mirrors the
reference's tests/test_fingerprint.py strategy (Haar oracle + roundtrip,
resize constants, top-K oracle with ties and sign encoding, MAD definition,
error taxonomy) plus golden vectors produced by the reference itself."""

import math

import numpy as np
import pytest

from oracle import fingerprint as ofp

pytestmark = pytest.mark.gpu

ULP = 1


@pytest.fixture(scope="module")
def fp():
    from paper_1803_09835_b200 import fingerprint
    return fingerprint


def _params(fp, p):
    return fp.FingerprintParams(window_len_s=p["window_len_s"], window_lag_s=p["window_lag_s"],
                                freq_bins=p["freq_bins"], time_bins=p["time_bins"],
                                top_k=p["top_k"], band_low_hz=p["band_low_hz"],
                                band_high_hz=p["band_high_hz"],
                                stft=fp.StftParams(p["frame_len_s"], p["hop_s"]))


def _close(got, want, per_row=False):
    """|got - want| <= ULP float32 ulps of want (elementwise), or of the row's
    largest magnitude (per_row: Haar detail coefficients near zero)."""
    got = np.asarray(got, np.float32).astype(np.float64)
    want = np.asarray(want, np.float32)
    if per_row:
        w2 = want.reshape(want.shape[0], -1)
        scale = np.abs(w2).max(axis=1, keepdims=True).astype(np.float32)
        ulp = np.broadcast_to(np.spacing(scale), w2.shape).reshape(want.shape)
    else:
        ulp = np.spacing(np.abs(want))
    err = np.abs(got - want.astype(np.float64))
    assert np.all(err <= ULP * ulp.astype(np.float64)), float((err / ulp).max())


def _ts(x, sr=100.0, start=0.0):
    from paper_1803_09835_b200.ingest import TimeSeries
    return TimeSeries("ST0", "HHZ", sr, start, x)


def test_golden_cfg0_chain(fp, golden_fingerprint):
    from paper_1803_09835_b200 import workloads
    case = golden_fingerprint["cfg0_half_hour"]
    params = _params(fp, workloads.CFG0_PARAMS)
    ts = _ts(case["samples"], start=1000.0)
    freqs, times, logpow = fp.spectrogram(ts, params)
    r0, r1 = (int(v) for v in case["band_rows"])
    _close(logpow[r0:r1].T, case["band"])
    exact = np.mean(logpow[r0:r1].T == case["band"])
    assert exact > 0.9999
    (idx, ep, imgs), = list(fp.iter_image_batches(ts, params, indices=case["sel"]))
    _close(imgs, case["images"])
    (idx, ep, coeffs), = list(fp.iter_coeff_batches(ts, params, indices=case["sel"]))
    _close(coeffs, case["coeffs"], per_row=True)
    assert np.array_equal(idx, case["sel"]) and np.allclose(ep, 1000.0 + case["sel"] * 1.0)
    fps, mad = fp.fingerprint_series(ts, params, mad_rate=0.1, mad_seed=0)
    assert (mad.n_sampled, mad.n_total) == tuple(int(v) for v in case["meta"])
    np.testing.assert_allclose(mad.median, case["median"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(mad.mad, case["mad"], rtol=1e-12, atol=0)
    assert np.array_equal(mad.mad > 0, case["mad"] > 0)  # the structural zero-MAD coefficients
    assert fps.bits.shape == case["bits"].shape and fps.bits.dtype == np.uint32
    assert np.array_equal(fps.bits, case["bits"])
    fps.validate()
    assert fps.meta["station"] == "ST0" and fps.d == 4096


def test_golden_small_full_band(fp, golden_fingerprint):
    case = golden_fingerprint["small_full_band"]
    params = fp.FingerprintParams(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12,
                                  top_k=24, stft=fp.StftParams(frame_len_s=0.5, hop_s=0.05))
    fps, mad = fp.fingerprint_series(_ts(case["samples"]), params, mad_rate=1.0)
    np.testing.assert_allclose(mad.median, case["median"], rtol=1e-12, atol=0)
    assert np.array_equal(fps.bits, case["bits"])


def test_random_traces_vs_oracle(fp):
    rng = np.random.default_rng(11)
    for n, params in [(20_000, dict(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=16,
                                    top_k=24, band_low_hz=None, band_high_hz=None,
                                    frame_len_s=0.5, hop_s=0.05)),
                      (9_000, dict(window_len_s=4.0, window_lag_s=0.7, freq_bins=6, time_bins=10,
                                   top_k=9, band_low_hz=3.0, band_high_hz=20.0,
                                   frame_len_s=0.64, hop_s=0.13))]:
        x = rng.standard_normal(n)  # float64 trace
        res = ofp.fingerprint(x, 100.0, params, mad_rate=0.5, mad_seed=3)
        fps, mad = fp.fingerprint_series(_ts(x), _params(fp, params), mad_rate=0.5, mad_seed=3)
        np.testing.assert_allclose(mad.median, res["median"], rtol=1e-9, atol=1e-12)
        agree = float(np.mean(fps.bits == res["bits"]))
        print(f"random trace n={n}: bits agreement {agree:.6f}")
        assert agree >= 0.9999


def test_haar_matches_oracle_and_roundtrip(fp):
    rng = np.random.default_rng(5)
    for shape in [(2, 2), (4, 4), (8, 2), (2, 8), (4, 6), (3, 8), (32, 128), (5, 7, 12)]:
        a = rng.standard_normal(shape)
        np.testing.assert_allclose(fp.haar2d(a), ofp.haar2d(a), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(fp.ihaar2d(fp.haar2d(a)), a, rtol=1e-9, atol=1e-9)
    c = fp.haar2d(np.full((32, 128), 1.5))
    assert c[0, 0] == pytest.approx(1.5 * math.sqrt(32 * 128), rel=1e-12)
    from paper_1803_09835_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        fp.haar2d(np.zeros(4))


def test_topk_oracle_ties_and_signs(fp):
    rng = np.random.default_rng(2)
    n = 64
    med = rng.standard_normal(n)
    mad = np.abs(rng.standard_normal(n)) + 0.1
    mad[[3, 10, 40]] = 0.0  # ineligible
    stats = fp.MadStats(median=med, mad=mad, rate=1.0, seed=0, n_sampled=1, n_total=1)
    c = rng.standard_normal((50, n)).astype(np.float32)
    # engineered ties: several coefficients at the same |v'|
    c[:, 20] = (med[20] + 1.5 * mad[20]).astype(np.float32)
    c[:, 21] = (med[21] - 1.5 * mad[21]).astype(np.float32)
    c[:5] = np.float32(0.0)
    for k in (1, 7, 30, 61):
        got = fp.topk_bits(c, stats, k)
        want = ofp.topk_bits(c, med, mad, k)
        assert np.array_equal(got, want), k
    scores = fp.normalize(c, stats)
    want = np.where(mad > 0, (c.astype(np.float64) - med) / np.where(mad > 0, mad, 1.0), 0.0)
    np.testing.assert_allclose(scores, want, rtol=1e-15, atol=0)
    # float64 input stays float64 (the reference's np.asarray(coeffs, float64))
    c64 = rng.standard_normal((7, n)) * 1e-3 + 1.0 / 3.0
    want64 = np.where(mad > 0, (c64 - med) / np.where(mad > 0, mad, 1.0), 0.0)
    assert np.array_equal(fp.normalize(c64, stats), want64)
    from paper_1803_09835_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        fp.normalize(np.zeros((2, n + 1), np.float32), stats)


def test_errors(fp):
    from paper_1803_09835_b200.errors import DataError, ParameterError
    params = fp.FingerprintParams(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=16,
                                  top_k=24, stft=fp.StftParams(frame_len_s=0.5, hop_s=0.05))
    with pytest.raises(DataError):
        fp.fingerprint_series(_ts(np.zeros(100)), params)
    with pytest.raises(ParameterError):
        fp.FingerprintParams(top_k=0).validate()
    stats = fp.MadStats(median=np.zeros(4), mad=np.array([1.0, 0.0, 0.0, 0.0]), rate=1.0, seed=0,
                        n_sampled=1, n_total=1)
    with pytest.raises(ParameterError):
        fp.topk_bits(np.zeros((1, 4)), stats, 2)
    with pytest.raises(DataError):
        fp.topk_bits(np.array([[np.nan, 0, 0, 0]]), stats, 1)


def test_device_trace_and_search_integration(fp):
    import torch
    from oracle import minmax as omm
    from oracle import search as osr
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import workloads
    x, _ = workloads.cfg0_trace(n_samples=90_000, seed=9, copies=3)
    params = _params(fp, workloads.CFG0_PARAMS)
    fps_h, mad = fp.fingerprint_series(_ts(x), params)
    fps_d, _ = fp.fingerprint_series(_ts(torch.from_numpy(x).cuda()), params)
    assert fps_d.bits.is_cuda
    assert np.array_equal(fps_d.bits.cpu().numpy().view(np.uint32), fps_h.bits)
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=0.01)
    rec, st, mapping = ls.search_fingerprints(fps_h, cfg)
    sigs = omm.signatures_c(fps_h.bits, mapping.values, 100, 2, threads=4)
    want, wst = osr.search(sigs, tables=100, min_matches=5, partitions=1,
                           occurrence_threshold=0.01, exclusion_windows=10)
    assert rec.tobytes() == want.tobytes()
    assert st.distinct_pairs == wst["distinct_pairs"]


def test_host_trace_upload_paths(fp, monkeypatch):
    """The host -> device copy of the trace changes nothing: a float32
    recording (coerced to float64 by TimeSeries, every sample exactly a
    float32) goes up narrowed to float32; a float64 trace with inexact samples
    falls back to the float64 copy; page-locked arrays are copied in place.
    All equal the device-resident float64 trace's fingerprints."""
    import torch
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import workloads
    x64, _ = workloads.cfg0_trace(n_samples=120_000, seed=4, copies=3)
    x64 = np.array(x64, dtype=np.float64)
    x64[1000] = 0.1  # not a float32
    params = _params(fp, workloads.CFG0_PARAMS)
    for name, x in (("float32 recording", x64.astype(np.float32)), ("float64", x64)):
        xf = np.asarray(x, np.float64)
        exact = bool(np.array_equal(xf.astype(np.float32).astype(np.float64), xf))
        assert exact == (name == "float32 recording")
        want, wmad = fp.fingerprint_series(_ts(torch.from_numpy(xf).cuda()), params)
        want_bits = want.bits.cpu().numpy().view(np.uint32)
        got, gmad = fp.fingerprint_series(_ts(x), params)
        assert np.array_equal(got.bits, want_bits), name
        assert np.array_equal(gmad.median, wmad.median) and np.array_equal(gmad.mad, wmad.mad)
        monkeypatch.setenv("QS_H2D_NARROW", "0")
        got2, _ = fp.fingerprint_series(_ts(x), params)
        monkeypatch.delenv("QS_H2D_NARROW")
        assert np.array_equal(got2.bits, want_bits), name
        hold = torch.empty(xf.shape, dtype=torch.float64, pin_memory=True)
        hold.numpy()[...] = xf
        assert ls._host_pinned(hold.numpy())
        got3, _ = fp.fingerprint_series(_ts(hold.numpy()), params)
        assert np.array_equal(got3.bits, want_bits), name
