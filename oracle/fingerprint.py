"""ORACLE — test infrastructure only. Fingerprint chain restatement (numpy).

Restates reference pkg/src/quakescan/fingerprint.py:
  STFT geometry + log-power    :125-151  symmetric Hann taper (np.hanning),
                                         rfft in float64, log10(|X|^2 + 1e-12)
                                         in float64, stored float32, (n_cols, n_freq)
  band rows                    :166-173  rows with low-1e-9 <= f <= high+1e-9
  area-overlap resize weights  :176-186  (dst, src), rows sum to 1
  window geometry              :189-195, 224-231  c0 = ceil(i*lag/hop),
                                         c1 = (i*lag + win - frame)//hop + 1
  spectral image               :232-241  (B, F, T) = w_f . band(spec) . w_t^T in
                                         float64, stored float32
  2-D Haar                     :256-300  row pass then column pass per level over
                                         the current block, 1/sqrt(2) scaling,
                                         float64; coefficients stored float32 (:334)
  MAD statistics               :341-389  sorted default_rng(seed).choice sample,
                                         per column median and median(|x - med|) in f64
  normalize / top-K            :425-466  v' = (v - med)/mad (0 where mad == 0),
                                         |v'| with ineligible -> -1, K-th largest,
                                         ties to the lower index, bit 2j + (v' < 0)
"""

import math

import numpy as np

LOG_EPS = 1e-12
INV_SQRT2 = 1.0 / math.sqrt(2.0)


def geometry(sr, n_samples, window_len_s, window_lag_s, frame_len_s, hop_s):
    frame = int(round(frame_len_s * sr))
    hop = max(1, int(round(hop_s * sr)))
    win = int(round(window_len_s * sr))
    lag = max(1, int(round(window_lag_s * sr)))
    n_cols = (n_samples - frame) // hop + 1 if n_samples >= frame else 0
    n_win = (n_samples - win) // lag + 1 if n_samples >= win else 0
    return dict(frame=frame, hop=hop, win=win, lag=lag, n_cols=n_cols, n_win=n_win)


def stft_logpow(samples, frame: int, hop: int):
    """(n_cols, frame//2+1) float32 log-power, frames-major."""
    x = np.asarray(samples, dtype=np.float64)
    n_cols = (x.size - frame) // hop + 1
    taper = np.hanning(frame)
    out = np.empty((n_cols, frame // 2 + 1), np.float32)
    frames = np.lib.stride_tricks.sliding_window_view(x, frame)[::hop]
    step = max(1, 4_000_000 // frame)
    for a in range(0, n_cols, step):
        b = min(n_cols, a + step)
        X = np.fft.rfft(frames[a:b] * taper, axis=1)
        out[a:b] = np.log10(X.real ** 2 + X.imag ** 2 + LOG_EPS).astype(np.float32)
    return out


def band_rows(freqs, low, high):
    if low is None:
        return 0, len(freqs)
    idx = np.flatnonzero((freqs >= low - 1e-9) & (freqs <= high + 1e-9))
    return int(idx[0]), int(idx[-1]) + 1


def resize_weights(src: int, dst: int) -> np.ndarray:
    r = src / dst
    w = np.zeros((dst, src))
    for i in range(dst):
        a, b = i * r, (i + 1) * r
        for j in range(int(math.floor(a)), min(int(math.ceil(b)), src)):
            w[i, j] = (min(b, j + 1) - max(a, j)) / r
    return w


def window_columns(idx, lag, win, frame, hop):
    off = np.asarray(idx, np.int64) * lag
    c0 = -(-off // hop)
    c1 = (off + win - frame) // hop + 1
    return c0, c1


def images(spec_band, idx, g, freq_bins, time_bins):
    """(B, F, T) float32 spectral images of windows `idx`."""
    c0, c1 = window_columns(idx, g["lag"], g["win"], g["frame"], g["hop"])
    w_f = resize_weights(spec_band.shape[1], freq_bins)
    out = np.empty((len(idx), freq_bins, time_bins), np.float32)
    for width in np.unique(c1 - c0):
        rows = np.flatnonzero((c1 - c0) == width)
        cols = c0[rows, None] + np.arange(width)
        w_t = resize_weights(int(width), time_bins)
        out[rows] = np.einsum("bwf,Ff,Tw->bFT", spec_band[cols], w_f, w_t,
                              optimize=True).astype(np.float32)
    return out


def haar_levels(h: int, w: int):
    lv = []
    while h % 2 == 0 and h > 1 and w % 2 == 0 and w > 1:
        lv.append((h, w, True, True))
        h //= 2
        w //= 2
    while w % 2 == 0 and w > 1:
        lv.append((h, w, True, False))
        w //= 2
    while h % 2 == 0 and h > 1:
        lv.append((h, w, False, True))
        h //= 2
    return lv


def haar2d(a) -> np.ndarray:
    out = np.array(a, dtype=np.float64, copy=True)
    for h, w, do_rows, do_cols in haar_levels(out.shape[-2], out.shape[-1]):
        if do_rows:
            e = out[..., :h, 0:w:2].copy()
            o = out[..., :h, 1:w:2].copy()
            out[..., :h, : w // 2] = (e + o) * INV_SQRT2
            out[..., :h, w // 2: w] = (e - o) * INV_SQRT2
        if do_cols:
            e = out[..., 0:h:2, :w].copy()
            o = out[..., 1:h:2, :w].copy()
            out[..., : h // 2, :w] = (e + o) * INV_SQRT2
            out[..., h // 2: h, :w] = (e - o) * INV_SQRT2
    return out


def coeffs(spec_band, idx, g, freq_bins, time_bins, batch=512):
    """(B, F*T) float32 Haar coefficients of windows `idx`."""
    idx = np.asarray(idx, np.int64)
    out = np.empty((idx.size, freq_bins * time_bins), np.float32)
    for a in range(0, idx.size, batch):
        im = images(spec_band, idx[a:a + batch], g, freq_bins, time_bins)
        out[a:a + batch] = haar2d(im).reshape(im.shape[0], -1).astype(np.float32)
    return out


def mad_sample(n_windows: int, rate: float, seed: int) -> np.ndarray:
    n = max(1, int(round(rate * n_windows)))
    if n >= n_windows:
        return np.arange(n_windows)
    return np.sort(np.random.default_rng(seed).choice(n_windows, size=n, replace=False))


def mad_stats(sample_coeffs):
    c = np.asarray(sample_coeffs, np.float64)
    med = np.median(c, axis=0)
    return med, np.median(np.abs(c - med), axis=0)


def topk_bits(c, median, mad, top_k):
    c = np.atleast_2d(np.asarray(c, np.float64))
    ok = mad > 0
    scores = np.where(ok, (c - median) / np.where(ok, mad, 1.0), 0.0)
    mag = np.abs(scores)
    mag[:, ~ok] = -1.0
    n = c.shape[1]
    # ordering key: descending magnitude, ascending index (stable)
    order = np.argsort(-mag, axis=1, kind="stable")[:, :top_k]
    cols = np.sort(order, axis=1)
    neg = np.take_along_axis(scores, cols, axis=1) < 0
    return (2 * cols + neg).astype(np.uint32)


def fingerprint(samples, sr, params: dict, mad_rate=0.1, mad_seed=0, stats=None):
    """Whole chain. params keys: window_len_s, window_lag_s, freq_bins, time_bins,
    top_k, band_low_hz, band_high_hz, frame_len_s, hop_s.
    Returns dict(bits, median, mad, spec_band, g, sample)."""
    x = np.asarray(samples, np.float64)
    g = geometry(sr, x.size, params["window_len_s"], params["window_lag_s"],
                 params["frame_len_s"], params["hop_s"])
    spec = stft_logpow(x, g["frame"], g["hop"])
    freqs = np.fft.rfftfreq(g["frame"], 1.0 / sr)
    r0, r1 = band_rows(freqs, params.get("band_low_hz"), params.get("band_high_hz"))
    band = np.ascontiguousarray(spec[:, r0:r1])
    F, T = params["freq_bins"], params["time_bins"]
    sample = None
    if stats is None:
        sample = mad_sample(g["n_win"], mad_rate, mad_seed)
        med, mad = mad_stats(coeffs(band, sample, g, F, T))
    else:
        med, mad = stats
    all_idx = np.arange(g["n_win"])
    bits = np.empty((g["n_win"], params["top_k"]), np.uint32)
    for a in range(0, g["n_win"], 2048):
        bits[a:a + 2048] = topk_bits(coeffs(band, all_idx[a:a + 2048], g, F, T),
                                     med, mad, params["top_k"])
    return dict(bits=bits, median=med, mad=mad, spec_band=band, g=g, sample=sample,
                band_rows=(r0, r1))
