"""Waveform fingerprinting on the B200 — drop-in for reference fingerprint.py.

Chain per overlapping window (reference fingerprint.py:1-17): band-limited
log-power STFT -> area-resampled spectral image -> full 2-D orthonormal Haar
-> MAD-normalised deviation scores -> top-K sign binarisation.
"""

import math
import os
from dataclasses import dataclass, field

import numpy as np

from .errors import CorruptInputError, ParameterError


@dataclass
class StftParams:
    """Spectrogram geometry in seconds (converted per channel sample rate)."""

    frame_len_s: float = 2.0
    hop_s: float = 0.2


@dataclass
class FingerprintParams:
    window_len_s: float = 30.0
    window_lag_s: float = 2.0
    freq_bins: int = 32
    time_bins: int = 128
    top_k: int = 800
    band_low_hz: float | None = None
    band_high_hz: float | None = None
    stft: StftParams = field(default_factory=StftParams)

    @property
    def n_coeffs(self) -> int:
        return self.freq_bins * self.time_bins

    @property
    def d(self) -> int:
        """Fingerprint dimensionality: two sign bits per Haar coefficient."""
        return 2 * self.n_coeffs

    def validate(self) -> None:
        if self.window_lag_s <= 0 or self.window_len_s <= 0:
            raise ParameterError("window length and lag must be positive")
        if self.window_lag_s > self.window_len_s:
            raise ParameterError("window lag must not exceed window length")
        if self.freq_bins < 1 or self.time_bins < 1:
            raise ParameterError("spectral image shape must be at least 1x1")
        if not 1 <= self.top_k <= self.n_coeffs:
            raise ParameterError(f"top_k must be in [1, {self.n_coeffs}], got {self.top_k}")
        if (self.band_low_hz is None) != (self.band_high_hz is None):
            raise ParameterError("band corners must be given together")
        if self.band_low_hz is not None and not 0 < self.band_low_hz < self.band_high_hz:
            raise ParameterError("need 0 < band_low_hz < band_high_hz")
        if self.stft.frame_len_s <= 0 or self.stft.hop_s <= 0:
            raise ParameterError("STFT frame and hop must be positive")


@dataclass
class SpectralImage:
    window_index: int
    start_epoch_s: float
    values: np.ndarray  # (freq_bins, time_bins) float32


@dataclass
class MadStats:
    """Per-coefficient median and median absolute deviation (fingerprint.py:98-119)."""

    median: np.ndarray
    mad: np.ndarray
    rate: float
    seed: int
    n_sampled: int
    n_total: int

    @property
    def eligible(self) -> np.ndarray:
        return self.mad > 0

    @property
    def n_coeffs(self) -> int:
        return self.median.shape[0]


@dataclass
class Fingerprint:
    index: int
    window_start_epoch_s: float
    bits: np.ndarray  # (top_k,) uint32, strictly ascending


@dataclass
class FingerprintSet:
    """Column-oriented batch of fingerprints from one channel (fingerprint.py:490-526).

    `bits` is a host (n, top_k) uint32 array, or a CUDA int32 tensor when the
    chain ran on a device-resident trace."""

    d: int
    top_k: int
    window_len_s: float
    window_lag_s: float
    indices: np.ndarray  # (n,) uint64
    epochs: np.ndarray   # (n,) float64
    bits: np.ndarray     # (n, top_k) uint32
    meta: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return self.indices.shape[0]

    def __getitem__(self, i: int) -> Fingerprint:
        b = self.bits[i]
        if not isinstance(b, np.ndarray):
            b = b.cpu().numpy().view(np.uint32)
        return Fingerprint(int(self.indices[i]), float(self.epochs[i]), b)

    def validate(self) -> None:
        n = len(self)
        bits = self.bits
        if not isinstance(bits, np.ndarray):
            bits = bits.cpu().numpy().view(np.uint32)
        if bits.shape != (n, self.top_k) or self.epochs.shape != (n,):
            raise CorruptInputError("fingerprint arrays are inconsistent")
        if n == 0:
            return
        if int(bits.max()) >= self.d:
            raise CorruptInputError("fingerprint bit index out of range")
        halves = bits >> 1
        if self.top_k > 1 and not (np.diff(halves.astype(np.int64), axis=1) >= 1).all():
            raise CorruptInputError(
                "fingerprint bits must be ascending with one sign bit per coefficient")


def n_windows(ts, params: FingerprintParams) -> int:
    sr = ts.sample_rate_hz
    win = int(round(params.window_len_s * sr))
    lag = max(1, int(round(params.window_lag_s * sr)))
    if ts.n_samples < win:
        return 0
    return (ts.n_samples - win) // lag + 1


def jaccard(bits_a, bits_b) -> float:
    """Jaccard similarity of two sorted bit-index arrays (1.0 if both empty)."""
    a = np.asarray(bits_a)
    b = np.asarray(bits_b)
    if a.size == 0 and b.size == 0:
        return 1.0
    inter = np.intersect1d(a, b, assume_unique=True).size
    return inter / (a.size + b.size - inter)


# ---------------------------------------------------------------------------
# device chain (csrc/qs_fingerprint.cu)

from functools import lru_cache  # noqa: E402

from . import _native as nat  # noqa: E402
from .errors import ConsistencyError, DataError  # noqa: E402

_LOG_EPS = 1e-12


def _stft_geometry(ts, params: FingerprintParams):
    sr = ts.sample_rate_hz
    frame = int(round(params.stft.frame_len_s * sr))
    hop = max(1, int(round(params.stft.hop_s * sr)))
    if frame < 2:
        raise ParameterError("STFT frame shorter than 2 samples")
    if ts.n_samples < frame:
        raise DataError("series shorter than one STFT frame")
    return frame, hop


def _band_rows(freqs: np.ndarray, params: FingerprintParams):
    """Rows inside the band corners (fingerprint.py:166-173)."""
    if params.band_low_hz is None:
        return 0, len(freqs)
    keep = np.flatnonzero((freqs >= params.band_low_hz - 1e-9) & (freqs <= params.band_high_hz + 1e-9))
    if keep.size == 0:
        raise ParameterError("no spectrogram rows inside configured band")
    return int(keep[0]), int(keep[-1]) + 1


@lru_cache(maxsize=64)
def _resize_weights(src: int, dst: int) -> np.ndarray:
    """Area-overlap resampling matrix (dst, src); every row sums to 1 (fingerprint.py:176-186)."""
    r = src / dst
    w = np.zeros((dst, src))
    for i in range(dst):
        lo, hi = i * r, (i + 1) * r
        for j in range(int(math.floor(lo)), min(int(math.ceil(hi)), src)):
            w[i, j] = (min(hi, j + 1) - max(lo, j)) / r
    w.setflags(write=False)
    return w


def _haar_schedule(h: int, w: int):
    steps = []
    while h % 2 == 0 and h > 1 and w % 2 == 0 and w > 1:
        steps.append((h, w, 3))
        h //= 2
        w //= 2
    while w % 2 == 0 and w > 1:
        steps.append((h, w, 1))
        w //= 2
    while h % 2 == 0 and h > 1:
        steps.append((h, w, 2))
        h //= 2
    return steps


def _csr(mat: np.ndarray):
    rows, cols = np.nonzero(mat)
    off = np.zeros(mat.shape[0] + 1, np.int32)
    np.add.at(off, rows + 1, 1)
    return np.cumsum(off).astype(np.int32), cols.astype(np.int32), mat[rows, cols].astype(np.float64)


def _to_host_pinned(t) -> np.ndarray:
    """D2H into pinned host memory (the returned array keeps it alive)."""
    buf = nat.torch().empty(t.shape, dtype=t.dtype, pin_memory=True)
    buf.copy_(t)
    return buf.numpy()


class _Chain:
    """Device state of one channel: samples, band spectrogram and the
    window-kernel tables (geometry of fingerprint.py:198-243)."""

    def __init__(self, ts, params: FingerprintParams, full_band: bool = False,
                 windows: bool = False):
        params.validate()
        self.torch = torch = nat.torch()
        self.params = params
        sr = ts.sample_rate_hz
        self.frame, self.hop = _stft_geometry(ts, params)
        self.win = int(round(params.window_len_s * sr))
        self.lag = max(1, int(round(params.window_lag_s * sr)))
        self.n_win = n_windows(ts, params)
        self.n_cols = (ts.n_samples - self.frame) // self.hop + 1
        self.freqs = np.fft.rfftfreq(self.frame, 1.0 / sr)
        self.r0, self.r1 = (0, len(self.freqs)) if full_band else _band_rows(self.freqs, params)
        self.nb = self.r1 - self.r0
        taper = np.hanning(self.frame)
        j = np.arange(self.frame)
        k = np.arange(self.r0, self.r1)[:, None]
        ang = 2.0 * np.pi * ((k * j) % self.frame) / self.frame
        tw = np.stack([taper * np.cos(ang), -taper * np.sin(ang)], axis=-1)
        self.tw = torch.from_numpy(np.ascontiguousarray(tw)).cuda()
        self.band = torch.empty((max(self.n_cols, 1), self.nb), dtype=torch.float32, device="cuda")
        if windows:
            # the window tables go up before the STFT launch: their pageable
            # H2D copies would otherwise wait for it, and the host work that
            # follows (the MAD sample draw) would no longer overlap it
            self.prepare_windows()
        x = ts.samples
        n_samples = ts.n_samples
        frame, hop, nb = self.frame, self.hop, self.nb

        def stft(xd, c_lo, c_hi):
            # columns [c_lo, c_hi) only read samples [c_lo hop, (c_hi - 1) hop + frame)
            if c_hi <= c_lo:
                return
            es = xd.element_size()
            nat.call("qs_fp_band_stft", nat.ctypes.c_void_p(xd.data_ptr() + c_lo * hop * es),
                     int(xd.dtype == torch.float32), n_samples - c_lo * hop, frame, hop,
                     c_hi - c_lo, nb, nat.ptr(self.tw),
                     nat.ctypes.c_void_p(self.band.data_ptr() + c_lo * nb * 4), nat.stream())

        if nat.is_device_tensor(x):
            xd = x.contiguous()
            if xd.dtype not in (torch.float32, torch.float64):
                xd = xd.to(torch.float64)
            stft(xd, 0, self.n_cols)
        else:
            # host trace: the STFT of every column whose samples have landed runs
            # while the later chunks are still being copied
            from .lsh_search import _host_pinned, _to_device_staged
            holder, state = [], [0]

            def on_chunk(done):
                c_hi = min(self.n_cols, (done - frame) // hop + 1) if done >= frame else 0
                stft(holder[0], state[0], c_hi)
                state[0] = max(state[0], c_hi)

            arr = np.ascontiguousarray(x, dtype=np.float64)
            xd = None
            if not _host_pinned(arr) and os.environ.get("QS_H2D_NARROW", "1") != "0":
                # a float32 recording coerced to float64 (ingest.py:36) goes up as
                # float32 — half the staging writes and DMA bytes; the chain widens
                # float32 samples exactly.  Any inexact sample: float64 instead.
                x32 = torch.empty(arr.shape, dtype=torch.float32, device="cuda")
                holder.append(x32)
                xd = _to_device_staged(arr, on_chunk=on_chunk, out=x32, narrow_f32=True)
                if xd is None:
                    holder.clear()
                    state[0] = 0
                    del x32
            if xd is None:
                xd = torch.empty(arr.shape, dtype=torch.float64, device="cuda")
                holder.append(xd)
                xd = _to_device_staged(arr, on_chunk=on_chunk, out=xd)
            stft(xd, state[0], self.n_cols)
        self.x = xd

    def prepare_windows(self):
        params, torch = self.params, self.torch
        if self.n_win == 0:
            raise DataError("series shorter than one fingerprint window")
        if self.win < self.frame:
            raise ParameterError("fingerprint window shorter than one STFT frame")
        probe = np.arange(min(self.n_win, self.hop * 2 + 1), dtype=np.int64) * self.lag
        c0 = -(-probe // self.hop)
        c1 = (probe + self.win - self.frame) // self.hop + 1
        widths = c1 - c0
        if widths.min() < 1:
            raise ParameterError("window contains no complete STFT frame")
        self.wmin, self.wmax = int(widths.min()), int(widths.max())
        F, T = params.freq_bins, params.time_bins
        wf_off, wf_idx, wf_val = _csr(_resize_weights(self.nb, F))
        offs, idxs, vals, base = [], [], [], 0
        for width in range(self.wmin, self.wmax + 1):
            o, i, v = _csr(_resize_weights(width, T))
            offs.append(o + base)
            idxs.append(i)
            vals.append(v)
            base += len(i)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        self.wf = (dev(wf_off), dev(wf_idx), dev(wf_val))
        self.wt = (dev(np.concatenate(offs)), dev(np.concatenate(idxs)), dev(np.concatenate(vals)))
        sched = _haar_schedule(F, T)
        self.n_levels = len(sched)
        self.sched = dev(np.array(sched, np.int32).reshape(-1) if sched else np.zeros(3, np.int32))
        self.flags = torch.zeros(1, dtype=torch.int32, device="cuda")

    def windows(self, mode, out, widx=None, win0=0, n=None, med=None, mad=None, top_k=0):
        n = self.n_win if n is None else n
        F, T = self.params.freq_bins, self.params.time_bins
        nat.call("qs_fp_windows", nat.ptr(self.band), self.n_cols, self.nb, nat.ptr(widx), win0, n,
                 self.lag, self.win, self.frame, self.hop, nat.ptr(self.wf[0]), nat.ptr(self.wf[1]),
                 nat.ptr(self.wf[2]), nat.ptr(self.wt[0]), nat.ptr(self.wt[1]), nat.ptr(self.wt[2]),
                 self.wmin, self.wmax, F, T, nat.ptr(self.sched), self.n_levels, mode, nat.ptr(med),
                 nat.ptr(mad), top_k, nat.ptr(out), nat.ptr(self.flags), nat.stream())

    def check_finite(self):
        if int(self.flags.item()) & 1:
            raise DataError("non-finite Haar coefficient")


def spectrogram(ts, params: FingerprintParams | None = None):
    """Full-series log-power spectrogram (fingerprint.py:154-163).

    Returns (freqs_hz, column_epochs_s, logpow) with logpow (n_freqs, n_cols) float32."""
    params = params or FingerprintParams()
    ch = _Chain(ts, params, full_band=True)
    times = ts.start_epoch_s + np.arange(ch.n_cols) * (ch.hop / ts.sample_rate_hz)
    return ch.freqs, times, ch.band[: ch.n_cols].t().contiguous().cpu().numpy()


def _window_indices(chain, indices):
    if indices is None:
        return np.arange(chain.n_win, dtype=np.int64)
    idx = np.asarray(indices, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= chain.n_win):
        raise ParameterError("window index out of range")
    return idx


def _iter_batches(ts, params, indices, batch, mode):
    params.validate()
    ch = _Chain(ts, params)
    ch.prepare_windows()
    idx = _window_indices(ch, indices)
    torch = ch.torch
    F, T = params.freq_bins, params.time_bins
    for b0 in range(0, idx.size, batch):
        sel = idx[b0: b0 + batch]
        widx = torch.from_numpy(sel).cuda()
        shape = (sel.size, F, T) if mode == 0 else (sel.size, F * T)
        out = torch.empty(shape, dtype=torch.float32, device="cuda")
        ch.windows(mode, out, widx=widx, n=sel.size)
        epochs = ts.start_epoch_s + sel * params.window_lag_s
        yield sel, epochs, out.cpu().numpy()


def iter_image_batches(ts, params: FingerprintParams, indices=None, batch: int = 512):
    """Yield (window_indices, start_epochs, images (B, F, T) float32) (fingerprint.py:198-243)."""
    yield from _iter_batches(ts, params, indices, batch, 0)


def iter_coeff_batches(ts, params: FingerprintParams, indices=None, batch: int = 512):
    """Yield (window_indices, epochs, coeffs (B, F*T) float32) (fingerprint.py:326-335)."""
    yield from _iter_batches(ts, params, indices, batch, 1)


def compute_spectral_images(ts, params: FingerprintParams):
    """Generator of SpectralImage over all windows of a channel (fingerprint.py:246-250)."""
    for idx, epochs, images in iter_image_batches(ts, params):
        for i, e, v in zip(idx, epochs, images):
            yield SpectralImage(int(i), float(e), v)


def _haar_call(a, inverse):
    torch = nat.torch()
    arr = np.array(a, dtype=np.float64, copy=True)
    if arr.ndim < 2:
        raise ParameterError("haar2d needs at least a 2-D array" if not inverse
                             else "ihaar2d needs at least a 2-D array")
    H, W = arr.shape[-2:]
    sched = _haar_schedule(H, W)
    if not sched or arr.size == 0:
        return arr
    dev = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    sd = torch.from_numpy(np.array(sched, np.int32).reshape(-1)).cuda()
    nat.call("qs_fp_haar2d", nat.ptr(dev), arr.size // (H * W), H, W, nat.ptr(sd), len(sched),
             int(inverse), nat.stream())
    return dev.cpu().numpy().reshape(arr.shape)


def haar2d(a) -> np.ndarray:
    """Full orthonormal 2-D Haar decomposition of (..., H, W) arrays (fingerprint.py:271-300)."""
    return _haar_call(a, False)


def ihaar2d(a) -> np.ndarray:
    """Inverse of haar2d (fingerprint.py:303-323)."""
    return _haar_call(a, True)


def _mad_sample(rate, seed, total):
    """The sampled window indices, drawn by the reference's own numpy RNG call
    (fingerprint.py:352-357)."""
    n_sample = max(1, int(round(rate * total)))
    if n_sample >= total:
        return np.arange(total), total
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(total, size=n_sample, replace=False)), n_sample


def _mad_from_chain(ch, params, rate, seed, total, sample=None):
    torch = ch.torch
    sample, n_sample = sample.result() if sample is not None else _mad_sample(rate, seed, total)
    n_coeffs = params.n_coeffs
    # one coefficient row per sampled window (coalesced stores), then one
    # transpose into the per-coefficient columns the order statistics read
    rows = torch.empty((n_sample, n_coeffs), dtype=torch.float32, device="cuda")
    ch.windows(1, rows, widx=torch.from_numpy(sample.astype(np.int64)).cuda(), n=n_sample)
    cols = torch.empty((n_coeffs, n_sample), dtype=torch.float32, device="cuda")
    nat.call("qs_fp_transpose_f32", nat.ptr(rows), n_sample, n_coeffs, nat.ptr(cols), nat.stream())
    del rows
    med = torch.empty(n_coeffs, dtype=torch.float64, device="cuda")
    mad = torch.empty(n_coeffs, dtype=torch.float64, device="cuda")
    ws = torch.empty(2 * n_coeffs, dtype=torch.float64, device="cuda")
    nat.call("qs_fp_mad", nat.ptr(cols), n_coeffs, n_sample, nat.ptr(med), nat.ptr(mad), nat.ptr(ws),
             nat.stream())
    return med, mad, n_sample


def estimate_mad(ts, params: FingerprintParams, rate: float = 0.1, seed: int = 0,
                 batch: int = 512) -> MadStats:
    """Median and MAD per Haar coefficient from a random sample of windows
    (fingerprint.py:341-389); the sample is drawn by the reference's own numpy
    RNG call, the coefficients and order statistics are computed on the GPU."""
    params.validate()
    if not 0 < rate <= 1:
        raise ParameterError(f"sampling rate must be in (0, 1], got {rate}")
    total = n_windows(ts, params)
    if total == 0:
        raise DataError("series shorter than one fingerprint window")
    ch = _Chain(ts, params, windows=True)
    med, mad, n_sample = _mad_from_chain(ch, params, rate, seed, total)
    return MadStats(median=med.cpu().numpy(), mad=mad.cpu().numpy(), rate=float(rate),
                    seed=int(seed), n_sampled=int(n_sample), n_total=int(total))


def normalize(coeffs, stats: MadStats) -> np.ndarray:
    """Deviation scores v' = (v - median) / MAD in float64; zero-MAD columns
    give 0 (fingerprint.py:425-430).  float32 rows (the chain's coefficients)
    are read as float32, anything else as float64 — the reference's
    np.asarray(coeffs, dtype=np.float64) either way."""
    torch = nat.torch()
    c = np.asarray(coeffs)
    is_f64 = c.dtype != np.float32
    c = np.ascontiguousarray(c, dtype=np.float64 if is_f64 else np.float32)
    shape = c.shape
    n = shape[-1] if c.ndim else 1
    if n != stats.n_coeffs:
        raise ParameterError("coefficient count does not match MAD stats")
    cd = torch.from_numpy(c.reshape(-1, n)).cuda()
    med = torch.from_numpy(np.ascontiguousarray(stats.median, np.float64)).cuda()
    mad = torch.from_numpy(np.ascontiguousarray(stats.mad, np.float64)).cuda()
    out = torch.empty(cd.shape, dtype=torch.float64, device="cuda")
    nat.call("qs_fp_normalize", nat.ptr(cd), int(is_f64), cd.shape[0], n, nat.ptr(med),
             nat.ptr(mad), nat.ptr(out), nat.stream())
    return out.cpu().numpy().reshape(shape)


def topk_bits(coeffs, stats: MadStats, top_k: int) -> np.ndarray:
    """Sign-encoded bit indices of the top_k most anomalous coefficients
    (fingerprint.py:433-466): (B, top_k) uint32, ascending per row."""
    torch = nat.torch()
    c = np.atleast_2d(np.asarray(coeffs, dtype=np.float64))
    n = c.shape[1]
    if n != stats.n_coeffs:
        raise ParameterError("coefficient count does not match MAD stats")
    n_eligible = int(stats.eligible.sum())
    if not 1 <= top_k <= n:
        raise ParameterError(f"top_k must be in [1, {n}]")
    if top_k > n_eligible:
        raise ParameterError(f"top_k={top_k} exceeds {n_eligible} coefficients with nonzero MAD")
    if not np.isfinite(c).all():
        raise DataError("non-finite Haar coefficient")
    cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
    med = torch.from_numpy(np.ascontiguousarray(stats.median, np.float64)).cuda()
    mad = torch.from_numpy(np.ascontiguousarray(stats.mad, np.float64)).cuda()
    out = torch.empty((c.shape[0], top_k), dtype=torch.int32, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.call("qs_fp_topk_bits", nat.ptr(cd), 1, c.shape[0], n, nat.ptr(med), nat.ptr(mad), top_k,
             nat.ptr(out), nat.ptr(flags), nat.stream())
    return out.cpu().numpy().view(np.uint32)


def _index_columns(ts, params, total):
    # window index and start epoch per fingerprint (fingerprint.py:612-613)
    indices = np.arange(total, dtype=np.uint64)
    epochs = ts.start_epoch_s + np.arange(total) * params.window_lag_s
    return indices, epochs


def fingerprint_series(ts, params: FingerprintParams, stats: MadStats | None = None,
                       mad_rate: float = 0.1, mad_seed: int = 0,
                       batch: int = 512) -> tuple[FingerprintSet, MadStats]:
    """Fingerprint every window of a channel (fingerprint.py:581-623).

    One STFT of the series serves both the MAD sample and the main pass.
    Host traces give host FingerprintSet.bits; a CUDA trace gives CUDA bits."""
    params.validate()
    torch = nat.torch()
    total = n_windows(ts, params)
    if total == 0:
        raise DataError("series shorter than one fingerprint window")
    draw = None
    if stats is None:
        if not 0 < mad_rate <= 1:
            raise ParameterError(f"sampling rate must be in (0, 1], got {mad_rate}")
        # the sample draw (~50 ms of host work at 8e6 windows) runs beside the
        # trace upload and the STFT instead of after them
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(1) as ex:
            draw = ex.submit(_mad_sample, mad_rate, mad_seed, total)
            ch = _Chain(ts, params, windows=True)
    else:
        ch = _Chain(ts, params, windows=True)
    if stats is None:
        med, mad, n_sample = _mad_from_chain(ch, params, mad_rate, mad_seed, total, sample=draw)
        stats = MadStats(median=med.cpu().numpy(), mad=mad.cpu().numpy(), rate=float(mad_rate),
                         seed=int(mad_seed), n_sampled=int(n_sample), n_total=int(total))
    else:
        med = torch.from_numpy(np.ascontiguousarray(stats.median, np.float64)).cuda()
        mad = torch.from_numpy(np.ascontiguousarray(stats.mad, np.float64)).cuda()
    if stats.n_coeffs != params.n_coeffs:
        raise ConsistencyError("MAD stats shape does not match params")
    n_eligible = int(stats.eligible.sum())
    if params.top_k > n_eligible:
        raise ParameterError(f"top_k={params.top_k} exceeds {n_eligible} coefficients with nonzero MAD")
    bits = torch.empty((total, params.top_k), dtype=torch.int32, device="cuda")
    # the host-side index/epoch columns are filled while the main pass runs
    if nat.is_device_tensor(ts.samples):
        ch.windows(3, bits, win0=0, n=total, med=med, mad=mad, top_k=params.top_k)
        indices, epochs = _index_columns(ts, params, total)
        ch.check_finite()
        out_bits = bits
    else:
        # host trace: the main pass runs in window chunks and each chunk's bits
        # go to pinned host memory on a copy stream while the next chunk
        # computes (the D2H overlaps the kernel instead of following it)
        host = torch.empty((total, params.top_k), dtype=torch.int32, pin_memory=True)
        compute = torch.cuda.current_stream()
        copy = torch.cuda.Stream()
        nchunk = 8 if total >= 8 * 4096 else 1
        step = -(-total // nchunk)
        for c0 in range(0, total, step):
            c1 = min(total, c0 + step)
            ch.windows(3, bits[c0:c1], win0=c0, n=c1 - c0, med=med, mad=mad, top_k=params.top_k)
            ev = torch.cuda.Event()
            ev.record(compute)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                host[c0:c1].copy_(bits[c0:c1], non_blocking=True)
        bits.record_stream(copy)
        indices, epochs = _index_columns(ts, params, total)
        copy.synchronize()
        ch.check_finite()
        out_bits = host.numpy().view(np.uint32)
    fps = FingerprintSet(d=params.d, top_k=params.top_k, window_len_s=params.window_len_s,
                         window_lag_s=params.window_lag_s, indices=indices, epochs=epochs,
                         bits=out_bits,
                         meta={"station": ts.station_id, "channel": ts.channel_id,
                               "sample_rate_hz": ts.sample_rate_hz,
                               "start_epoch_s": ts.start_epoch_s})
    return fps, stats


# ---------------------------------------------------------------------------
# fingerprint and MAD files (fingerprint.py:392-417, 529-578)

import os  # noqa: E402

from . import container as _container  # noqa: E402
from . import hostio  # noqa: E402
from .errors import ConsistencyError as _ConsistencyError  # noqa: E402

FP_MAGIC = b"QSFP0001"
MAD_MAGIC = b"QSMD0001"
_FP_KIND = "fingerprint"
_MAD_KIND = "mad-stats"
_FP_KEYS = ("d", "top_k", "window_len_s", "window_lag_s")


def _fp_record_dtype(top_k: int):
    return np.dtype([("index", "<u8"), ("epoch", "<f8"), ("bits", "<u4", (top_k,))])


def _validate_device(fps) -> None:
    torch = nat.torch()
    n = len(fps)
    b = fps.bits
    if tuple(b.shape) != (n, fps.top_k) or fps.epochs.shape != (n,):
        raise CorruptInputError("fingerprint arrays are inconsistent")
    if n == 0:
        return
    if int(b.max().item()) >= fps.d or int(b.min().item()) < 0:
        raise CorruptInputError("fingerprint bit index out of range")
    if fps.top_k > 1 and not bool(torch.all((b[:, 1:] >> 1) - (b[:, :-1] >> 1) >= 1).item()):
        raise CorruptInputError(
            "fingerprint bits must be ascending with one sign bit per coefficient")


def write_fingerprint_file(path, fps: FingerprintSet, extra: dict | None = None) -> None:
    """Binary .fp file (fingerprint.py:529-551), byte-identical to the reference's.
    CUDA bits are packed into records on the device and streamed to the file."""
    device = nat.is_device_tensor(fps.bits)
    if device:
        _validate_device(fps)
    else:
        fps.validate()
    header = {"d": fps.d, "top_k": fps.top_k, "window_len_s": fps.window_len_s,
              "window_lag_s": fps.window_lag_s}
    header.update(fps.meta)
    if extra:
        header.update(extra)
    n = len(fps)
    with open(path, "wb") as f:
        _container.write_preamble(f, FP_MAGIC, header, count=n)
        if not device:
            rec = np.zeros(n, dtype=_fp_record_dtype(fps.top_k))
            rec["index"] = fps.indices
            rec["epoch"] = fps.epochs
            rec["bits"] = fps.bits
            rec.tofile(f)
            return
        torch = nat.torch()
        dev = fps.bits.device
        idx = torch.from_numpy(np.ascontiguousarray(fps.indices, dtype=np.uint64).view(np.int64)).to(dev)
        ep = torch.from_numpy(np.ascontiguousarray(fps.epochs, dtype=np.float64)).to(dev)
        bits = fps.bits.contiguous()
        out = torch.empty(n * (16 + 4 * fps.top_k), dtype=torch.uint8, device=dev)
        nat.call("qs_fp_pack_records", nat.ptr(idx), nat.ptr(ep), nat.ptr(bits), n, fps.top_k,
                 nat.ptr(out), nat.stream())
        hostio.write_device_bytes(f, out)


def read_fingerprint_file(path, device: bool = False) -> FingerprintSet:
    """Read a .fp file (fingerprint.py:554-578).  device=True returns CUDA
    bits (int32), unpacked from the records on the GPU."""
    with open(path, "rb") as f:
        header, count, off = _container.read_preamble(f, FP_MAGIC, _FP_KIND)
        for key in _FP_KEYS:
            if key not in header:
                raise _ConsistencyError(f"fingerprint header missing '{key}'")
        top_k = int(header["top_k"])
        dtype = _fp_record_dtype(top_k)
        size = os.fstat(f.fileno()).st_size
        _container.check_payload_size(size, off, count, dtype.itemsize, _FP_KIND)
        if device:
            torch = nat.torch()
            raw = hostio.read_to_device(f, count * dtype.itemsize)
            idx = torch.empty(count, dtype=torch.int64, device="cuda")
            ep = torch.empty(count, dtype=torch.float64, device="cuda")
            bits = torch.empty((count, top_k), dtype=torch.int32, device="cuda")
            nat.call("qs_fp_unpack_records", nat.ptr(raw), count, top_k, nat.ptr(idx),
                     nat.ptr(ep), nat.ptr(bits), nat.stream())
            del raw
            indices = idx.cpu().numpy().view(np.uint64)
            epochs = ep.cpu().numpy()
        else:
            rec = np.fromfile(f, dtype=dtype, count=count)
            indices = rec["index"].astype(np.uint64)
            epochs = rec["epoch"].astype(np.float64)
            bits = np.ascontiguousarray(rec["bits"])
    meta = {k: v for k, v in header.items() if k not in _FP_KEYS}
    fps = FingerprintSet(d=int(header["d"]), top_k=top_k,
                         window_len_s=float(header["window_len_s"]),
                         window_lag_s=float(header["window_lag_s"]),
                         indices=indices, epochs=epochs, bits=bits, meta=meta)
    if device:
        _validate_device(fps)
    else:
        fps.validate()
    return fps


def write_mad_file(path, stats: MadStats, extra: dict | None = None) -> None:
    """Binary MAD statistics (fingerprint.py:392-404): f64 medians then f64 MADs."""
    header = {"rate": stats.rate, "seed": stats.seed, "n_sampled": stats.n_sampled,
              "n_total": stats.n_total}
    if extra:
        header.update(extra)
    with open(path, "wb") as f:
        _container.write_preamble(f, MAD_MAGIC, header, count=stats.n_coeffs)
        f.write(np.asarray(stats.median).astype("<f8").tobytes())
        f.write(np.asarray(stats.mad).astype("<f8").tobytes())


def read_mad_file(path):
    """-> (MadStats, header) (fingerprint.py:407-417)."""
    with open(path, "rb") as f:
        header, count, off = _container.read_preamble(f, MAD_MAGIC, _MAD_KIND)
        size = os.fstat(f.fileno()).st_size
        _container.check_payload_size(size, off, count, 16, _MAD_KIND)
        median = np.fromfile(f, dtype="<f8", count=count)
        mad = np.fromfile(f, dtype="<f8", count=count)
    stats = MadStats(median=median, mad=mad, rate=float(header.get("rate", 1.0)),
                     seed=int(header.get("seed", 0)),
                     n_sampled=int(header.get("n_sampled", count)),
                     n_total=int(header.get("n_total", count)))
    return stats, header
