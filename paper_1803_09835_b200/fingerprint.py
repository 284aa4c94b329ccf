"""Waveform fingerprinting on the B200 — drop-in for reference fingerprint.py.

Chain per overlapping window (reference fingerprint.py:1-17): band-limited
log-power STFT -> area-resampled spectral image -> full 2-D orthonormal Haar
-> MAD-normalised deviation scores -> top-K sign binarisation.
"""

import math
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
