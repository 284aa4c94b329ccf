"""Input container of the hot path (reference ingest.py:25-52).

Only `TimeSeries` is on the path; data generation, file IO and band-pass
filtering of the reference's ingest module are outside this drop-in
(SURVEY.md §2 row 9, §8f).
"""

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError


@dataclass
class TimeSeries:
    """A single channel of evenly sampled data (samples coerced to float64,
    as reference ingest.py:36)."""

    station_id: str
    channel_id: str
    sample_rate_hz: float
    start_epoch_s: float
    samples: np.ndarray

    def __post_init__(self):
        if not _is_device_tensor(self.samples):
            self.samples = np.asarray(self.samples, dtype=np.float64)
            if self.samples.ndim != 1:
                raise ParameterError("samples must be 1-D")
        elif self.samples.dim() != 1:
            raise ParameterError("samples must be 1-D")
        if not self.sample_rate_hz > 0:
            raise ParameterError("sample_rate_hz must be positive")

    @property
    def n_samples(self) -> int:
        return int(self.samples.shape[0])

    @property
    def duration_s(self) -> float:
        return self.n_samples / self.sample_rate_hz

    @property
    def end_epoch_s(self) -> float:
        return self.start_epoch_s + self.duration_s


def _is_device_tensor(x) -> bool:
    """A torch CUDA tensor is accepted as-is (device-resident trace; float32 or
    float64 — a float32 trace widens to float64 exactly, so the chain sees the
    same values as the reference's float64 coercion)."""
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)


# ---------------------------------------------------------------------------
# zero-phase band-pass (reference ingest.py:55-84), computed on the GPU

@dataclass
class BandpassSpec:
    low_hz: float
    high_hz: float
    order: int = 4

    def validate(self, sample_rate_hz: float) -> None:
        nyq = sample_rate_hz / 2.0
        if not 0 < self.low_hz < self.high_hz < nyq:
            raise ParameterError(f"need 0 < low < high < Nyquist ({nyq} Hz), "
                                 f"got [{self.low_hz}, {self.high_hz}]")
        if self.order < 1:
            raise ParameterError("filter order must be >= 1")


def bandpass(ts: TimeSeries, spec: BandpassSpec) -> TimeSeries:
    """Forward-backward Butterworth band-pass (zero phase distortion).

    Same filter as the reference: scipy's Butterworth second-order sections
    and steady-state initial conditions (tiny host computations), then the
    odd-extended forward/backward cascade on the device
    (csrc/qs_filter.cu).  Host samples in -> host float64 out; CUDA samples in
    -> CUDA float64 out."""
    from scipy import signal

    from . import _native as nat
    from .errors import DataError
    spec.validate(ts.sample_rate_hz)
    sos = np.ascontiguousarray(signal.butter(spec.order, [spec.low_hz, spec.high_hz],
                                             btype="bandpass", fs=ts.sample_rate_hz,
                                             output="sos"), dtype=np.float64)
    zi = np.ascontiguousarray(signal.sosfilt_zi(sos), dtype=np.float64)
    S = sos.shape[0]
    ntaps = 2 * S + 1 - min(int((sos[:, 2] == 0).sum()), int((sos[:, 5] == 0).sum()))
    pad = 3 * ntaps
    n = ts.n_samples
    if n <= pad:
        raise DataError(f"series too short to filter: the length of the input vector x must be "
                        f"greater than padlen, which is {pad}.")
    torch = nat.torch()
    on_device = _is_device_tensor(ts.samples)
    if on_device:
        x = ts.samples.to(torch.float64).contiguous()
    else:
        from .lsh_search import _to_device_staged
        x = _to_device_staged(np.ascontiguousarray(ts.samples, dtype=np.float64))
    out = torch.empty(n, dtype=torch.float64, device=x.device)
    lib = nat.lib()
    ws = torch.empty(lib.qs_sosfiltfilt_ws_bytes(n, pad), dtype=torch.uint8, device=x.device)
    nat.call("qs_sosfiltfilt", nat.ptr(x), n, sos.ctypes.data_as(nat.ctypes.c_void_p), S,
             zi.ctypes.data_as(nat.ctypes.c_void_p), pad, nat.ptr(out), nat.ptr(ws), ws.numel(),
             nat.stream())
    samples = out if on_device else out.cpu().numpy()
    return TimeSeries(ts.station_id, ts.channel_id, ts.sample_rate_hz, ts.start_epoch_s, samples)
