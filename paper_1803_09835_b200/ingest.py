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
