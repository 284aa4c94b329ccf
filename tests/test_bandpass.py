"""Zero-phase band-pass (reference ingest.py:55-84 -> scipy.signal.sosfiltfilt,
scipy 1.18.1 in this image) on the GPU: against the reference's own outputs
(tests/golden/bandpass.npz) and, at larger sizes, against scipy directly.
Tolerance: |gpu - ref| <= 1e-9 * max|ref| (float64 recurrences, chunked
carry of the filter state reassociates the arithmetic)."""

import numpy as np
import pytest

from conftest import load_npz

TOL = 1e-9


def _check(got, want):
    got = np.asarray(got)
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= TOL * max(1.0, np.max(np.abs(want)))


def test_golden_oracle_is_scipy():
    """The oracle (scipy sosfiltfilt + butter) reproduces the reference fixtures."""
    from scipy import signal
    for name, c in load_npz("bandpass.npz").items():
        lo, hi, order, sr = c["spec"]
        sos = signal.butter(int(order), [lo, hi], btype="bandpass", fs=sr, output="sos")
        np.testing.assert_array_equal(signal.sosfiltfilt(sos, c["x"]), c["y"])


def test_spec_validation():
    from paper_1803_09835_b200.errors import ParameterError
    from paper_1803_09835_b200.ingest import BandpassSpec
    for lo, hi, order in [(0.0, 5.0, 4), (5.0, 5.0, 4), (5.0, 60.0, 4), (1.0, 5.0, 0)]:
        with pytest.raises(ParameterError):
            BandpassSpec(lo, hi, order).validate(100.0)


@pytest.mark.gpu
def test_bandpass_golden():
    from paper_1803_09835_b200.ingest import BandpassSpec, TimeSeries, bandpass
    for name, c in load_npz("bandpass.npz").items():
        lo, hi, order, sr = c["spec"]
        ts = TimeSeries("ST0", "HHZ", float(sr), 0.0, c["x"])
        out = bandpass(ts, BandpassSpec(float(lo), float(hi), int(order)))
        assert isinstance(out.samples, np.ndarray) and out.samples.dtype == np.float64
        _check(out.samples, c["y"])


@pytest.mark.gpu
def test_bandpass_device_and_long():
    import torch
    from scipy import signal
    from paper_1803_09835_b200.errors import DataError
    from paper_1803_09835_b200.ingest import BandpassSpec, TimeSeries, bandpass
    rng = np.random.default_rng(3)
    for n, lo, hi, order in [(3_000_000, 4.0, 10.0, 4), (777_777, 0.5, 40.0, 6), (70_001, 10.0, 12.0, 3)]:
        x = rng.standard_normal(n)
        sos = signal.butter(order, [lo, hi], btype="bandpass", fs=100.0, output="sos")
        want = signal.sosfiltfilt(sos, x)
        ts = TimeSeries("ST0", "HHZ", 100.0, 0.0, torch.from_numpy(x).cuda())
        out = bandpass(ts, BandpassSpec(lo, hi, order))
        assert out.samples.is_cuda
        _check(out.samples.cpu().numpy(), want)
    with pytest.raises(DataError):
        bandpass(TimeSeries("ST0", "HHZ", 100.0, 0.0, np.zeros(27)), BandpassSpec(4.0, 10.0, 4))
