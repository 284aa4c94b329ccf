"""The one-call C entry qs_fingerprint_chain through ctypes, as a non-Python
caller binds it: caller workspace, MAD sample indices or
given median/MAD, bits out.  Must equal the reference's golden outputs."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _params_c(nat, p):
    return nat.FpParamsC(p["window_len_s"], p["window_lag_s"], p["freq_bins"], p["time_bins"],
                         p["top_k"], p.get("band_low_hz") or 0.0, p.get("band_high_hz") or 0.0,
                         p["frame_len_s"], p["hop_s"])


def capi_chain(x, sr, p, mad_rate=0.1, mad_seed=0, stats=None):
    import torch
    from paper_1803_09835_b200 import _native as nat
    lib = nat.lib()
    pc = _params_c(nat, p)
    nw = ctypes.c_uint64(0)
    nat.check(lib.qs_fp_n_windows(x.size, sr, ctypes.byref(pc), ctypes.byref(nw)))
    nw = nw.value
    nc = p["freq_bins"] * p["time_bins"]
    if stats is None:
        ns = max(1, int(round(mad_rate * nw)))
        sample = (np.arange(nw) if ns >= nw else
                  np.sort(np.random.default_rng(mad_seed).choice(nw, size=ns, replace=False)))
        sd = torch.from_numpy(sample.astype(np.int64)).cuda()
        med = torch.empty(nc, dtype=torch.float64, device="cuda")
        mad = torch.empty(nc, dtype=torch.float64, device="cuda")
    else:
        sd, ns = None, 0
        med = torch.from_numpy(np.ascontiguousarray(stats[0], np.float64)).cuda()
        mad = torch.from_numpy(np.ascontiguousarray(stats[1], np.float64)).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    is_f32 = int(x.dtype == np.float32)
    wsb = lib.qs_fingerprint_chain_ws_bytes(x.size, sr, ctypes.byref(pc), ns)
    ws = torch.empty(max(1, wsb), dtype=torch.uint8, device="cuda")
    bits = torch.empty((nw, p["top_k"]), dtype=torch.int32, device="cuda")
    out_nw = ctypes.c_uint64(0)
    rc = lib.qs_fingerprint_chain(nat.ptr(xd), is_f32, x.size, sr, ctypes.byref(pc), nat.ptr(sd), ns,
                                  nat.ptr(med), nat.ptr(mad), nat.ptr(bits), ctypes.byref(out_nw),
                                  nat.ptr(ws), wsb, nat.stream())
    nat.check(rc, "qs_fingerprint_chain")
    assert out_nw.value == nw
    return bits.cpu().numpy().view(np.uint32), med.cpu().numpy(), mad.cpu().numpy()


def test_capi_chain_golden(golden_fingerprint):
    from paper_1803_09835_b200 import workloads
    case = golden_fingerprint["cfg0_half_hour"]
    bits, med, mad = capi_chain(case["samples"], 100.0, workloads.CFG0_PARAMS)
    np.testing.assert_allclose(med, case["median"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(mad, case["mad"], rtol=1e-12, atol=0)
    assert np.array_equal(bits, case["bits"])
    bits2, _, _ = capi_chain(case["samples"], 100.0, workloads.CFG0_PARAMS,
                             stats=(case["median"], case["mad"]))
    assert np.array_equal(bits2, case["bits"])


def test_capi_chain_full_band_vs_python():
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200.ingest import TimeSeries
    rng = np.random.default_rng(4)
    x = rng.standard_normal(30_000)
    p = dict(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12, top_k=24,
             band_low_hz=None, band_high_hz=None, frame_len_s=0.5, hop_s=0.05)
    params = fp.FingerprintParams(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12,
                                  top_k=24, stft=fp.StftParams(0.5, 0.05))
    fps, st = fp.fingerprint_series(TimeSeries("S", "C", 100.0, 0.0, x), params, mad_rate=1.0)
    bits, med, mad = capi_chain(x, 100.0, p, mad_rate=1.0)
    np.testing.assert_allclose(med, st.median, rtol=1e-12, atol=0)
    assert np.array_equal(bits, fps.bits)


def test_capi_chain_errors():
    import torch
    from paper_1803_09835_b200 import _native as nat
    from paper_1803_09835_b200 import workloads
    lib = nat.lib()
    pc = _params_c(nat, workloads.CFG0_PARAMS)
    nw = ctypes.c_uint64(0)
    assert lib.qs_fp_n_windows(500, 100.0, ctypes.byref(pc), ctypes.byref(nw)) == nat.QS_ERR_DATA
    bad = _params_c(nat, dict(workloads.CFG0_PARAMS, top_k=0))
    assert lib.qs_fp_n_windows(10_000, 100.0, ctypes.byref(bad), ctypes.byref(nw)) == nat.QS_ERR_ARG
    # top_k above the eligible (nonzero-MAD) coefficients -> ParameterError
    x = np.random.default_rng(1).standard_normal(5_000)
    p = dict(window_len_s=3.0, window_lag_s=0.5, freq_bins=4, time_bins=4, top_k=10,
             band_low_hz=None, band_high_hz=None, frame_len_s=0.5, hop_s=0.05)
    mad = np.zeros(16)
    mad[:5] = 1.0
    from paper_1803_09835_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        capi_chain(x, 100.0, p, stats=(np.zeros(16), mad))
    torch.cuda.synchronize()
