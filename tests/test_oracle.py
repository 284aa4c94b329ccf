"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The KATs re-check the reference's own frozen values (reference
tests/test_minmax_hash.py:53-71) as captured by tests/golden/make_golden.py.
"""

import numpy as np
import pytest

import oracle
from oracle import fingerprint as ofp
from oracle import minmax as omm
from oracle import search as osr

# the reference's frozen regression values (tests/test_minmax_hash.py:53-71)
FMIX_FROZEN = {0x0: 0x0, 0x1: 0xB456BCFC34C2CB2C, 0xDEADBEEF: 0xD24BD59F862A1DAC,
               0xFFFFFFFFFFFFFFFF: 0x64B5720B4B825F21}
HASH_FROZEN = {(0, 0): 0x9CA066F1A4AB2EEA, (1, 0): 0xD30B054265133DD7,
               (0, 1): 0x25B775FAECA8F520, (12345, 67890): 0x8761E9A53AFF2D33}
COMBINE_FROZEN = {(0,): 0x9E3779B97F4A7C15, (1, 2): 0xC3A9E841E0AB654D,
                  (5, 9, 3): 0x16157B14B0332EF2}
SIG_FROZEN = [0xEC797BCAD18E750C, 0x168878915D63A8D2, 0x684B9C6319F40596]


def test_kat_frozen_c_and_numpy(golden_kat):
    lib = oracle.c_lib()
    for x, want in FMIX_FROZEN.items():
        assert lib.qso_fmix64(x) == want
        assert int(omm.fmix64(np.uint64(x))) == want
    for (x, s), want in HASH_FROZEN.items():
        assert lib.qso_hash(x, s) == want
        assert int(omm.hash_values(np.array([x]), s)[0]) == want
    for ws, want in COMBINE_FROZEN.items():
        assert omm.combine(ws) == want
        arr = np.array(ws, np.uint64)
        assert lib.qso_combine(arr.ctypes.data, arr.size) == want
    for x, want in golden_kat["fmix64"].items():
        assert lib.qso_fmix64(int(x, 16)) == int(want, 16)
    for xs, want in golden_kat["hash"].items():
        x, s = (int(v) for v in xs.split(","))
        assert lib.qso_hash(x, s) == int(want, 16)
    for ws, want in golden_kat["combine"].items():
        assert omm.combine([int(w) for w in ws.split(",")]) == int(want, 16)
    vals = omm.gen_mapping(64, 3, 4, 42)
    sig = omm.signatures_c(np.array([[0, 5, 17, 63]], np.uint32), vals, 3, 2)[0]
    assert [int(v) for v in sig] == SIG_FROZEN
    assert [hex(int(v)) for v in sig] == golden_kat["sig_d64_t3_k4_s42_bits_0_5_17_63"]


def test_mapping_c_equals_numpy():
    vals = omm.gen_mapping(257, 7, 6, 2**64 - 5)
    c = np.empty_like(vals)
    oracle.c_lib().qso_gen_mapping(c.ctypes.data, 257, 21, 2**64 - 5)
    assert np.array_equal(c, vals)


def test_signature_oracles_vs_golden(golden_minmax):
    for name, case in golden_minmax.items():
        d, t, k = (int(v) for v in case["meta"])
        seed = int(case["seed"][0])
        vals = omm.gen_mapping(d, t, k, seed)
        want = case["sigs"]
        assert np.array_equal(omm.signatures_c(case["bits"], vals, t, k // 2, threads=3), want), name
        assert np.array_equal(omm.signatures_function_major(case["bits"], vals, t, k // 2), want), name
        ref = omm.signatures_reference_kernel(case["bits"], vals, t, k // 2, threads=2)
        if ref is not None:
            assert np.array_equal(ref, want), name


def _tuples(rec):
    return [(int(a), int(b), int(c)) for a, b, c in zip(rec["dt"], rec["idx1"], rec["sim"])]


def test_search_oracle_vs_golden(golden_search):
    for name, case in golden_search.items():
        cfg = dict(case["cfg"])
        rec, st = osr.search(case["sigs"], tables=cfg["tables"], min_matches=cfg["min_matches"],
                             partitions=cfg.get("partitions", 1),
                             occurrence_threshold=cfg.get("occurrence_threshold"),
                             exclusion_windows=cfg.get("exclusion_windows", 0))
        assert rec.tobytes() == case["trip"].tobytes(), name
        for key, want in case["stats"].items():
            got = st[key]
            if isinstance(want, float):
                assert got == pytest.approx(want, rel=1e-12, abs=1e-15), (name, key)
            else:
                assert got == want, (name, key)


def test_brute_force_equals_golden_without_filter(golden_search):
    for name in ("prone_p1", "tiny_alpha_excl0", "burst_off", "all_same"):
        case = golden_search[name]
        cfg = case["cfg"]
        want = sorted(_tuples(case["trip"]))
        got = osr.brute_force_triplets(case["sigs"], cfg["min_matches"], cfg.get("exclusion_windows", 0))
        assert got == want, name


def test_detection_probability_frozen():
    frozen = {(0.5, 6, 5, 100): 0.020679842345574547, (0.5, 4, 2, 100): 0.98792925094422222,
              (0.2, 6, 5, 100): 8.0430827162469282e-14, (0.1, 2, 1, 10): 0.09561792499119552}
    for (s, k, m, t), want in frozen.items():
        assert osr.detection_probability(s, k, m, t) == pytest.approx(want, abs=1e-12)


def test_fingerprint_oracle_vs_golden(golden_fingerprint):
    case = golden_fingerprint["cfg0_half_hour"]
    from paper_1803_09835_b200 import workloads
    res = ofp.fingerprint(case["samples"], 100.0, workloads.CFG0_PARAMS)
    assert tuple(res["band_rows"]) == tuple(case["band_rows"])
    np.testing.assert_array_equal(res["spec_band"], case["band"])
    np.testing.assert_allclose(res["median"], case["median"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(res["mad"], case["mad"], rtol=1e-6, atol=1e-9)
    assert np.array_equal(res["mad"] > 0, case["mad"] > 0)
    agree = np.mean(res["bits"] == case["bits"])
    assert agree >= 0.999
    c = ofp.coeffs(res["spec_band"], case["sel"], res["g"], 32, 64)
    np.testing.assert_allclose(c, case["coeffs"], rtol=1e-5, atol=1e-5)


def test_fingerprint_oracle_small_geometry(golden_fingerprint):
    case = golden_fingerprint["small_full_band"]
    params = dict(window_len_s=3.0, window_lag_s=0.5, freq_bins=8, time_bins=12, top_k=24,
                  band_low_hz=None, band_high_hz=None, frame_len_s=0.5, hop_s=0.05)
    res = ofp.fingerprint(case["samples"], 100.0, params, mad_rate=1.0)
    np.testing.assert_allclose(res["median"], case["median"], rtol=1e-6, atol=1e-9)
    assert np.mean(res["bits"] == case["bits"]) >= 0.999
