"""End-to-end drop-in proof against the reference-held golden report.

The reference freezes the detection report of its bundled demo run in
pkg/tests/data/demo_golden.json (copied by tests/golden/make_golden.py to
tests/golden/demo_golden.json after re-deriving it with the reference's own
serial harness).  Its serial oracle (pkg/tests/test_cli.py:54-100) composes

    synthesize -> bandpass -> fingerprint_series -> search_fingerprints
    -> per-station channel sum -> cluster_records -> network_associate

in memory.  Here the three hot-path stages are bound to this package
(device band-pass, device fingerprint chain, device Min-Max + LSH search) and
everything else — config loader, synthesis, clustering, association — is the
UNMODIFIED reference, installed into baseline/_ref (git-ignored, travels to
the GPU box; `python -m pip install --no-index --no-deps --target baseline/_ref`
of /root/reference/pkg).  The report must equal the golden
byte for byte.
"""

import json
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden", "demo_golden.json")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "quakescan")):
        pytest.fail("baseline/_ref/quakescan missing: install the reference (DESIGN.md §3)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import quakescan  # noqa: F401
    from quakescan import align, config, ingest, lsh_search
    return dict(align=align, config=config, ingest=ingest, lsh_search=lsh_search)


def detection_report(ref, cfg, bandpass, fingerprint_series, search_fingerprints):
    """The serial composition of test_cli.py:54-100 with the three hot-path
    stages injected."""
    align, ingest, rls = ref["align"], ref["ingest"], ref["lsh_search"]
    series = {(ts.station_id, ts.channel_id): ts for ts in ingest.synthesize(cfg.synth_spec())}
    pairs = []
    for st in cfg.stations:
        merged = {}
        lag = start = None
        for entry in st.channels:
            name = os.path.basename(entry)
            ch = name[len(st.station_id) + 1:].split(".")[0]
            ts = series[(st.station_id, ch)]
            if st.bandpass is not None:
                ts = bandpass(ts, st.bandpass)
            fps, _ = fingerprint_series(ts, cfg.fingerprint, mad_rate=cfg.mad_rate,
                                        mad_seed=cfg.seeds["mad"])
            rec, _, _ = search_fingerprints(fps, cfg.search, workers=1)
            for dt, i1, sim in zip(rec["dt"].tolist(), rec["idx1"].tolist(), rec["sim"].tolist()):
                merged[(dt, i1)] = merged.get((dt, i1), 0) + sim
            lag, start = fps.window_lag_s, ts.start_epoch_s
        kept = sorted((dt, i1, s) for (dt, i1), s in merged.items()
                      if s >= cfg.align.station_threshold)
        clusters = align.cluster_records(np.array(kept, dtype=rls.TRIPLET_DTYPE),
                                         cfg.align.cluster_params())
        pairs.extend(align.station_pairs_from_clusters(clusters, st.station_id, lag, start))
    dets = align.network_associate(pairs, dt_tol_s=cfg.align.dt_tol_s,
                                   start_tol_s=cfg.align.start_tol_s,
                                   min_stations=cfg.align.min_stations)
    doc = {
        "config_hash": cfg.config_hash,
        "min_stations": cfg.align.min_stations,
        "n_station_pairs": len(pairs),
        "n_detections": len(dets),
        "detections": [
            {"station_count": d.station_count, "score": d.score, "delta_t_s": d.delta_t_s,
             "event1_epoch_s": d.event1_epoch_s,
             "arrivals": {s: [a1, a2] for s, (a1, a2) in sorted(d.arrivals.items())}}
            for d in dets
        ],
    }
    return (json.dumps(doc, sort_keys=True, separators=(",", ":")) + "\n").encode()


def _demo_cfg(ref, tmp_path):
    from importlib import resources
    src = resources.files("quakescan").joinpath("data/demo.toml")
    dst = tmp_path / "demo.toml"
    dst.write_text(src.read_text(encoding="utf-8"), encoding="utf-8")
    return ref["config"].load_config(str(dst))


def test_demo_report_through_drop_in(ref, tmp_path):
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200 import ingest as ing
    from paper_1803_09835_b200 import lsh_search as ls
    cfg = _demo_cfg(ref, tmp_path)
    got = detection_report(ref, cfg, ing.bandpass, fp.fingerprint_series, ls.search_fingerprints)
    with open(GOLDEN, "rb") as f:
        want = f.read()
    assert got == want


def test_demo_intermediates_match_reference(ref, tmp_path):
    """Per-channel intermediates of the same run: fingerprints bit-identical
    to the reference's, triplets byte-identical (the golden report above sums
    and clusters them, so this localises any difference)."""
    from quakescan import fingerprint as rfp
    from paper_1803_09835_b200 import fingerprint as fp
    from paper_1803_09835_b200 import ingest as ing
    from paper_1803_09835_b200 import lsh_search as ls
    cfg = _demo_cfg(ref, tmp_path)
    rls = ref["lsh_search"]
    for ts in ref["ingest"].synthesize(cfg.synth_spec()):
        st = cfg.station(ts.station_id)
        want_ts = ref["ingest"].bandpass(ts, st.bandpass)
        got_ts = ing.bandpass(ts, st.bandpass)
        scale = float(np.abs(want_ts.samples).max())
        assert np.abs(got_ts.samples - want_ts.samples).max() <= 1e-9 * scale
        want_fp, want_mad = rfp.fingerprint_series(want_ts, cfg.fingerprint, mad_rate=cfg.mad_rate,
                                                   mad_seed=cfg.seeds["mad"])
        got_fp, got_mad = fp.fingerprint_series(want_ts, cfg.fingerprint, mad_rate=cfg.mad_rate,
                                                mad_seed=cfg.seeds["mad"])
        assert np.array_equal(got_fp.bits, want_fp.bits), ts.channel_id
        np.testing.assert_allclose(got_mad.median, want_mad.median, rtol=1e-6, atol=1e-9)
        want_rec, want_st, _ = rls.search_fingerprints(want_fp, cfg.search)
        got_rec, got_st, _ = ls.search_fingerprints(want_fp, cfg.search)
        assert got_rec.tobytes() == want_rec.tobytes()
        gd, wd = got_st.to_dict(), want_st.to_dict()
        for k, v in wd.items():
            if isinstance(v, float):
                assert gd[k] == pytest.approx(v, rel=1e-12, abs=1e-15), k
            else:
                assert gd[k] == v, k
