"""Artifact formats (.tri / .fp / .mad / triplet CSV) against files written by
the reference's own writers (tests/golden/make_golden.py files()).  Mirrors
the reference's test_lsh_search / test_fingerprint file round-trip and error
taxonomy tests: byte-identical rewrite, record equality, FormatError on a bad
magic, CorruptInputError on truncation, ConsistencyError on a header without
the geometry keys."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_1803_09835_b200 import fingerprint as fp
from paper_1803_09835_b200 import lsh_search as ls
from paper_1803_09835_b200.errors import ConsistencyError, CorruptInputError, FormatError

FILES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "files")


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def ref_inputs():
    with open(os.path.join(FILES, "ref_inputs.json")) as f:
        return json.load(f)


def test_triplet_file_roundtrip(tmp_path, golden_search, ref_inputs):
    rec, header = ls.read_triplet_file(os.path.join(FILES, "ref.tri"))
    want = golden_search["cfg1_small_occ"]["trip"]
    assert rec.tobytes() == want.tobytes() and rec.size == ref_inputs["n_triplets"]
    assert header == ref_inputs["tri_header"]
    out = tmp_path / "x.tri"
    ls.write_triplet_file(out, rec, header)
    assert _bytes(out) == _bytes(os.path.join(FILES, "ref.tri"))
    assert ls.read_triplet_header(out)["count"] == rec.size
    got = np.concatenate(list(ls.iter_triplet_batches(out, batch=7)))
    assert got.tobytes() == rec.tobytes()
    part = np.concatenate(list(ls.iter_triplet_batches(out, start=3, stop=11, batch=4)))
    assert part.tobytes() == rec[3:11].tobytes()


def test_triplet_csv(tmp_path, golden_search):
    rec = golden_search["cfg1_small_occ"]["trip"]
    out = tmp_path / "x.csv"
    ls.write_triplet_csv(out, rec)
    assert _bytes(out) == _bytes(os.path.join(FILES, "ref.csv"))
    assert ls.read_triplet_csv(os.path.join(FILES, "ref.csv")).tobytes() == rec.tobytes()
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(CorruptInputError):
        ls.read_triplet_csv(bad)
    bad.write_text("dt,idx1,sim\n1,2\n")
    with pytest.raises(CorruptInputError):
        ls.read_triplet_csv(bad)


def test_fingerprint_file_roundtrip(tmp_path):
    src = os.path.join(FILES, "ref.fp")
    fps = fp.read_fingerprint_file(src)
    assert fps.meta["station"] == "ST1" and fps.meta["config_hash"] == "abc123"
    assert fps.bits.dtype == np.uint32 and fps.bits.shape[1] == fps.top_k == 24
    assert np.allclose(fps.epochs, 12.5 + np.arange(len(fps)) * 0.5)
    out = tmp_path / "x.fp"
    fp.write_fingerprint_file(out, fps)
    assert _bytes(out) == _bytes(src)


def test_mad_file_roundtrip(tmp_path):
    src = os.path.join(FILES, "ref.mad")
    stats, header = fp.read_mad_file(src)
    assert stats.n_coeffs == 8 * 12 and header["station"] == "ST1"
    out = tmp_path / "x.mad"
    fp.write_mad_file(out, stats, extra={"station": header["station"]})
    assert _bytes(out) == _bytes(src)


def test_file_errors(tmp_path):
    tri = os.path.join(FILES, "ref.tri")
    raw = _bytes(tri)
    bad = tmp_path / "bad.tri"
    bad.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(FormatError):
        ls.read_triplet_file(bad)
    bad.write_bytes(raw[:-5])
    with pytest.raises(CorruptInputError):
        ls.read_triplet_file(bad)
    bad.write_bytes(raw[:15])
    with pytest.raises(CorruptInputError):
        ls.read_triplet_file(bad)
    with pytest.raises(FormatError):
        fp.read_fingerprint_file(tri)  # a triplet file is not a fingerprint file
    # fingerprint header without the geometry keys
    from paper_1803_09835_b200 import container
    fpb = tmp_path / "nokeys.fp"
    with open(fpb, "wb") as f:
        container.write_preamble(f, fp.FP_MAGIC, {"top_k": 2}, count=0)
    with pytest.raises(ConsistencyError):
        fp.read_fingerprint_file(fpb)
    # non-positive dt
    rec, header = ls.read_triplet_file(tri)
    rec = rec.copy()
    rec["dt"][0] = 0
    zero = tmp_path / "zero.tri"
    ls.write_triplet_file(zero, rec, header)
    with pytest.raises(CorruptInputError):
        ls.read_triplet_file(zero)


@pytest.mark.gpu
def test_device_file_paths(tmp_path, golden_search):
    import torch
    src = os.path.join(FILES, "ref.fp")
    fps_d = fp.read_fingerprint_file(src, device=True)
    fps_h = fp.read_fingerprint_file(src)
    assert fps_d.bits.is_cuda
    assert np.array_equal(fps_d.bits.cpu().numpy().view(np.uint32), fps_h.bits)
    assert np.array_equal(fps_d.indices, fps_h.indices) and np.array_equal(fps_d.epochs, fps_h.epochs)
    out = tmp_path / "d.fp"
    fp.write_fingerprint_file(out, fps_d)
    assert _bytes(out) == _bytes(src)
    # device search result straight to a .tri file
    c = golden_search["cfg1_small_occ"]
    sigs = torch.from_numpy(np.ascontiguousarray(c["sigs"]).view(np.int64)).cuda()
    cfg = ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, occurrence_threshold=0.04)
    trip, _ = ls.search_signatures(sigs, cfg)
    assert trip.is_cuda
    _, header = ls.read_triplet_file(os.path.join(FILES, "ref.tri"))
    out = tmp_path / "d.tri"
    ls.write_triplet_file(out, trip, header)
    assert _bytes(out) == _bytes(os.path.join(FILES, "ref.tri"))
    rec_d, h2 = ls.read_triplet_file(out, device=True)
    assert rec_d.is_cuda and h2 == header
    assert bytes(rec_d.cpu().numpy().tobytes()) == c["trip"].tobytes()
