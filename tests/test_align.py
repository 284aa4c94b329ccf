"""Channel combine and triplet sort (reference align.py:87-140) against the
reference-written fixtures (tests/golden/files: ch*.tri -> combined.tri at
threshold 6, unsorted.tri -> sorted.tri) and the oracle restatement."""

import os

import numpy as np
import pytest

from oracle import align as oal
from paper_1803_09835_b200 import lsh_search as ls

FILES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "files")
CH = [os.path.join(FILES, f"ch{c}.tri") for c in range(3)]


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def test_oracle_matches_reference_files():
    chans = [ls.read_triplet_file(p)[0] for p in CH]
    want, _ = ls.read_triplet_file(os.path.join(FILES, "combined.tri"))
    assert oal.combine(chans, 6).tobytes() == want.tobytes()
    uns, _ = ls.read_triplet_file(os.path.join(FILES, "unsorted.tri"))
    srt, _ = ls.read_triplet_file(os.path.join(FILES, "sorted.tri"))
    assert oal.sort_records(uns).tobytes() == srt.tobytes()


@pytest.mark.gpu
def test_combine_and_sort_files(tmp_path):
    from paper_1803_09835_b200 import align
    from paper_1803_09835_b200.errors import ConsistencyError, ParameterError
    out = tmp_path / "c.tri"
    n = align.combine_channel_triplets(CH, out, 6, {"station": "ST1", "combined": True})
    assert _bytes(out) == _bytes(os.path.join(FILES, "combined.tri"))
    assert n == ls.read_triplet_header(out)["count"]
    out2 = tmp_path / "s.tri"
    align.sort_triplet_file(os.path.join(FILES, "unsorted.tri"), out2, {"channel": "C0", "sorted": True})
    assert _bytes(out2) == _bytes(os.path.join(FILES, "sorted.tri"))
    with pytest.raises(ConsistencyError):
        align.combine_channel_triplets([os.path.join(FILES, "unsorted.tri")], tmp_path / "x.tri", 1, {})
    with pytest.raises(ParameterError):
        align.combine_channel_triplets([], tmp_path / "x.tri", 1, {})
    with pytest.raises(ParameterError):
        align.combine_channel_triplets(CH, tmp_path / "x.tri", 0, {})
    with pytest.raises(ParameterError):
        align.sort_triplet_file(CH[0], tmp_path / "x.tri", {}, chunk_records=0)


@pytest.mark.gpu
def test_combine_random_vs_oracle():
    from paper_1803_09835_b200 import align
    rng = np.random.default_rng(17)
    for n_ch, n, hi, thr in [(1, 0, 10, 1), (2, 1000, 50, 3), (4, 200_000, 3000, 9),
                             (3, 50_000, 2**31, 2)]:
        recs = []
        for _ in range(n_ch):
            r = np.zeros(n, dtype=oal.TRIPLET_DTYPE)
            r["dt"] = rng.integers(1, hi, n)
            r["idx1"] = rng.integers(0, hi, n)
            r["sim"] = rng.integers(1, 100, n)
            recs.append(oal.sort_records(r))
        got = align.combine_host(recs, thr)
        assert got.tobytes() == oal.combine(recs, thr).tobytes()
