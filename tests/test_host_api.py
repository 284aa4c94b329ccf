"""Host-side API of the drop-in that needs no GPU: scalar math and
validation (reference tests/test_lsh_search.py:12-22, 45-70)."""

import json
import math
import os

import pytest

from conftest import GOLDEN


def test_detection_probability_matches_reference():
    """The product detection_probability (lsh_search.py:112-136 restated) at
    the reference's DP_FROZEN points and a grid, against values the reference
    itself computed (tests/golden/kat.json, make_golden.py --kat)."""
    from paper_1803_09835_b200 import lsh_search as ls
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        rows = json.load(f)["dp_frozen"]
    assert len(rows) >= 8
    for s, k, m, t, want in rows:
        got = ls.detection_probability(s, k, m, t)
        assert got == pytest.approx(want, rel=1e-12, abs=1e-300), (s, k, m, t)
    # the reference's own frozen literals (test_lsh_search.py:13-22), abs 1e-12
    for (s, k, m, t), want in {(0.5, 6, 5, 100): 0.020679842345574547,
                               (0.95, 2, 90, 100): 0.61603768190921333,
                               (0.1, 2, 1, 10): 0.09561792499119552}.items():
        assert ls.detection_probability(s, k, m, t) == pytest.approx(want, abs=1e-12)


def test_detection_probability_errors_and_limits():
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200.errors import ParameterError
    for bad in [(-0.1, 4, 5, 100), (1.1, 4, 5, 100), (0.5, 0, 5, 100), (0.5, 4, 0, 100),
                (0.5, 4, 101, 100)]:
        with pytest.raises(ParameterError):
            ls.detection_probability(*bad)
    assert ls.detection_probability(0.0, 4, 5, 100) == 0.0
    assert ls.detection_probability(1.0, 4, 5, 100) == 1.0
    # monotone in s
    prev = 0.0
    for i in range(1, 20):
        v = ls.detection_probability(i / 20, 4, 5, 100)
        assert v >= prev - 1e-12 and not math.isnan(v)  # log-space sum: 1e-14 wiggle near 1
        prev = v
