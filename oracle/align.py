"""ORACLE — test infrastructure only.  Channel combine / triplet sort restated
from reference pkg/src/quakescan/align.py:
  sort_triplet_file         :87-110   records ordered by (dt, idx1), stable
  combine_channel_triplets  :113-140  k-way merge of sorted channel streams,
                                      sims of equal (dt, idx1) summed, sums
                                      below threshold dropped
"""

import numpy as np

TRIPLET_DTYPE = np.dtype([("dt", "<u8"), ("idx1", "<u8"), ("sim", "<u4")])


def sort_records(rec):
    rec = np.asarray(rec, dtype=TRIPLET_DTYPE)
    return rec[np.lexsort((rec["idx1"], rec["dt"]))]


def combine(records, threshold: int):
    allr = sort_records(np.concatenate([np.asarray(r, dtype=TRIPLET_DTYPE) for r in records]))
    if allr.size == 0:
        return allr
    key_change = np.ones(allr.size, bool)
    key_change[1:] = (allr["dt"][1:] != allr["dt"][:-1]) | (allr["idx1"][1:] != allr["idx1"][:-1])
    starts = np.flatnonzero(key_change)
    sums = np.add.reduceat(allr["sim"].astype(np.int64), starts)
    keep = sums >= threshold
    out = np.empty(int(keep.sum()), dtype=TRIPLET_DTYPE)
    out["dt"] = allr["dt"][starts][keep]
    out["idx1"] = allr["idx1"][starts][keep]
    out["sim"] = sums[keep]
    return out
