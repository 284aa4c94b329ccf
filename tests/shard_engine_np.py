"""TEST INFRASTRUCTURE — numpy stand-in for DeviceSearch restricted to a set
of tables, so the table-sharded host protocol (paper_1803_09835_b200/
sharded.py) can run on CPU under gloo.

It restates, bucket by bucket, what the device kernels compute for the
engine interface: buckets (stable sort per table), first-colliding-table pair
enumeration in the three modes of qs_lsh_pairs, the three occurrence-filter
steps, exclusion compaction, the bucket statistics walk of k_bucket_stats and
the (dt, idx1) finalisation.  Pure Python loops: small inputs only.
"""

import numpy as np
import torch

from paper_1803_09835_b200.lsh_search import TRIPLET_DTYPE, _HIST_LEN


class NumpyShardEngine:
    MODE_FULL, MODE_MATCHED, MODE_DISTINCT = 0, 1, 2

    def __init__(self, sigs, tables):
        self.sigs = np.ascontiguousarray(sigs, dtype=np.uint64)
        self.n, self.t = self.sigs.shape
        self.tables = list(tables)
        self.dev = torch.device("cpu")

    def buckets(self):
        self.blist, self.heads = [], 0
        for T in self.tables:
            col = self.sigs[:, T]
            order = np.argsort(col, kind="stable")
            scol = col[order]
            starts = np.flatnonzero(np.concatenate(([True], scol[1:] != scol[:-1])))
            ends = np.append(starts[1:], self.n)
            self.heads += len(starts)
            for a, b in zip(starts, ends):
                if b - a >= 2:
                    self.blist.append((T, order[a:b].astype(np.int64)))
        self.nb = len(self.blist)

    def compact(self, emask):
        em = emask.numpy().astype(bool)
        out = []
        for T, mem in self.blist:
            keep = mem[~em[mem]]
            if keep.size >= 2:
                out.append((T, keep))
        return out

    def _part(self, edges, p):
        e = edges.numpy()
        return lambda x: int(np.searchsorted(e, x, side="right") - 1) if p > 1 else 0

    def pairs(self, mode, m, excl, emask, edges, p, lists=None, cap=None):
        part = self._part(edges, p)
        em = None if emask is None else emask.numpy().astype(bool)
        keys, sims, distinct = [], [], 0
        for T, mem in (self.blist if lists is None else lists):
            for i in range(mem.size):
                for j in range(i + 1, mem.size):
                    a, b = int(mem[i]), int(mem[j])
                    eq = self.sigs[a] == self.sigs[b]
                    if eq[:T].any():
                        continue  # counted in the bucket of an earlier table
                    if b - a <= excl:
                        continue
                    sim = int(eq.sum())
                    if mode == self.MODE_MATCHED:
                        if sim >= m:
                            keys.append(((b - a) << 32) | a)
                            sims.append(sim)
                        continue
                    if em is not None and (em[a] or (em[b] and part(a) == part(b))):
                        continue
                    distinct += 1
                    if mode == self.MODE_FULL and sim >= m:
                        keys.append(((b - a) << 32) | a)
                        sims.append(sim)
        pk = torch.tensor(keys, dtype=torch.int64)
        ps = torch.tensor(sims, dtype=torch.int32)
        return pk, ps, len(keys), distinct

    def occ_degree(self, pk, matched, edges, p):
        part = self._part(edges, p)
        deg = torch.zeros(self.n, dtype=torch.int32)
        for k in pk[:matched].tolist():
            c, q = k & 0xFFFFFFFF, (k & 0xFFFFFFFF) + (k >> 32)
            if part(c) == part(q):
                deg[c] += 1
                deg[q] += 1
        return deg

    def occ_mark(self, pk, matched, deg, threshold, edges, p):
        part = self._part(edges, p)
        e = edges.numpy()
        mark = torch.zeros(self.n, dtype=torch.uint8)
        for i in range(self.n):
            P = part(i)
            if float(deg[i]) > threshold * float(e[P + 1] - e[P]):
                mark[i] = 2
        for k in pk[:matched].tolist():
            c, q = k & 0xFFFFFFFF, (k & 0xFFFFFFFF) + (k >> 32)
            if part(c) == part(q) and (mark[c] == 2 or mark[q] == 2):
                if mark[c] == 0:
                    mark[c] = 1
                if mark[q] == 0:
                    mark[q] = 1
        return mark

    def occ_finish(self, mark):
        mark = (mark > 0).to(torch.uint8)
        return mark, int(mark.sum())

    def filter_pairs(self, pk, ps, matched, emask, edges, p):
        part = self._part(edges, p)
        em = emask.numpy().astype(bool)
        keep = []
        for i, k in enumerate(pk[:matched].tolist()):
            c, q = k & 0xFFFFFFFF, (k & 0xFFFFFFFF) + (k >> 32)
            if em[c] or (em[q] and part(c) == part(q)):
                continue
            keep.append(i)
        idx = torch.tensor(keep, dtype=torch.int64)
        return pk[idx], ps[idx], len(keep)

    def bucket_stats(self, emask, edges, p):
        part = self._part(edges, p)
        em = None if emask is None else emask.numpy().astype(bool)
        e = edges.numpy()
        looks = pieces = mx = 0
        hist = np.zeros(_HIST_LEN, dtype=np.int64)
        big = []
        for _, mem in self.blist:
            s = mem.size
            j, cum_e, e_tot, lb = 0, 0, 0, 0
            while j < s:
                P = part(int(mem[j]))
                end = e[P + 1] if p > 1 else np.iinfo(np.int64).max
                nP = eP = 0
                while j < s and mem[j] < end:
                    nP += 1
                    eP += int(em is not None and em[mem[j]])
                    j += 1
                cum_e += eP
                e_tot += eP
                lb += nP * (s - cum_e)
                pieces += 1
                mx = max(mx, nP)
                if nP < _HIST_LEN:
                    hist[nP] += 1
                else:
                    big.append(nP)
            looks += lb - (s - e_tot)
        return looks, pieces, mx, hist, np.array(big, dtype=np.int64)

    def complete_sims(self, pk, ps, matched):
        """Sims here are exact already (DeviceSearch counts MATCHED lazily)."""
        return None

    def finalize(self, pk, ps, matched):
        k = pk[:matched].numpy().astype(np.uint64)
        s = ps[:matched].numpy().astype(np.uint32)
        o = np.argsort(k, kind="stable")
        rec = np.empty(matched, TRIPLET_DTYPE)
        rec["dt"] = k[o] >> np.uint64(32)
        rec["idx1"] = k[o] & np.uint64(0xFFFFFFFF)
        rec["sim"] = s[o]
        return torch.from_numpy(rec.view(np.uint8).copy())
