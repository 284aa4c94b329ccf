"""Seeded synthetic workloads standing in for BASELINE.json configs 0-4.

The reference measures on no public dataset, so every
configuration is seeded synthetic data with the shapes and value
distributions BASELINE.json states; SURVEY.md §8(d) fixes the generators.

  cfg0  one day at 100 Hz of N(0,1) float32 noise plus 5 damped-chirp 30 s
        templates x 20 copies (amplitude log-uniform 0.2..2 x noise RMS)
  cfg1  N sparse 4096-bit fingerprints with exactly 400 set bits (uniform),
        N/80 planted near-duplicate pairs (Jaccard U(0.4, 0.9)) and N/400
        noise groups of 200 rows at Jaccard 0.7 to a group template
  cfg2  colored (1/f) noise plus planted template repeats, fingerprinting only

These generators are test/bench inputs, not part of the hot path.
"""

import math

import numpy as np

SR_HZ = 100.0

CFG0_PARAMS = dict(window_len_s=10.0, window_lag_s=1.0, freq_bins=32, time_bins=64,
                   top_k=200, band_low_hz=4.0, band_high_hz=10.0,
                   frame_len_s=2.0, hop_s=0.1)
CFG0_SEARCH = dict(tables=100, hash_funcs=4, min_matches=5, seed=0, partitions=1,
                   occurrence_threshold=0.01)
CFG1_SEARCH = dict(tables=100, hash_funcs=4, min_matches=5, seed=0, partitions=1)
CFG1_OCC = 1.5e-5   # limit 120 matches at N=8e6: removes the noise groups


# ---------------------------------------------------------------------------
# continuous traces

def chirp_templates(rng, n_templates=5, length_s=30.0, sr=SR_HZ):
    t = np.arange(int(round(length_s * sr))) / sr
    out = []
    for _ in range(n_templates):
        f0 = rng.uniform(4.0, 6.0)
        f1 = rng.uniform(8.0, 10.0)
        tau = rng.uniform(5.0, 15.0)
        w = np.exp(-t / tau) * np.sin(2 * np.pi * (f0 * t + (f1 - f0) * t * t / (2 * length_s)))
        out.append((w / np.abs(w).max()).astype(np.float32))
    return out


def plant(x, rng, templates, copies, rms=1.0):
    n = x.size
    truth = []
    for ti, w in enumerate(templates):
        offs = rng.integers(0, n - w.size, size=copies)
        amps = 10.0 ** rng.uniform(math.log10(0.2), math.log10(2.0), size=copies)
        for o, a in zip(offs, amps):
            x[o:o + w.size] += np.float32(a * rms) * w
            truth.append((ti, int(o), float(a)))
    return truth


def cfg0_trace(n_samples=8_640_000, seed=0, copies=20, n_templates=5):
    """cfg0: Gaussian noise + planted damped chirps. Returns (float32 samples, truth)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n_samples, dtype=np.float32)
    truth = plant(x, rng, chirp_templates(rng, n_templates), copies)
    return x, truth


def colored_noise(n_samples, seed=0, slope=-1.0, chunk=1 << 22):
    """1/f^|slope| noise by shaping the rfft of white noise chunkwise (float32)."""
    rng = np.random.default_rng(seed)
    out = np.empty(n_samples, np.float32)
    f = np.fft.rfftfreq(chunk, 1.0 / SR_HZ)
    shape = np.ones_like(f)
    shape[1:] = f[1:] ** (slope / 2.0)
    shape[0] = 0.0
    shape /= math.sqrt(np.mean(shape ** 2))
    for a in range(0, n_samples, chunk):
        b = min(n_samples, a + chunk)
        w = rng.standard_normal(chunk)
        y = np.fft.irfft(np.fft.rfft(w) * shape, n=chunk)
        out[a:b] = y[: b - a].astype(np.float32)
    return out


def cfg2_trace(n_samples=795_000_000, seed=2, repeats=500):
    rng = np.random.default_rng(seed + 1)
    x = colored_noise(n_samples, seed)
    templates = chirp_templates(rng)
    truth = plant(x, rng, templates, copies=max(1, repeats // len(templates)))
    return x, truth


# ---------------------------------------------------------------------------
# sparse fingerprints (cfg1)

def _random_rows(rng, n, d, K, chunk=2048):
    out = np.empty((n, K), np.uint32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        keys = rng.random((b - a, d), dtype=np.float32)
        out[a:b] = np.argpartition(keys, K, axis=1)[:, :K]
    out.sort(axis=1)
    return out


def _mutate(rng, template, keep, d):
    """Keep `keep` of the template's bits, replace the rest by non-members."""
    K = template.size
    kept = rng.choice(template, keep, replace=False)
    mask = np.ones(d, bool)
    mask[template] = False
    pool = np.flatnonzero(mask)
    new = rng.choice(pool, K - keep, replace=False)
    return np.sort(np.concatenate([kept, new])).astype(np.uint32)


def cfg1_bits(n=8_000_000, d=4096, K=400, seed=1, pair_frac=1 / 80, group_frac=1 / 400,
              group_size=200, group_j=0.7):
    """cfg1 generator (numpy; practical up to ~1e6 rows).

    Returns (bits (n, K) uint32 ascending, info dict with planted pairs/groups)."""
    rng = np.random.default_rng(seed)
    bits = _random_rows(rng, n, d, K)
    perm = rng.permutation(n)
    n_pairs = int(round(n * pair_frac))
    n_groups = int(round(n * group_frac))
    if 2 * n_pairs + n_groups * group_size > n:
        raise ValueError("workload does not fit")
    pairs = perm[: 2 * n_pairs].reshape(n_pairs, 2)
    jac = rng.uniform(0.4, 0.9, size=n_pairs)
    for (a, b), j in zip(pairs, jac):
        s = int(round(2 * K * j / (1 + j)))
        bits[b] = _mutate(rng, bits[a], s, d)
    groups = perm[2 * n_pairs: 2 * n_pairs + n_groups * group_size].reshape(n_groups, group_size)
    s_grp = int(round(2 * K * group_j / (1 + group_j)))
    for g in groups:
        for r in g[1:]:
            bits[r] = _mutate(rng, bits[g[0]], s_grp, d)
    return bits, dict(pairs=pairs, jaccard=jac, groups=groups)


def cfg1_bits_torch(n=8_000_000, d=4096, K=400, seed=1, device="cuda", pair_frac=1 / 80,
                    group_frac=1 / 400, group_size=200, group_j=0.7, chunk=65536):
    """cfg1 generator on the GPU (torch RNG; same distribution as cfg1_bits,
    different stream). Returns a (n, K) int32 CUDA tensor, ascending rows."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bits = torch.empty((n, K), dtype=torch.int32, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        keys = torch.rand((b - a, d), generator=g, device=device)
        bits[a:b] = torch.topk(keys, K, dim=1, sorted=False).indices.to(torch.int32)
    perm = torch.randperm(n, generator=g, device=device)
    n_pairs = int(round(n * pair_frac))
    n_groups = int(round(n * group_frac))
    pairs = perm[: 2 * n_pairs].view(n_pairs, 2)
    groups = perm[2 * n_pairs: 2 * n_pairs + n_groups * group_size].view(n_groups, group_size)

    def mutate(src_rows, keep):
        # keep[i] of the template row's bits (random subset), rest from its complement
        m = src_rows.shape[0]
        tmpl = bits[src_rows].long()                                   # (m, K)
        pr = torch.rand((m, K), generator=g, device=device)
        order = torch.argsort(pr, dim=1)
        kept_sorted = torch.gather(tmpl, 1, order)                     # random order
        member = torch.zeros((m, d), dtype=torch.bool, device=device)
        member.scatter_(1, tmpl, True)
        ck = torch.rand((m, d), generator=g, device=device)
        ck.masked_fill_(member, 2.0)                                   # members last
        fresh = torch.argsort(ck, dim=1)[:, :K]                        # non-members first
        col = torch.arange(K, device=device)[None, :]
        out = torch.where(col < keep[:, None], kept_sorted, fresh)
        return out.to(torch.int32)

    jac = torch.rand(n_pairs, generator=g, device=device) * 0.5 + 0.4
    s = torch.round(2 * K * jac / (1 + jac)).long()
    for a in range(0, n_pairs, 8192):
        b = min(n_pairs, a + 8192)
        bits[pairs[a:b, 1]] = mutate(pairs[a:b, 0], s[a:b])
    s_grp = int(round(2 * K * group_j / (1 + group_j)))
    tmpl_rows = groups[:, 0:1].expand(-1, group_size - 1).reshape(-1)
    dst_rows = groups[:, 1:].reshape(-1)
    for a in range(0, dst_rows.numel(), 8192):
        b = min(dst_rows.numel(), a + 8192)
        keep = torch.full((b - a,), s_grp, dtype=torch.long, device=device)
        bits[dst_rows[a:b]] = mutate(tmpl_rows[a:b], keep)
    bits, _ = torch.sort(bits, dim=1)
    return bits, dict(pairs=pairs, jaccard=jac, groups=groups)


def cfg2_trace_torch(n_samples=795_000_000, seed=2, repeats=500, device="cuda", slope=-1.0,
                     chunk=1 << 22):
    """cfg2 on the GPU: 1/f^|slope| noise (white noise shaped in the rfft
    domain chunkwise, unit RMS, as colored_noise) plus `repeats` planted
    copies of the cfg0 chirp templates (amplitude log-uniform 0.2..2 x RMS).
    torch RNG for the noise (a different stream from the numpy generator, same
    distribution); templates, offsets and amplitudes from numpy.  Returns a
    float32 CUDA tensor and the truth list."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty(n_samples, dtype=torch.float32, device=device)
    f = torch.fft.rfftfreq(chunk, 1.0 / SR_HZ, device=device, dtype=torch.float64)
    shape = torch.ones_like(f)
    shape[1:] = f[1:] ** (slope / 2.0)
    shape[0] = 0.0
    shape /= torch.sqrt(torch.mean(shape ** 2))
    shape = shape.to(torch.complex64)
    for a in range(0, n_samples, chunk):
        b = min(n_samples, a + chunk)
        w = torch.randn(chunk, generator=g, device=device, dtype=torch.float32)
        y = torch.fft.irfft(torch.fft.rfft(w) * shape, n=chunk)
        out[a:b] = y[: b - a]
    rng = np.random.default_rng(seed + 1)
    templates = chirp_templates(rng)
    copies = max(1, repeats // len(templates))
    truth = []
    for ti, wv in enumerate(templates):
        offs = rng.integers(0, n_samples - wv.size, size=copies)
        amps = 10.0 ** rng.uniform(math.log10(0.2), math.log10(2.0), size=copies)
        wd = torch.from_numpy(wv).to(device)
        for o, amp in zip(offs, amps):
            out[int(o):int(o) + wv.size] += float(amp) * wd
            truth.append((ti, int(o), float(amp)))
    return out, truth


def cfg3_trace_torch(n_samples=3_150_000_000, seed=3, repeats=2000, periodic=50, period_s=60.0,
                     periodic_amp=(0.1, 0.3), jitter_s=2.0, device="cuda", chunk=1 << 26):
    """cfg3 (1 year at 100 Hz) on the GPU: N(0, 1) float32 noise, `repeats`
    planted copies of the cfg0 chirp templates (amplitude log-uniform
    0.2..2 x RMS) and `periodic` noise templates repeating every `period_s`.

    The periodic templates are BOUNDED as SURVEY.md §7.2 item 2 requires (an
    exact repeat every 60 s for a year makes 525,600 near-identical windows per
    template, whose pairs the reference's occurrence filter must enumerate
    before it can exclude them): each is weak (amplitude U(0.1, 0.3) x RMS,
    below the noise) and every repetition is jittered by U(-2, 2) s in 0.1 s
    steps.  Returns a float32 CUDA tensor and a dict of what was planted."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.empty(n_samples, dtype=torch.float32, device=device)
    for a in range(0, n_samples, chunk):
        b = min(n_samples, a + chunk)
        x[a:b] = torch.randn(b - a, generator=g, device=device, dtype=torch.float32)
    rng = np.random.default_rng(seed + 1)
    events = chirp_templates(rng)
    per = max(1, repeats // len(events))
    ev_truth = []
    for ti, wv in enumerate(events):
        offs = rng.integers(0, n_samples - wv.size, size=per)
        amps = 10.0 ** rng.uniform(math.log10(0.2), math.log10(2.0), size=per)
        wd = torch.from_numpy(wv).to(device)
        for o, amp in zip(offs, amps):
            x[int(o):int(o) + wv.size] += float(amp) * wd
            ev_truth.append((ti, int(o), float(amp)))
    # periodic templates: damped chirps of a second family, one 60 s cell each
    cell = int(round(period_s * SR_HZ))
    cells = n_samples // cell
    view = x[: cells * cell].view(cells, cell)
    ptemps = chirp_templates(rng, n_templates=periodic, length_s=20.0)
    L = ptemps[0].size
    jmax = int(round(jitter_s * 10))
    span = cell - L - 2 * jmax * 10
    for p, wv in enumerate(ptemps):
        amp = float(rng.uniform(*periodic_amp))
        base = jmax * 10 + (p * span) // max(1, periodic - 1)
        jit = torch.randint(-jmax, jmax + 1, (cells,), generator=g, device=device) * 10
        src = torch.zeros((1, cell), dtype=torch.float32, device=device)
        wd = torch.from_numpy(wv).to(device) * amp
        for v in range(-jmax, jmax + 1):
            rows = torch.nonzero(jit == v * 10).view(-1)
            if rows.numel() == 0:
                continue
            s0 = base + v * 10
            src.zero_()
            src[0, s0:s0 + L] = wd
            view.index_add_(0, rows, src.expand(rows.numel(), cell))
    return x, {"events": ev_truth, "periodic": periodic, "cells": cells}


def cfg4_events(n_samples=3_150_000_000, seed=4, repeats=2000, stations=10, max_delay_s=8.0,
                gain=(0.3, 3.0)):
    """cfg4's shared event catalogue: `repeats` planted copies of the cfg0
    chirp templates at uniform times (amplitude log-uniform 0.2..2 x RMS at a
    unit-gain station), each arriving at every station with its own delay
    U(0, max_delay_s), and one gain per station, log-uniform in `gain`."""
    rng = np.random.default_rng(seed)
    events = chirp_templates(rng)
    per = max(1, repeats // len(events))
    L = events[0].size
    span = n_samples - L - int(max_delay_s * SR_HZ) - 1
    cat = []
    for ti in range(len(events)):
        offs = rng.integers(0, span, size=per)
        amps = 10.0 ** rng.uniform(math.log10(0.2), math.log10(2.0), size=per)
        cat.extend((ti, int(o), float(a)) for o, a in zip(offs, amps))
    delays = np.round(rng.uniform(0.0, max_delay_s, size=(stations, len(cat))) * SR_HZ).astype(np.int64)
    gains = 10.0 ** rng.uniform(math.log10(gain[0]), math.log10(gain[1]), size=stations)
    return {"templates": events, "catalogue": cat, "delays": delays, "gains": gains}


def cfg4_station_torch(station, ev, n_samples=3_150_000_000, seed=4, device="cuda",
                       chunk=1 << 26):
    """cfg4 (10 stations x 1 year at 100 Hz) on the GPU, one station at a
    time: independent seeded N(0, 1) float32 noise per station plus the shared
    catalogue of `cfg4_events`, delayed and scaled per station."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1000 + station)
    x = torch.empty(n_samples, dtype=torch.float32, device=device)
    for a in range(0, n_samples, chunk):
        b = min(n_samples, a + chunk)
        x[a:b] = torch.randn(b - a, generator=g, device=device, dtype=torch.float32)
    wds = [torch.from_numpy(w).to(device) for w in ev["templates"]]
    gain = float(ev["gains"][station])
    for (ti, o, amp), dl in zip(ev["catalogue"], ev["delays"][station]):
        s0 = o + int(dl)
        x[s0:s0 + wds[ti].numel()] += gain * amp * wds[ti]
    return x
