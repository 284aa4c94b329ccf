// One-call fingerprint chain of the C ABI (fingerprint.fingerprint_series,
// fingerprint.py:581-623, for non-Python callers): the host geometry the
// Python layer computes (paper_1803_09835_b200/fingerprint.py _Chain) —
// STFT frame/hop, band rows (fingerprint.py:166-173), hanning-tapered DFT
// twiddles of the band bins, area-overlap resize weights (:176-186) as CSR,
// the Haar level schedule (:256-268) — then the same device stages: band
// STFT, the MAD sample pass + per-coefficient median/MAD (estimate_mad,
// :341-389) and the top-K sign-bit pass (:433-466).  Every buffer comes from
// one caller workspace.
//
// The MAD sample is an input (sorted window indices): the reference draws it
// with numpy's default_rng(seed).choice (fingerprint.py:356-362), which a C
// caller cannot reproduce; passing median/MAD instead skips the MAD pass
// (fingerprint_series(stats=...)).
#include <math.h>

#include <algorithm>
#include <vector>

#include "qs_common.cuh"

namespace {

struct Geo {
    uint32_t frame, hop, r0, r1, nb, wmin, wmax, F, T;
    uint64_t win, lag, n_cols, n_win;
};

int geometry(uint64_t n, double sr, const qs_fp_params* p, Geo& g) {
    QS_ARG(p != nullptr && sr > 0, "sample rate must be positive");
    QS_ARG(p->window_lag_s > 0 && p->window_len_s > 0, "window length and lag must be positive");
    QS_ARG(p->window_lag_s <= p->window_len_s, "window lag must not exceed window length");
    QS_ARG(p->freq_bins >= 1 && p->time_bins >= 1, "spectral image shape must be at least 1x1");
    const uint64_t nc = (uint64_t)p->freq_bins * p->time_bins;
    QS_ARG(p->top_k >= 1 && p->top_k <= nc, "top_k must be in [1, %llu], got %u",
           (unsigned long long)nc, p->top_k);
    const bool band = p->band_low_hz > 0 || p->band_high_hz > 0;
    QS_ARG(!band || (p->band_low_hz > 0 && p->band_low_hz < p->band_high_hz),
           "need 0 < band_low_hz < band_high_hz");
    QS_ARG(p->frame_len_s > 0 && p->hop_s > 0, "STFT frame and hop must be positive");
    // int(round(x)) of Python: round half to even
    g.frame = (uint32_t)nearbyint(p->frame_len_s * sr);
    g.hop = (uint32_t)std::max(1.0, nearbyint(p->hop_s * sr));
    g.win = (uint64_t)nearbyint(p->window_len_s * sr);
    g.lag = (uint64_t)std::max(1.0, nearbyint(p->window_lag_s * sr));
    QS_ARG(g.frame >= 2, "STFT frame shorter than 2 samples");
    QS_DATA(n >= g.frame, "series shorter than one STFT frame");
    g.n_cols = (n - g.frame) / g.hop + 1;
    g.n_win = n >= g.win ? (n - g.win) / g.lag + 1 : 0;
    QS_DATA(g.n_win > 0, "series shorter than one fingerprint window");
    QS_ARG(g.win >= g.frame, "fingerprint window shorter than one STFT frame");
    // rfftfreq(frame, 1 / sr) and the band rows
    const uint32_t nf = g.frame / 2 + 1;
    const double val = 1.0 / ((double)g.frame * (1.0 / sr));
    g.r0 = 0;
    g.r1 = nf;
    if (band) {
        int64_t a = -1, b = -1;
        for (uint32_t k = 0; k < nf; ++k) {
            const double f = (double)k * val;
            if (f >= p->band_low_hz - 1e-9 && f <= p->band_high_hz + 1e-9) {
                if (a < 0) a = k;
                b = k;
            }
        }
        QS_ARG(a >= 0, "no spectrogram rows inside configured band");
        g.r0 = (uint32_t)a;
        g.r1 = (uint32_t)b + 1;
    }
    g.nb = g.r1 - g.r0;
    // window widths in STFT columns (c0 = ceil(i lag / hop), c1 = (i lag + win - frame) // hop + 1)
    g.wmin = UINT32_MAX;
    g.wmax = 0;
    const uint64_t probe = std::min<uint64_t>(g.n_win, (uint64_t)g.hop * 2 + 1);
    for (uint64_t i = 0; i < probe; ++i) {
        const uint64_t off = i * g.lag;
        const uint64_t c0 = (off + g.hop - 1) / g.hop;
        const int64_t c1 = (int64_t)((off + g.win - g.frame) / g.hop) + 1;
        const int64_t w = c1 - (int64_t)c0;
        QS_ARG(w >= 1, "window contains no complete STFT frame");
        g.wmin = std::min<uint32_t>(g.wmin, (uint32_t)w);
        g.wmax = std::max<uint32_t>(g.wmax, (uint32_t)w);
    }
    g.F = p->freq_bins;
    g.T = p->time_bins;
    return QS_OK;
}

// area-overlap resampling (fingerprint.py:176-186) of src -> dst as CSR
void resize_csr(uint32_t src, uint32_t dst, std::vector<int32_t>& off, std::vector<int32_t>& idx,
                std::vector<double>& val, int32_t base) {
    const double r = (double)src / (double)dst;
    for (uint32_t i = 0; i < dst; ++i) {
        const double lo = i * r, hi = (i + 1) * r;
        for (int64_t j = (int64_t)floor(lo); j < std::min<int64_t>((int64_t)ceil(hi), src); ++j) {
            const double w = (std::min(hi, (double)(j + 1)) - std::max(lo, (double)j)) / r;
            if (w != 0.0) {
                idx.push_back((int32_t)j);
                val.push_back(w);
            }
        }
        off.push_back(base + (int32_t)idx.size());
    }
}

struct Tables {
    std::vector<double> tw;
    std::vector<int32_t> wf_off, wf_idx, wt_off, wt_idx, sched;
    std::vector<double> wf_val, wt_val;
};

void tables(const Geo& g, Tables& tb) {
    // hanning taper (np.hanning: 0.5 + 0.5 cos(pi n / (M - 1)), n = 1-M, 3-M, ...)
    const double M = g.frame;
    std::vector<double> taper(g.frame);
    for (uint32_t j = 0; j < g.frame; ++j) {
        const double nn = (1.0 - M) + 2.0 * j;
        taper[j] = 0.5 + 0.5 * cos(M_PI * nn / (M - 1.0));
    }
    tb.tw.resize((size_t)g.nb * g.frame * 2);
    for (uint32_t b = 0; b < g.nb; ++b) {
        const uint64_t k = g.r0 + b;
        for (uint32_t j = 0; j < g.frame; ++j) {
            const double ang = 2.0 * M_PI * (double)((k * j) % g.frame) / (double)g.frame;
            tb.tw[((size_t)b * g.frame + j) * 2 + 0] = taper[j] * cos(ang);
            tb.tw[((size_t)b * g.frame + j) * 2 + 1] = -taper[j] * sin(ang);
        }
    }
    tb.wf_off = {0};
    resize_csr(g.nb, g.F, tb.wf_off, tb.wf_idx, tb.wf_val, 0);
    // one (T + 1)-offset CSR block per window width, concatenated
    tb.wt_off.clear();
    for (uint32_t w = g.wmin; w <= g.wmax; ++w) {
        tb.wt_off.push_back((int32_t)tb.wt_idx.size());
        std::vector<int32_t> off, idx;
        std::vector<double> val;
        resize_csr(w, g.T, off, idx, val, (int32_t)tb.wt_idx.size());
        tb.wt_off.insert(tb.wt_off.end(), off.begin(), off.end());
        tb.wt_idx.insert(tb.wt_idx.end(), idx.begin(), idx.end());
        tb.wt_val.insert(tb.wt_val.end(), val.begin(), val.end());
    }
    // Haar schedule (fingerprint.py:256-268): (h, w, 3) levels, then (h, w, 1), then (h, w, 2)
    uint32_t h = g.F, w = g.T;
    tb.sched.clear();
    while (h % 2 == 0 && h > 1 && w % 2 == 0 && w > 1) {
        tb.sched.insert(tb.sched.end(), {(int32_t)h, (int32_t)w, 3});
        h /= 2;
        w /= 2;
    }
    while (w % 2 == 0 && w > 1) {
        tb.sched.insert(tb.sched.end(), {(int32_t)h, (int32_t)w, 1});
        w /= 2;
    }
    while (h % 2 == 0 && h > 1) {
        tb.sched.insert(tb.sched.end(), {(int32_t)h, (int32_t)w, 2});
        h /= 2;
    }
}

struct Bump {
    uint8_t* base;
    size_t cap, off;
    bool ok = true;
    template <class T>
    T* take(uint64_t count) {
        off = (off + 255) & ~(size_t)255;
        const size_t bytes = (size_t)count * sizeof(T);
        if (!base) {
            off += bytes;
            return nullptr;
        }
        if (off + bytes > cap) {
            ok = false;
            return nullptr;
        }
        T* p = (T*)(base + off);
        off += bytes;
        return p;
    }
};

struct Dev {
    double* tw;
    float* band;
    int32_t *wf_off, *wf_idx, *wt_off, *wt_idx, *sched;
    double *wf_val, *wt_val, *mws;
    uint32_t* flags;
    float* cols;
    float* rows;  // the MAD sample, one coefficient row per window (transposed into cols)
};

void carve(Bump& a, const Geo& g, const Tables& tb, uint64_t n_sample, Dev& d) {
    d.tw = a.take<double>(tb.tw.size());
    d.band = a.take<float>(g.n_cols * g.nb);
    d.wf_off = a.take<int32_t>(tb.wf_off.size());
    d.wf_idx = a.take<int32_t>(std::max<size_t>(1, tb.wf_idx.size()));
    d.wf_val = a.take<double>(std::max<size_t>(1, tb.wf_val.size()));
    d.wt_off = a.take<int32_t>(tb.wt_off.size());
    d.wt_idx = a.take<int32_t>(std::max<size_t>(1, tb.wt_idx.size()));
    d.wt_val = a.take<double>(std::max<size_t>(1, tb.wt_val.size()));
    d.sched = a.take<int32_t>(std::max<size_t>(3, tb.sched.size()));
    d.flags = a.take<uint32_t>(4);
    d.mws = a.take<double>(2 * (uint64_t)g.F * g.T);
    d.cols = a.take<float>((uint64_t)g.F * g.T * n_sample);
    d.rows = a.take<float>((uint64_t)g.F * g.T * n_sample);
}

template <class T>
int h2d(T* dst, const std::vector<T>& v, cudaStream_t st) {
    if (v.empty()) return QS_OK;
    QS_CUDA(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    return QS_OK;
}

#define QS_TRY(x)            \
    do {                     \
        int _rc = (x);       \
        if (_rc) return _rc; \
    } while (0)

}  // namespace

extern "C" {

int qs_fp_n_windows(uint64_t n_samples, double sample_rate_hz, const qs_fp_params* params,
                    uint64_t* n_windows_out) {
    Geo g;
    QS_TRY(geometry(n_samples, sample_rate_hz, params, g));
    *n_windows_out = g.n_win;
    return QS_OK;
}

size_t qs_fingerprint_chain_ws_bytes(uint64_t n_samples, double sample_rate_hz,
                                     const qs_fp_params* params, uint64_t n_mad_sample) {
    Geo g;
    if (geometry(n_samples, sample_rate_hz, params, g)) return 0;
    Tables tb;
    tables(g, tb);
    Bump a{nullptr, 0, 0};
    Dev d;
    carve(a, g, tb, n_mad_sample, d);
    return a.off + 256;
}

int qs_fingerprint_chain(const void* x_dev, int x_is_f32, uint64_t n_samples,
                         double sample_rate_hz, const qs_fp_params* params,
                         const int64_t* mad_sample_dev, uint64_t n_mad_sample, double* med_dev,
                         double* mad_dev, uint32_t* bits_dev, uint64_t* n_windows_out, void* ws_dev,
                         size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Geo g;
    QS_TRY(geometry(n_samples, sample_rate_hz, params, g));
    if (n_windows_out) *n_windows_out = g.n_win;
    QS_ARG(med_dev && mad_dev && bits_dev, "median, MAD and bits buffers are required");
    Tables tb;
    tables(g, tb);
    Bump a{(uint8_t*)ws_dev, ws_bytes, 0};
    Dev d;
    carve(a, g, tb, mad_sample_dev ? n_mad_sample : 0, d);
    QS_ARG(ws_dev && a.ok, "fingerprint workspace too small (%zu bytes)", ws_bytes);
    QS_TRY(h2d(d.tw, tb.tw, st));
    QS_TRY(h2d(d.wf_off, tb.wf_off, st));
    QS_TRY(h2d(d.wf_idx, tb.wf_idx, st));
    QS_TRY(h2d(d.wf_val, tb.wf_val, st));
    QS_TRY(h2d(d.wt_off, tb.wt_off, st));
    QS_TRY(h2d(d.wt_idx, tb.wt_idx, st));
    QS_TRY(h2d(d.wt_val, tb.wt_val, st));
    QS_TRY(h2d(d.sched, tb.sched, st));
    QS_CUDA(cudaMemsetAsync(d.flags, 0, 16, st), "memset");
    const uint32_t nlev = (uint32_t)(tb.sched.size() / 3);
    QS_TRY(qs_fp_band_stft(x_dev, x_is_f32, n_samples, g.frame, g.hop, g.n_cols, g.nb, d.tw,
                           d.band, stream));
    const uint32_t nc = g.F * g.T;
    if (mad_sample_dev) {
        QS_ARG(n_mad_sample >= 1 && n_mad_sample <= g.n_win, "MAD sample size out of range");
        QS_TRY(qs_fp_windows(d.band, g.n_cols, g.nb, mad_sample_dev, 0, n_mad_sample, g.lag, g.win,
                             g.frame, g.hop, d.wf_off, d.wf_idx, d.wf_val, d.wt_off, d.wt_idx,
                             d.wt_val, g.wmin, g.wmax, g.F, g.T, d.sched, nlev, 1, nullptr, nullptr,
                             0, d.rows, d.flags, stream));
        QS_TRY(qs_fp_transpose_f32(d.rows, n_mad_sample, nc, d.cols, stream));
        QS_TRY(qs_fp_mad(d.cols, nc, n_mad_sample, med_dev, mad_dev, d.mws, stream));
    }
    // top_k must not exceed the coefficients with a nonzero MAD (fingerprint.py:448-451)
    std::vector<double> madh(nc);
    QS_CUDA(cudaMemcpyAsync(madh.data(), mad_dev, nc * 8, cudaMemcpyDeviceToHost, st), "D2H");
    QS_CUDA(cudaStreamSynchronize(st), "sync");
    uint64_t elig = 0;
    for (double v : madh) elig += v > 0;
    QS_ARG(params->top_k <= elig, "top_k=%u exceeds %llu coefficients with nonzero MAD",
           params->top_k, (unsigned long long)elig);
    QS_TRY(qs_fp_windows(d.band, g.n_cols, g.nb, nullptr, 0, g.n_win, g.lag, g.win, g.frame, g.hop,
                         d.wf_off, d.wf_idx, d.wf_val, d.wt_off, d.wt_idx, d.wt_val, g.wmin, g.wmax,
                         g.F, g.T, d.sched, nlev, 3, med_dev, mad_dev, params->top_k, bits_dev,
                         d.flags, stream));
    uint32_t fl = 0;
    QS_CUDA(cudaMemcpyAsync(&fl, d.flags, 4, cudaMemcpyDeviceToHost, st), "D2H");
    QS_CUDA(cudaStreamSynchronize(st), "sync");
    QS_DATA(!(fl & 1), "non-finite Haar coefficient");
    return QS_OK;
}

}  // extern "C"
