// Fingerprint chain on sm_100a: band-limited STFT, spectral image, 2-D Haar,
// MAD statistics, MAD normalisation and top-K sign binarisation.
//
// Reference: fingerprint.py:125-466.  The reference computes in float64 and
// stores float32 at fixed points (spectrogram :148-149, images :239-241,
// coefficients :334); this chain computes in float64 on the CUDA cores and
// rounds to float32 at exactly those points, so the downstream float64 top-K
// sees the reference's values up to summation-order rounding.
//
//   k_band_stft     one thread per STFT column, f64 accumulators for the band
//                   bins only (a direct DFT of the band rows is cheaper than a
//                   full FFT when nb << frame/2), taper folded into the twiddles
//   k_windows       one CTA per window: band rows -> area-resampled image
//                   (sparse CSR weights) -> in-place 2-D Haar -> coefficients;
//                   mode 3 continues with (c - median)/MAD, a radix select of
//                   the K-th largest |score| and an index-ordered tie break
//   k_col_select    per-column radix select for the MAD medians
#include <math.h>

#include "qs_common.cuh"

namespace qs {

constexpr int STFT_COLS = 128;  // columns per CTA
constexpr int STFT_NBC = 16;    // band bins per register chunk
#ifndef QS_WIN_THREADS
#define QS_WIN_THREADS 256
#endif
constexpr int WIN_THREADS = QS_WIN_THREADS;

// ------------------------------------------------------------------ STFT
// bins [b_first, b_first + nb) of a table with ld_out bins per column
template <typename TX>
__global__ void __launch_bounds__(STFT_COLS) k_band_stft(const TX* __restrict__ x, uint64_t n_samples,
                                                         uint32_t frame, uint32_t hop, uint64_t n_cols,
                                                         uint32_t nb, const double* __restrict__ tw,
                                                         float* __restrict__ out, uint32_t b_first,
                                                         uint32_t ld_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* xs = (double*)smem;                                  // span of samples
    const uint32_t span = (STFT_COLS - 1) * hop + frame;
    double* tws = xs + span;                                     // [nb][frame][2]
    for (uint32_t i = threadIdx.x; i < nb * frame * 2; i += blockDim.x)
        tws[i] = tw[(uint64_t)b_first * frame * 2 + i];
    for (uint64_t c0 = (uint64_t)blockIdx.x * STFT_COLS; c0 < n_cols;
         c0 += (uint64_t)gridDim.x * STFT_COLS) {
        __syncthreads();
        const uint64_t s0 = c0 * hop;
        for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
            xs[i] = (s0 + i < n_samples) ? (double)x[s0 + i] : 0.0;
        __syncthreads();
        const uint64_t c = c0 + threadIdx.x;
        if (c < n_cols) {
            const double* xr = xs + threadIdx.x * hop;
            for (uint32_t b0 = 0; b0 < nb; b0 += STFT_NBC) {
                double re[STFT_NBC], im[STFT_NBC];
#pragma unroll
                for (int q = 0; q < STFT_NBC; ++q) re[q] = im[q] = 0.0;
                const uint32_t nbc = min((uint32_t)STFT_NBC, nb - b0);
                for (uint32_t j = 0; j < frame; ++j) {
                    const double v = xr[j];
#pragma unroll
                    for (int q = 0; q < STFT_NBC; ++q) {
                        if ((uint32_t)q < nbc) {
                            const double* t2 = tws + ((uint64_t)(b0 + q) * frame + j) * 2;
                            re[q] = fma(v, t2[0], re[q]);
                            im[q] = fma(v, t2[1], im[q]);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < STFT_NBC; ++q) {
                    if ((uint32_t)q < nbc) {
                        // power = re^2 + im^2 (no contraction), log10 in f64, stored f32
                        const double pw = __dadd_rn(__dmul_rn(re[q], re[q]), __dmul_rn(im[q], im[q]));
                        out[c * ld_out + b_first + b0 + q] = (float)log10(__dadd_rn(pw, 1e-12));
                    }
                }
            }
        }
    }
}

// --------------------------------------------------------------- windows
struct WinGeom {
    uint64_t n_cols, lag, win, win0, n_win;
    uint32_t frame, hop, nb, F, T, wmin, wmax, n_levels, top_k, mode;
};

// quotient by a warp-uniform divisor: a shift when it is a power of two (the
// Haar block sizes and time bins usually are), else a division
__device__ __forceinline__ uint32_t udiv_u(uint32_t p, uint32_t d) {
    return (d & (d - 1)) == 0 ? p >> (__ffs(d) - 1) : p / d;
}

__device__ __forceinline__ uint64_t mag_key(double s) {
    return (uint64_t)__double_as_longlong(fabs(s));  // non-negative doubles order as integers
}

// block-wide exclusive scan of one uint32 per thread (WIN_THREADS threads)
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t* wsum, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < WIN_THREADS / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const uint32_t r = (warp ? wsum[warp - 1] : 0) + x - v;
    if (total) *total = wsum[WIN_THREADS / 32 - 1];
    __syncthreads();
    return r;
}

// Top-K sign binarisation of one coefficient row held in shared memory as f64
// (fingerprint.py:433-466): v' = (c - median)/MAD (0 where MAD == 0), the K
// largest |v'| among eligible coefficients with ties to the lower index, bit
// 2j + (v' < 0), ascending.  `row` is overwritten with the scores.  Returns
// false (and writes nothing) when a coefficient is not finite.
// Radix select over keys |v'| bits + 1 (0: ineligible; recomputed from the
// scores), 8 bits per pass from the top; after each pass only the members
// matching the selected prefix stay on a candidate list (la / lb, ping-pong),
// so the later passes touch a handful of coefficients.  Scratch: la / lb
// u16[n].
__device__ bool topk_row(double* row, uint32_t n, const double* __restrict__ med,
                         const double* __restrict__ mad, uint32_t top_k, uint32_t* __restrict__ ob,
                         uint32_t* hist, uint32_t* wsum, uint64_t* s_prefix, uint32_t* s_krem,
                         uint16_t* la, uint16_t* lb, uint32_t* s_cnt) {
    bool nonfinite = false;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double c = row[i];
        if (!isfinite(c)) nonfinite = true;
        const double md = mad[i];
        // ineligible coefficients carry a NaN score (never selected; the
        // reference's 0 score is never output for them)
        row[i] = md > 0.0 ? (c - med[i]) / md : __longlong_as_double(0x7FF8000000000000ll);
    }
    // select key of coefficient i: |v'| bits + 1, 0 when ineligible
    auto key_of = [&](uint32_t i) -> uint64_t {
        const double v = row[i];
        return v != v ? 0ull : mag_key(v) + 1;
    };
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
        *s_prefix = 0;
        *s_krem = top_k;
        s_cnt[0] = 0;
    }
    if (__syncthreads_or(nonfinite)) return false;
    // pass 0: histogram of the top byte over all eligible coefficients
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t k = key_of(i);
        if (k) atomicAdd(&hist[k >> 56], 1u);
    }
    uint16_t* cur = la;
    uint16_t* nxt = lb;
    uint32_t ncur = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        __syncthreads();
        if (threadIdx.x < 32) {
            // warp 0 finds the digit holding the need-th largest key: lane l owns
            // bins [8l, 8l + 8); suffix sums over lanes, then one lane scans its bins
            const uint32_t lane = threadIdx.x, need = *s_krem;
            uint32_t c[8], sum = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                c[e] = hist[8 * lane + e];
                sum += c[e];
            }
            uint32_t x = sum;  // sum over lanes >= lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            const uint32_t above = x - sum;
            if (above < need && need <= x) {
                uint32_t cum = above;
                int dsel = 8 * lane;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    if (cum + c[e] >= need) {
                        dsel = 8 * lane + e;
                        break;
                    }
                    cum += c[e];
                }
                *s_krem = need - cum;
                *s_prefix |= (uint64_t)dsel << shift;
            }
        }
        __syncthreads();
        if (shift == 0) break;
        // keep the members matching the selected digit, histogram their next digit
        const uint32_t dsel = (uint32_t)(*s_prefix >> shift) & 0xFFu;
        for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        if (threadIdx.x == 0) s_cnt[1] = 0;
        __syncthreads();
        const uint32_t lim = shift == 56 ? n : ncur;
        for (uint32_t j = threadIdx.x; j < lim; j += blockDim.x) {
            const uint32_t i = shift == 56 ? j : cur[j];
            const uint64_t k = key_of(i);
            if (k && ((uint32_t)(k >> shift) & 0xFFu) == dsel) {
                nxt[atomicAdd(&s_cnt[1], 1u)] = (uint16_t)i;
                atomicAdd(&hist[(k >> (shift - 8)) & 0xFF], 1u);
            }
        }
        __syncthreads();
        ncur = s_cnt[1];
        uint16_t* tsw = cur;
        cur = nxt;
        nxt = tsw;
    }
    const uint64_t thr = *s_prefix;  // key of the K-th largest (>= 1: eligible)
    // greater-than count and index-ordered ranks of ties (blocked ownership)
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
    uint32_t gt = 0, eq = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint64_t k = key_of(i);
        gt += k > thr;
        eq += k == thr;
    }
    uint32_t gt_tot;
    block_scan_u32(gt, wsum, &gt_tot);
    const uint32_t need = top_k - gt_tot;
    const uint32_t eq_before = block_scan_u32(eq, wsum, nullptr);
    uint32_t sel = 0, eqr = eq_before;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint64_t k = key_of(i);
        if (k > thr) ++sel;
        else if (k == thr) {
            if (eqr < need) ++sel;
            ++eqr;
        }
    }
    uint32_t pos = block_scan_u32(sel, wsum, nullptr);
    eqr = eq_before;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint64_t k = key_of(i);
        bool take = k > thr;
        if (k == thr) {
            take = eqr < need;
            ++eqr;
        }
        if (take) ob[pos++] = 2 * i + (row[i] < 0.0 ? 1u : 0u);
    }
    return true;
}

// Shared-memory layout of k_windows (host and device agree on it): img [n]
// f64 | hs [n] f64.  hs is the Haar scratch; before the Haar it holds the
// time-resample intermediate (T x nb f64), after it the top-K candidate
// lists (2n u16).  The band rows (wmax x nb f32) live in img until the
// frequency resample overwrites it.  Anything that does not fit its alias
// gets its own region after hs.
struct WinSmem {
    size_t tmp_off, gs_off, lists_off, bytes;
};
__host__ __device__ inline WinSmem win_smem(uint32_t F, uint32_t T, uint32_t wmax, uint32_t nb) {
    const size_t n = (size_t)F * T, img = n * 8, tmp = (size_t)T * nb * 8;
    const size_t gs = (((size_t)wmax * nb + 3) & ~(size_t)3) * 4, lists = n * 4;
    size_t end = 2 * img;
    WinSmem w;
    if (tmp <= img) w.tmp_off = img;
    else { w.tmp_off = end; end += tmp; }
    if (gs <= img) w.gs_off = 0;
    else { w.gs_off = end; end += gs; }
    w.lists_off = img;  // lists <= hs always (4n <= 8n bytes)
    w.bytes = end + 16;
    return w;
}

// One CTA per window (grid-stride).  mode 0: images (B,F,T) f32; 1: coeffs
// (B,F*T) f32; 2: coeffs column-major (F*T, B) f32; 3: bits (B, K) u32.
__global__ void __launch_bounds__(WIN_THREADS) k_windows(
    const float* __restrict__ band, WinGeom g, const int64_t* __restrict__ widx,
    const int32_t* __restrict__ wf_off, const int32_t* __restrict__ wf_idx,
    const double* __restrict__ wf_val, const int32_t* __restrict__ wt_off,
    const int32_t* __restrict__ wt_idx, const double* __restrict__ wt_val,
    const int32_t* __restrict__ sched, const double* __restrict__ med,
    const double* __restrict__ mad, void* __restrict__ out, uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t F = g.F, T = g.T, nb = g.nb, n = F * T;
    // layout: see WinSmem (resample scratch and top-K lists alias hs)
    const WinSmem ly = win_smem(F, T, g.wmax, nb);
    double* img = (double*)smem;
    double* hs = img + n;
    double* tmp = (double*)(smem + ly.tmp_off);
    float* gs = (float*)(smem + ly.gs_off);
    uint16_t* lists = (uint16_t*)(smem + ly.lists_off);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_cnt[2];
    __shared__ uint32_t wsum[32];
    __shared__ uint64_t s_prefix;
    __shared__ uint32_t s_krem;
    for (uint64_t wi = blockIdx.x; wi < g.n_win; wi += gridDim.x) {
        const uint64_t idx = widx ? (uint64_t)widx[wi] : g.win0 + wi;
        const uint64_t off = idx * g.lag;
        const uint64_t c0 = (off + g.hop - 1) / g.hop;
        const uint64_t c1 = (off + g.win - g.frame) / g.hop + 1;
        const uint32_t width = (uint32_t)(c1 - c0);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < width * nb; i += blockDim.x) gs[i] = band[c0 * nb + i];
        __syncthreads();
        // time resample first (the smaller intermediate): tmp[Ti][f] =
        // sum_w w_t[Ti, w] * band[w][f]; then frequency: img[Fi][Ti] =
        // sum_f w_f[Fi, f] * tmp[Ti][f], in f64, stored f32
        const int32_t* to = wt_off + (uint64_t)(width - g.wmin) * (T + 1);
        for (uint32_t i = threadIdx.x; i < T * nb; i += blockDim.x) {
            const uint32_t Ti = udiv_u(i, nb), f = i - Ti * nb;
            double acc = 0.0;
            for (int32_t e = to[Ti]; e < to[Ti + 1]; ++e)
                acc = fma(wt_val[e], (double)gs[wt_idx[e] * nb + f], acc);
            tmp[i] = acc;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t Fi = udiv_u(i, T), Ti = i - Fi * T;
            double acc = 0.0;
            for (int32_t e = wf_off[Fi]; e < wf_off[Fi + 1]; ++e)
                acc = fma(wf_val[e], tmp[Ti * nb + wf_idx[e]], acc);
            img[i] = (double)(float)acc;
        }
        __syncthreads();
        if (g.mode == 0) {
            float* o = (float*)out + wi * n;
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) o[i] = (float)img[i];
            continue;
        }
        // 2-D Haar (fingerprint.py:256-300): per level a row pass over the
        // (h, w) block then a column pass, each out of place through hs.
        const double s2 = 0.7071067811865475;  // 1.0 / math.sqrt(2.0), as the reference
        for (uint32_t lv = 0; lv < g.n_levels; ++lv) {
            const uint32_t h = sched[3 * lv], w = sched[3 * lv + 1], lmode = sched[3 * lv + 2];
            if (lmode & 1u) {  // rows (time axis)
                const uint32_t half = w / 2;
                for (uint32_t p = threadIdx.x; p < h * half; p += blockDim.x) {
                    const uint32_t r = udiv_u(p, half), j = p - r * half;
                    const double ev = img[r * T + 2 * j], od = img[r * T + 2 * j + 1];
                    hs[r * T + j] = (ev + od) * s2;
                    hs[r * T + half + j] = (ev - od) * s2;
                }
                __syncthreads();
                for (uint32_t p = threadIdx.x; p < h * w; p += blockDim.x) {
                    const uint32_t r = udiv_u(p, w), c = p - r * w;
                    img[r * T + c] = hs[r * T + c];
                }
                __syncthreads();
            }
            if (lmode & 2u) {  // columns (frequency axis)
                const uint32_t half = h / 2;
                for (uint32_t p = threadIdx.x; p < half * w; p += blockDim.x) {
                    const uint32_t i2 = udiv_u(p, w), c = p - i2 * w;
                    const double ev = img[(2 * i2) * T + c], od = img[(2 * i2 + 1) * T + c];
                    hs[i2 * T + c] = (ev + od) * s2;
                    hs[(half + i2) * T + c] = (ev - od) * s2;
                }
                __syncthreads();
                for (uint32_t p = threadIdx.x; p < h * w; p += blockDim.x) {
                    const uint32_t r = udiv_u(p, w), c = p - r * w;
                    img[r * T + c] = hs[r * T + c];
                }
                __syncthreads();
            }
        }
        // coefficients are stored float32 by the reference (fingerprint.py:334)
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) img[i] = (double)(float)img[i];
        __syncthreads();
        if (g.mode == 1) {
            float* o = (float*)out + wi * n;
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) o[i] = (float)img[i];
            continue;
        }
        if (g.mode == 2) {
            float* o = (float*)out;
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) o[(uint64_t)i * g.n_win + wi] = (float)img[i];
            continue;
        }
        // ---- mode 3: scores, K-th largest |score| (radix select), bits
        if (!topk_row(img, n, med, mad, g.top_k, (uint32_t*)out + wi * g.top_k, hist, wsum,
                      &s_prefix, &s_krem, lists, lists + n, s_cnt))
            if (threadIdx.x == 0) atomicOr(flags, 1u);
    }
}

// ------------------------------------------------------------ MAD select
// Order statistic k of each column (n_cols columns of S values).  mode 0:
// values x (f32 widened to f64); mode 1: |x - center[col]| (f64).  Radix
// select over order-preserving 64-bit keys of the f64 values.
__device__ __forceinline__ uint64_t ord_key(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_val(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)b);
}

__global__ void __launch_bounds__(512) k_col_select(const float* __restrict__ cols, uint64_t S,
                                                    uint64_t k, int mode,
                                                    const double* __restrict__ center,
                                                    double* __restrict__ out) {
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix, s_krem;
    const uint32_t col = blockIdx.x;
    const float* c = cols + (uint64_t)col * S;
    const double ctr = mode ? center[col] : 0.0;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_krem = k;  // 0-based rank among ascending keys
    }
    uint64_t pmask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (uint64_t i = threadIdx.x; i < S; i += blockDim.x) {
            const double v = mode ? fabs((double)c[i] - ctr) : (double)c[i];
            const uint64_t kk = ord_key(v);
            if ((kk & pmask) == prefix) atomicAdd(&hist[(kk >> shift) & 0xFF], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t rem = s_krem, cum = 0;
            int dsel = 255;
            for (int dgt = 0; dgt < 256; ++dgt) {
                if (cum + hist[dgt] > rem) {
                    dsel = dgt;
                    break;
                }
                cum += hist[dgt];
            }
            s_krem = rem - cum;
            s_prefix = prefix | ((uint64_t)dsel << shift);
        }
        pmask |= (uint64_t)0xFF << shift;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[col] = key_val(s_prefix);
}

__global__ void k_mid_mean(const double* __restrict__ a, const double* __restrict__ b, uint32_t n,
                           double* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (a[i] + b[i]) / 2.0;  // np.median of an even count
}

template <typename TC>
__global__ void k_normalize(const TC* __restrict__ c, uint64_t total, uint32_t n,
                            const double* __restrict__ med, const double* __restrict__ mad,
                            double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i % n);
        const double md = mad[j];
        out[i] = md > 0.0 ? ((double)c[i] - med[j]) / md : 0.0;
    }
}

// top-K bits of arbitrary coefficient rows (topk_bits API), one CTA per row
template <typename TC>
__global__ void __launch_bounds__(WIN_THREADS) k_topk_rows(const TC* __restrict__ c, uint64_t B,
                                                           uint32_t n, const double* __restrict__ med,
                                                           const double* __restrict__ mad,
                                                           uint32_t top_k, uint32_t* __restrict__ out,
                                                           uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* row = (double*)smem;
    uint16_t* lists = (uint16_t*)(row + n);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t wsum[32];
    __shared__ uint64_t s_prefix;
    __shared__ uint32_t s_krem;
    __shared__ uint32_t s_cnt[2];
    for (uint64_t r = blockIdx.x; r < B; r += gridDim.x) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) row[i] = (double)c[r * n + i];
        __syncthreads();
        if (!topk_row(row, n, med, mad, top_k, out + r * top_k, hist, wsum, &s_prefix, &s_krem,
                      lists, lists + n, s_cnt))
            if (threadIdx.x == 0) atomicOr(flags, 1u);
    }
}

// batched 2-D Haar / inverse on f64 (H, W) images in place, one CTA per image
__global__ void __launch_bounds__(WIN_THREADS) k_haar_batch(double* __restrict__ data, uint64_t B,
                                                            uint32_t H, uint32_t W,
                                                            const int32_t* __restrict__ sched,
                                                            uint32_t n_levels, int inverse) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t n = H * W;
    double* img = (double*)smem;
    double* hs = img + n;
    const double s2 = 0.7071067811865475;
    for (uint64_t b = blockIdx.x; b < B; b += gridDim.x) {
        double* d = data + b * n;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) img[i] = d[i];
        __syncthreads();
        for (uint32_t l = 0; l < n_levels; ++l) {
            const uint32_t lv = inverse ? n_levels - 1 - l : l;
            const uint32_t h = sched[3 * lv], w = sched[3 * lv + 1], lmode = sched[3 * lv + 2];
            for (int step = 0; step < 2; ++step) {
                // forward: rows then columns; inverse: columns then rows
                const bool rows = inverse ? (step == 1) : (step == 0);
                if (!(lmode & (rows ? 1u : 2u))) continue;
                if (rows) {
                    const uint32_t half = w / 2;
                    for (uint32_t p = threadIdx.x; p < h * half; p += blockDim.x) {
                        const uint32_t r = udiv_u(p, half), j = p - r * half;
                        if (!inverse) {
                            const double ev = img[r * W + 2 * j], od = img[r * W + 2 * j + 1];
                            hs[r * W + j] = (ev + od) * s2;
                            hs[r * W + half + j] = (ev - od) * s2;
                        } else {
                            const double sv = img[r * W + j], dv = img[r * W + half + j];
                            hs[r * W + 2 * j] = (sv + dv) * s2;
                            hs[r * W + 2 * j + 1] = (sv - dv) * s2;
                        }
                    }
                } else {
                    const uint32_t half = h / 2;
                    for (uint32_t p = threadIdx.x; p < half * w; p += blockDim.x) {
                        const uint32_t i2 = udiv_u(p, w), c = p - i2 * w;
                        if (!inverse) {
                            const double ev = img[(2 * i2) * W + c], od = img[(2 * i2 + 1) * W + c];
                            hs[i2 * W + c] = (ev + od) * s2;
                            hs[(half + i2) * W + c] = (ev - od) * s2;
                        } else {
                            const double sv = img[i2 * W + c], dv = img[(half + i2) * W + c];
                            hs[(2 * i2) * W + c] = (sv + dv) * s2;
                            hs[(2 * i2 + 1) * W + c] = (sv - dv) * s2;
                        }
                    }
                }
                __syncthreads();
                for (uint32_t p = threadIdx.x; p < h * w; p += blockDim.x) {
                    const uint32_t r = udiv_u(p, w), c = p - r * w;
                    img[r * W + c] = hs[r * W + c];
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = img[i];
    }
}

}  // namespace qs

using namespace qs;

// ------------------------------------------------------ .fp record packing
// record r (16 + 4K bytes, fingerprint.py:549-551): index u64 | epoch f64 |
// bits u32[K], little endian; one thread per 32-bit output word (coalesced).
__global__ void k_fp_pack(const uint64_t* __restrict__ idx, const double* __restrict__ ep,
                          const uint32_t* __restrict__ bits, uint64_t n, uint32_t K,
                          uint32_t* __restrict__ out) {
    const uint64_t words = n * (4ull + K);
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = w / (4ull + K);
        const uint32_t c = (uint32_t)(w - r * (4ull + K));
        uint32_t v;
        if (c < 2) v = (uint32_t)(idx[r] >> (32 * c));
        else if (c < 4) v = (uint32_t)(__double_as_longlong(ep[r]) >> (32 * (c - 2)));
        else v = bits[r * K + (c - 4)];
        out[w] = v;
    }
}

__global__ void k_fp_unpack(const uint32_t* __restrict__ in, uint64_t n, uint32_t K,
                            uint64_t* __restrict__ idx, double* __restrict__ ep,
                            uint32_t* __restrict__ bits) {
    const uint64_t words = n * (4ull + K);
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = w / (4ull + K);
        const uint32_t c = (uint32_t)(w - r * (4ull + K));
        if (c == 0) idx[r] = (uint64_t)in[w] | ((uint64_t)in[w + 1] << 32);
        else if (c == 2)
            ep[r] = __longlong_as_double((long long)((uint64_t)in[w] | ((uint64_t)in[w + 1] << 32)));
        else if (c >= 4) bits[r * K + (c - 4)] = in[w];
    }
}

extern "C" {

int qs_fp_band_stft(const void* x_dev, int x_is_f32, uint64_t n_samples, uint32_t frame,
                    uint32_t hop, uint64_t n_cols, uint32_t nb, const double* tw_dev,
                    float* out_dev, void* stream) {
    QS_ARG(frame >= 2 && hop >= 1 && nb >= 1, "bad STFT geometry");
    if (n_cols == 0) return QS_OK;
    QS_ARG((n_cols - 1) * hop + frame <= n_samples, "series shorter than the STFT columns");
    const size_t span_bytes = (size_t)((STFT_COLS - 1) * hop + frame) * 8;
    // bins per launch so that samples + twiddles fit in shared memory
    uint32_t chunk = nb;
    while (chunk > 1 && span_bytes + (size_t)chunk * frame * 16 > 200 * 1024) chunk = (chunk + 1) / 2;
    QS_ARG(span_bytes + (size_t)chunk * frame * 16 <= 200 * 1024, "STFT frame too long");
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t blocks = (n_cols + STFT_COLS - 1) / STFT_COLS;
    const unsigned grid = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
    for (uint32_t b0 = 0; b0 < nb; b0 += chunk) {
        const uint32_t nbc = min(chunk, nb - b0);
        const size_t smem = span_bytes + (size_t)nbc * frame * 16;
        if (x_is_f32) {
            QS_CUDA(cudaFuncSetAttribute(k_band_stft<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
            k_band_stft<float><<<grid, STFT_COLS, smem, st>>>((const float*)x_dev, n_samples, frame,
                                                             hop, n_cols, nbc, tw_dev, out_dev, b0, nb);
        } else {
            QS_CUDA(cudaFuncSetAttribute(k_band_stft<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
            k_band_stft<double><<<grid, STFT_COLS, smem, st>>>((const double*)x_dev, n_samples, frame,
                                                              hop, n_cols, nbc, tw_dev, out_dev, b0, nb);
        }
        QS_CHECK_LAUNCH("k_band_stft");
    }
    return QS_OK;
}

int qs_fp_windows(const float* band_dev, uint64_t n_cols, uint32_t nb, const int64_t* widx_dev,
                  uint64_t win0, uint64_t n_win, uint64_t lag, uint64_t win, uint32_t frame,
                  uint32_t hop, const int32_t* wf_off, const int32_t* wf_idx, const double* wf_val,
                  const int32_t* wt_off, const int32_t* wt_idx, const double* wt_val,
                  uint32_t wmin, uint32_t wmax, uint32_t F, uint32_t T, const int32_t* sched_dev,
                  uint32_t n_levels, int mode, const double* med_dev, const double* mad_dev,
                  uint32_t top_k, void* out_dev, uint32_t* flags_dev, void* stream) {
    QS_ARG(mode >= 0 && mode <= 3, "mode must be 0..3");
    QS_ARG(F >= 1 && T >= 1 && nb >= 1 && wmin >= 1 && wmax >= wmin, "bad window geometry");
    QS_ARG(mode != 3 || (top_k >= 1 && top_k <= F * T), "bad top_k");
    if (n_win == 0) return QS_OK;
    (void)n_cols;
    const size_t smem = win_smem(F, T, wmax, nb).bytes;
    QS_ARG(smem <= 200 * 1024, "spectral image too large for the window kernel");
    QS_CUDA(cudaFuncSetAttribute(k_windows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    WinGeom g{n_cols, lag, win, win0, n_win, frame, hop, nb, F, T, wmin, wmax, n_levels, top_k,
              (uint32_t)mode};
    const unsigned grid = (unsigned)(n_win < 148 * 32 ? n_win : 148 * 32);
    k_windows<<<grid, WIN_THREADS, smem, (cudaStream_t)stream>>>(
        band_dev, g, widx_dev, wf_off, wf_idx, wf_val, wt_off, wt_idx, wt_val, sched_dev, med_dev,
        mad_dev, out_dev, flags_dev);
    QS_CHECK_LAUNCH("k_windows");
    return QS_OK;
}

int qs_fp_mad(const float* cols_dev, uint32_t n_coeffs, uint64_t S, double* med_dev,
              double* mad_dev, double* ws_dev, void* stream) {
    QS_ARG(S >= 1 && n_coeffs >= 1, "empty MAD sample");
    cudaStream_t st = (cudaStream_t)stream;
    double* a = ws_dev;
    double* b = ws_dev + n_coeffs;
    for (int pass = 0; pass < 2; ++pass) {
        double* dst = pass == 0 ? med_dev : mad_dev;
        if (S & 1) {
            k_col_select<<<n_coeffs, 512, 0, st>>>(cols_dev, S, S / 2, pass, med_dev, dst);
        } else {
            k_col_select<<<n_coeffs, 512, 0, st>>>(cols_dev, S, S / 2 - 1, pass, med_dev, a);
            k_col_select<<<n_coeffs, 512, 0, st>>>(cols_dev, S, S / 2, pass, med_dev, b);
            k_mid_mean<<<(n_coeffs + 255) / 256, 256, 0, st>>>(a, b, n_coeffs, dst);
        }
    }
    QS_CHECK_LAUNCH("qs_fp_mad");
    return QS_OK;
}

int qs_fp_topk_bits(const void* coeffs_dev, int is_f64, uint64_t B, uint32_t n,
                    const double* med_dev, const double* mad_dev, uint32_t top_k, uint32_t* out_dev,
                    uint32_t* flags_dev, void* stream) {
    QS_ARG(top_k >= 1 && top_k <= n, "top_k must be in [1, n]");
    if (B == 0) return QS_OK;
    const size_t smem = (size_t)n * 12;  // row f64 + two u16 candidate lists
    QS_ARG(smem <= 200 * 1024, "coefficient rows too long");
    const unsigned grid = (unsigned)(B < 148 * 32 ? B : 148 * 32);
    cudaStream_t st = (cudaStream_t)stream;
    if (is_f64) {
        QS_CUDA(cudaFuncSetAttribute(k_topk_rows<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        k_topk_rows<double><<<grid, WIN_THREADS, smem, st>>>((const double*)coeffs_dev, B, n, med_dev,
                                                            mad_dev, top_k, out_dev, flags_dev);
    } else {
        QS_CUDA(cudaFuncSetAttribute(k_topk_rows<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        k_topk_rows<float><<<grid, WIN_THREADS, smem, st>>>((const float*)coeffs_dev, B, n, med_dev,
                                                           mad_dev, top_k, out_dev, flags_dev);
    }
    QS_CHECK_LAUNCH("k_topk_rows");
    return QS_OK;
}

int qs_fp_haar2d(double* data_dev, uint64_t B, uint32_t H, uint32_t W, const int32_t* sched_dev,
                 uint32_t n_levels, int inverse, void* stream) {
    if (B == 0 || n_levels == 0) return QS_OK;
    const size_t smem = (size_t)H * W * 16;
    QS_ARG(smem <= 200 * 1024, "haar2d image too large for the GPU kernel (H*W <= 12800)");
    QS_CUDA(cudaFuncSetAttribute(k_haar_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    const unsigned grid = (unsigned)(B < 148 * 32 ? B : 148 * 32);
    k_haar_batch<<<grid, WIN_THREADS, smem, (cudaStream_t)stream>>>(data_dev, B, H, W, sched_dev,
                                                                   n_levels, inverse);
    QS_CHECK_LAUNCH("k_haar_batch");
    return QS_OK;
}

int qs_fp_normalize(const void* coeffs_dev, int is_f64, uint64_t B, uint32_t n,
                    const double* med_dev, const double* mad_dev, double* out_dev, void* stream) {
    if (B == 0) return QS_OK;
    const unsigned g = qs_blocks(B * n, 256);
    if (is_f64)
        k_normalize<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)coeffs_dev, B * n, n,
                                                                 med_dev, mad_dev, out_dev);
    else
        k_normalize<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)coeffs_dev, B * n, n,
                                                                med_dev, mad_dev, out_dev);
    QS_CHECK_LAUNCH("k_normalize");
    return QS_OK;
}

int qs_fp_pack_records(const uint64_t* indices_dev, const double* epochs_dev,
                       const uint32_t* bits_dev, uint64_t n, uint32_t K, uint8_t* out_dev,
                       void* stream) {
    QS_ARG(K >= 1, "top_k must be >= 1");
    if (n == 0) return QS_OK;
    k_fp_pack<<<qs_blocks(n * (4ull + K), 256), 256, 0, (cudaStream_t)stream>>>(
        indices_dev, epochs_dev, bits_dev, n, K, (uint32_t*)out_dev);
    QS_CHECK_LAUNCH("k_fp_pack");
    return QS_OK;
}

int qs_fp_unpack_records(const uint8_t* in_dev, uint64_t n, uint32_t K, uint64_t* indices_dev,
                         double* epochs_dev, uint32_t* bits_dev, void* stream) {
    QS_ARG(K >= 1, "top_k must be >= 1");
    if (n == 0) return QS_OK;
    k_fp_unpack<<<qs_blocks(n * (4ull + K), 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint32_t*)in_dev, n, K, indices_dev, epochs_dev, bits_dev);
    QS_CHECK_LAUNCH("k_fp_unpack");
    return QS_OK;
}

}  // extern "C"
