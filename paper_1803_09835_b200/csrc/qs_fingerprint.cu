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
#include <stdlib.h>

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

// ------------------------------------------------- STFT on the FP64 tensor cores
// The band DFT is a dense contraction: out[c][n] = sum_j X[c][j] B[j][n] with
// X[c][j] = x[c hop + j] (a Toeplitz view of the trace, K = frame) and
// B[j][2b + r] the tapered twiddles of band bin b (r = 0: cos, 1: -sin).  One
// warp computes SM_MT m-tiles of 8 columns against 4 n-tiles of 8 outputs per
// k-step of 4 samples with DMMA (mma.sync m8n8k4 f64: A row = lane / 4,
// k = lane % 4; B k = lane % 4, n = lane / 4; C row = lane / 4, n = 2 (lane %
// 4) + {0, 1}, i.e. each lane ends with the (re, im) pair of one bin of one
// column).  B is staged once per CTA in fragment order (conflict-free 8-byte
// loads), the samples per 256-column slab as f64.  Padded k (frame % 4) reads
// zero samples; padded n reads zero twiddles.  Summation order differs from
// the FMA chain only at f64 rounding level; power, log10 and the f32 store
// are the same as k_band_stft.
constexpr int SM_WARPS = 8, SM_MT = 4;
constexpr int SM_COLS = SM_WARPS * SM_MT * 8;  // 256 columns per slab

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <typename TX>
__global__ void __launch_bounds__(SM_WARPS * 32, 2) k_band_stft_mma(
    const TX* __restrict__ x, uint64_t n_samples, uint32_t frame, uint32_t hop, uint64_t n_cols,
    uint32_t nb, const double* __restrict__ tw, float* __restrict__ out, uint32_t b_first,
    uint32_t ld_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ksteps = (frame + 3) / 4;
    const uint32_t ntiles = (2 * nb + 7) / 8;            // n-tiles of 8 outputs
    const uint32_t ngroups = (ntiles + 3) / 4;           // 4 n-tiles per pass
    double* bs = (double*)smem;                           // [ksteps][ngroups * 4][32]
    const uint32_t nt_pad = ngroups * 4;
    double* xs = bs + (uint64_t)ksteps * nt_pad * 32;     // slab samples
    const uint32_t span = (SM_COLS - 1) * hop + ksteps * 4;
    for (uint32_t i = threadIdx.x; i < ksteps * nt_pad * 32; i += blockDim.x) {
        const uint32_t l = i & 31, q = (i >> 5) % nt_pad, ks = (i >> 5) / nt_pad;
        const uint32_t k = ks * 4 + (l & 3), n = q * 8 + (l >> 2), b = n >> 1;
        bs[i] = (k < frame && b < nb) ? tw[((uint64_t)(b_first + b) * frame + k) * 2 + (n & 1)] : 0.0;
    }
    const uint32_t row = lane >> 2, kq = lane & 3;
    for (uint64_t c0 = (uint64_t)blockIdx.x * SM_COLS; c0 < n_cols;
         c0 += (uint64_t)gridDim.x * SM_COLS) {
        __syncthreads();
        const uint64_t s0 = c0 * hop;
        for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
            xs[i] = (s0 + i < n_samples) ? (double)x[s0 + i] : 0.0;
        __syncthreads();
        const uint32_t cl0 = warp * SM_MT * 8 + row;      // this lane's A row, m-tile 0
        for (uint32_t gq = 0; gq < ngroups; ++gq) {
            double acc[SM_MT][4][2];
#pragma unroll
            for (int mt = 0; mt < SM_MT; ++mt)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[mt][q][0] = acc[mt][q][1] = 0.0;
            const double* bq = bs + (uint64_t)gq * 4 * 32 + lane;
            for (uint32_t ks = 0; ks < ksteps; ++ks) {
                const uint32_t k = ks * 4 + kq;
                double a[SM_MT], b[4];
#pragma unroll
                for (int mt = 0; mt < SM_MT; ++mt)
                    a[mt] = k < frame ? xs[(cl0 + mt * 8) * hop + k] : 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) b[q] = bq[((uint64_t)ks * nt_pad + q) * 32];
#pragma unroll
                for (int mt = 0; mt < SM_MT; ++mt)
#pragma unroll
                    for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[mt][q][0], acc[mt][q][1], a[mt], b[q]);
            }
#pragma unroll
            for (int mt = 0; mt < SM_MT; ++mt) {
                const uint64_t c = c0 + cl0 + mt * 8;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t bin = (gq * 4 + q) * 4 + kq;
                    if (c < n_cols && bin < nb) {
                        const double re = acc[mt][q][0], im = acc[mt][q][1];
                        // power = re^2 + im^2 (no contraction), log10 in f64, stored f32
                        const double pw = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
                        out[c * ld_out + b_first + bin] = (float)log10(__dadd_rn(pw, 1e-12));
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


// ------------------------------------------------- one warp per window
// The BASELINE geometry (32 x 64 images, <= 16 band rows): one WARP per
// window and no block barriers.  Lane l owns the 8 x 8 pixel tile (8 (l >> 3),
// 8 (l & 7)): it computes its pixels straight from the time-resampled band
// (f64, per-warp shared memory), runs Haar levels 1-3 in registers — the
// 2-D Haar of fingerprint.py:256-300 is, per level, a 2 x 2 butterfly per
// block (row pass then column pass, the reference's operation order), and
// only the low-low value feeds the next level — and levels 4-6 with
// shuffles.  Coefficients are rounded to f32 where the reference rounds
// (:334), then written out (modes 1, 2) or turned into select keys (mode 3:
// |v'| bits + 1, 0 when ineligible, the sign of v' in bit 63) in a per-warp
// array; the K-th largest key is found by a warp radix select (8-bit digits
// from the first byte where the eligible keys differ; candidate lists by
// ordered ballot compaction) and the bits are emitted in index order by
// ballots over the 64 key words.  The resize weights are padded to fixed tap
// counts per output (zero weights add exact zeros).
constexpr int WW_WARPS = 8;
constexpr uint32_t WW_N = 2048, WW_T = 64, WW_NBMAX = 16;
constexpr uint32_t WW_FT = 2, WW_TT = 3, WW_NWID = 3;  // taps per w_f / w_t output, widths
constexpr size_t WW_WARP_BYTES = WW_N * 8 + WW_T * WW_NBMAX * 8 + 256 * 4;  // keys | tmp/lists | hist
constexpr size_t WW_TAB_BYTES = (32 * WW_FT + WW_NWID * WW_T * WW_TT) * 12 + 64;
constexpr uint64_t WW_SIGN = 1ull << 63;

__global__ void __launch_bounds__(WW_WARPS * 32, 1) k_win_warp(
    const float* __restrict__ band, WinGeom g, const int64_t* __restrict__ widx,
    const int32_t* __restrict__ wf_off, const int32_t* __restrict__ wf_idx,
    const double* __restrict__ wf_val, const int32_t* __restrict__ wt_off,
    const int32_t* __restrict__ wt_idx, const double* __restrict__ wt_val,
    const double* __restrict__ med, const double* __restrict__ mad, void* __restrict__ out,
    uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) unsigned char wsm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    // padded resize tables, once per CTA: tap t of output r at [r * taps + t]
    double* fv = (double*)wsm;                                    // [32][WW_FT]
    double* tv = fv + 32 * WW_FT;                                 // [widths][64][WW_TT]
    int32_t* fi = (int32_t*)(tv + WW_NWID * WW_T * WW_TT);        // [32][WW_FT]
    int32_t* ti = fi + 32 * WW_FT;                                // [widths][64][WW_TT]
    const uint32_t nwid = g.wmax - g.wmin + 1;
    for (uint32_t q = threadIdx.x; q < 32 * WW_FT; q += blockDim.x) {
        const uint32_t r = q / WW_FT, t = q - r * WW_FT;
        const int32_t e = wf_off[r] + (int32_t)t;
        const bool ok = e < wf_off[r + 1];
        fv[q] = ok ? wf_val[e] : 0.0;
        fi[q] = ok ? wf_idx[e] : 0;
    }
    for (uint32_t q = threadIdx.x; q < nwid * WW_T * WW_TT; q += blockDim.x) {
        const uint32_t row = q / WW_TT, t = q - row * WW_TT;       // row = width * 64 + Ti
        const uint32_t wd = row / WW_T, Ti = row - wd * WW_T;
        const int32_t* to = wt_off + (uint64_t)wd * (WW_T + 1);
        const int32_t e = to[Ti] + (int32_t)t;
        const bool ok = e < to[Ti + 1];
        tv[q] = ok ? wt_val[e] : 0.0;
        ti[q] = ok ? wt_idx[e] : 0;
    }
    __syncthreads();
    unsigned char* base = wsm + WW_TAB_BYTES + (size_t)warp * WW_WARP_BYTES;
    uint64_t* keys = (uint64_t*)base;                                 // [2048]
    double* tmp = (double*)(base + WW_N * 8);                         // [T][nb]
    uint16_t* la = (uint16_t*)tmp;                                    // lists alias tmp
    uint16_t* lb = la + WW_N;
    uint32_t* hist = (uint32_t*)(base + WW_N * 8 + WW_T * WW_NBMAX * 8);
    const uint32_t nb = g.nb, mode = g.mode;
    const double s2 = 0.7071067811865475;  // 1.0 / math.sqrt(2.0), as the reference
    const uint32_t tr = lane >> 3, tc = lane & 7;
    const uint64_t nwarp = (uint64_t)gridDim.x * WW_WARPS;
    for (uint64_t wi = (uint64_t)blockIdx.x * WW_WARPS + warp; wi < g.n_win; wi += nwarp) {
        const uint64_t idx = widx ? (uint64_t)widx[wi] : g.win0 + wi;
        const uint64_t off = idx * g.lag;
        const uint64_t c0 = (off + g.hop - 1) / g.hop;
        const uint64_t c1 = (off + g.win - g.frame) / g.hop + 1;
        const uint32_t width = (uint32_t)(c1 - c0);
        // band rows of the window -> per-warp shared memory (aliases the keys,
        // dead until the Haar), all loads in flight at once
        const float* bw = band + c0 * nb;
        float* gs = (float*)keys;
        __syncwarp();
        for (uint32_t i = lane; i < width * nb; i += 32) gs[i] = __ldg(bw + i);
        __syncwarp();
        // time resample: tmp[Ti][f] = sum_w w_t[Ti, w] band[w][f] (f64, CSR order)
        const double* tvw = tv + (uint64_t)(width - g.wmin) * WW_T * WW_TT;
        const int32_t* tiw = ti + (uint64_t)(width - g.wmin) * WW_T * WW_TT;
#pragma unroll 1
        for (uint32_t i = lane; i < WW_T * nb; i += 32) {
            const uint32_t Ti = i / nb, f = i - Ti * nb;
            double acc = 0.0;
#pragma unroll
            for (uint32_t t = 0; t < WW_TT; ++t)
                acc = fma(tvw[Ti * WW_TT + t], (double)gs[tiw[Ti * WW_TT + t] * nb + f], acc);
            tmp[i] = acc;
        }
        __syncwarp();
        bool nonfinite = false;
        uint64_t kmax = 0, kmin = ~0ull;
        auto emit = [&](uint32_t j, double v) {
            const float c = (float)v;  // coefficients are stored float32 (fingerprint.py:334)
            if (mode == 1) {
                ((float*)out)[wi * WW_N + j] = c;
            } else if (mode == 2) {
                ((float*)out)[(uint64_t)j * g.n_win + wi] = c;
            } else {
                const double cd = (double)c;
                if (!isfinite(cd)) nonfinite = true;
                const double md = __ldg(mad + j);
                uint64_t k = 0;
                if (md > 0.0) {
                    const double sc = __ddiv_rn(__dsub_rn(cd, __ldg(med + j)), md);
                    const uint64_t m = mag_key(sc) + 1;
                    kmax = m > kmax ? m : kmax;
                    kmin = m < kmin ? m : kmin;
                    k = m | (sc < 0.0 ? WW_SIGN : 0ull);
                }
                keys[j] = k;
            }
        };
        // 2 x 2 butterfly of one Haar level block [x00 x01; x10 x11] at block
        // (bi, bj) of an (h, w) level: emits LH, HL, HH, returns LL; explicit
        // round-to-nearest ops (no FMA contraction: the reference rounds every
        // add and multiply, and exact structural zeros depend on it)
        auto bfly = [&](double x00, double x01, double x10, double x11, uint32_t bi, uint32_t bj,
                        uint32_t h, uint32_t w) -> double {
            const double lo0 = __dmul_rn(__dadd_rn(x00, x01), s2), hi0 = __dmul_rn(__dsub_rn(x00, x01), s2);
            const double lo1 = __dmul_rn(__dadd_rn(x10, x11), s2), hi1 = __dmul_rn(__dsub_rn(x10, x11), s2);
            emit(bi * WW_T + w / 2 + bj, __dmul_rn(__dadd_rn(hi0, hi1), s2));
            emit((h / 2 + bi) * WW_T + bj, __dmul_rn(__dsub_rn(lo0, lo1), s2));
            emit((h / 2 + bi) * WW_T + w / 2 + bj, __dmul_rn(__dsub_rn(hi0, hi1), s2));
            return __dmul_rn(__dadd_rn(lo0, lo1), s2);
        };
        double q00 = 0, q01 = 0, q10 = 0, q11 = 0;  // LL2 of the four 4 x 4 sub-tiles
#pragma unroll 1
        for (uint32_t st = 0; st < 4; ++st) {
            const uint32_t si = st >> 1, sj = st & 1;
            double px[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const uint32_t r = 8 * tr + 4 * si + a;
                const double w0 = fv[r * WW_FT], w1 = fv[r * WW_FT + 1];
                const uint32_t i0 = fi[r * WW_FT], i1 = fi[r * WW_FT + 1];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t c = 8 * tc + 4 * sj + b;
                    const double acc = fma(w1, tmp[c * nb + i1], fma(w0, tmp[c * nb + i0], 0.0));
                    px[a][b] = (double)(float)acc;  // images are float32 (fingerprint.py:239-241)
                }
            }
            double l1[2][2];
#pragma unroll
            for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2)
                    l1[a2][b2] = bfly(px[2 * a2][2 * b2], px[2 * a2][2 * b2 + 1], px[2 * a2 + 1][2 * b2],
                                      px[2 * a2 + 1][2 * b2 + 1], 4 * tr + 2 * si + a2,
                                      4 * tc + 2 * sj + b2, 32, 64);
            const double l2 = bfly(l1[0][0], l1[0][1], l1[1][0], l1[1][1], 2 * tr + si, 2 * tc + sj, 16, 32);
            q00 = st == 0 ? l2 : q00;
            q01 = st == 1 ? l2 : q01;
            q10 = st == 2 ? l2 : q10;
            q11 = st == 3 ? l2 : q11;
        }
        const double ll3 = bfly(q00, q01, q10, q11, tr, tc, 8, 16);
        // level 4 (4 x 8): 2 x 2 lane blocks, computed by the even (tr, tc) lanes
        const double n01 = __shfl_down_sync(0xffffffffu, ll3, 1);
        const double n10 = __shfl_down_sync(0xffffffffu, ll3, 8);
        const double n11 = __shfl_down_sync(0xffffffffu, ll3, 9);
        double ll4 = 0.0;
        if (!(tr & 1) && !(tc & 1)) ll4 = bfly(ll3, n01, n10, n11, tr / 2, tc / 2, 4, 8);
        // level 5 (2 x 4): LL4 of block (bi4, bj4) lives in lane 16 bi4 + 2 bj4
        const double m01 = __shfl_down_sync(0xffffffffu, ll4, 2);
        const double m10 = __shfl_down_sync(0xffffffffu, ll4, 16);
        const double m11 = __shfl_down_sync(0xffffffffu, ll4, 18);
        double ll5 = 0.0;
        if (lane == 0 || lane == 4) ll5 = bfly(ll4, m01, m10, m11, 0, lane / 4, 2, 4);
        // level 6 (1 x 2, row pass only)
        const double x1 = __shfl_down_sync(0xffffffffu, ll5, 4);
        if (lane == 0) {
            emit(0, __dmul_rn(__dadd_rn(ll5, x1), s2));
            emit(1, __dmul_rn(__dsub_rn(ll5, x1), s2));
        }
        if (mode != 3) continue;
        if (__any_sync(0xffffffffu, nonfinite)) {
            if (lane == 0) atomicOr(flags, 1u);
            continue;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t a2 = __shfl_xor_sync(0xffffffffu, kmax, o);
            const uint64_t b2 = __shfl_xor_sync(0xffffffffu, kmin, o);
            kmax = a2 > kmax ? a2 : kmax;
            kmin = b2 < kmin ? b2 : kmin;
        }
        __syncwarp();
        // ---- the K-th largest key by radix select; bytes above the first one
        // where eligible keys differ are common to all of them
        int shift = 56;
        while (shift > 0 && ((kmax ^ kmin) >> shift) == 0) shift -= 8;
        uint64_t prefix = shift < 56 ? (kmax >> (shift + 8)) << (shift + 8) : 0ull;
        uint32_t krem = g.top_k, ncur = WW_N, gt = 0;
        bool full = true;  // candidates: every coefficient, else the list la
        for (;; shift -= 8) {
            for (uint32_t i = lane; i < 256; i += 32) hist[i] = 0;
            __syncwarp();
            const uint64_t hmask = shift < 56 ? ~0ull << (shift + 8) : 0ull;
            for (uint32_t j0 = 0; j0 < ncur; j0 += 32) {
                const uint32_t jj = j0 + lane;
                uint32_t d = 256;
                if (jj < ncur) {
                    const uint64_t k = keys[full ? jj : la[jj]] & ~WW_SIGN;
                    if (k && (k & hmask) == prefix) d = (uint32_t)(k >> shift) & 0xFFu;
                }
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                if (d < 256 && (peers & lt) == 0) atomicAdd(&hist[d], __popc(peers));
            }
            __syncwarp();
            // the digit holding the krem-th largest: lane l owns bins [8l, 8l + 8)
            uint32_t c[8], sum = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                c[e] = hist[8 * lane + e];
                sum += c[e];
            }
            uint32_t x = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            const uint32_t above = x - sum;
            uint32_t dsel = 0, knew = 0, cgt = 0;
            const bool mine = above < krem && krem <= x;
            if (mine) {
                uint32_t cum = above;
                dsel = 8 * lane;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    if (cum + c[e] >= krem) {
                        dsel = 8 * lane + e;
                        break;
                    }
                    cum += c[e];
                }
                knew = krem - cum;
                cgt = cum;  // candidates in digits above the selected one
            }
            const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
            dsel = __shfl_sync(0xffffffffu, dsel, owner);
            krem = __shfl_sync(0xffffffffu, knew, owner);
            gt += __shfl_sync(0xffffffffu, cgt, owner);
            prefix |= (uint64_t)dsel << shift;
            if (shift == 0) break;
            // keep the candidates matching the selected digit (ordered compaction)
            const uint64_t kmask = ~0ull << shift;
            uint32_t nn = 0;
            __syncwarp();
            for (uint32_t j0 = 0; j0 < ncur; j0 += 32) {
                const uint32_t jj = j0 + lane;
                bool keep = false;
                uint32_t j = 0;
                if (jj < ncur) {
                    j = full ? jj : la[jj];
                    const uint64_t k = keys[j] & ~WW_SIGN;
                    keep = k && (k & kmask) == prefix;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (keep) lb[nn + __popc(bal & lt)] = (uint16_t)j;
                nn += __popc(bal);
            }
            __syncwarp();
            uint16_t* t2 = la; la = lb; lb = t2;
            ncur = nn;
            full = false;
        }
        const uint64_t thr = prefix;  // the key of the K-th largest
        // emission in index order: word i of the key bitmap = keys 32 i .. 32 i + 31
        const uint32_t need = g.top_k - gt;
        uint32_t eqseen = 0, pos = 0;
        uint32_t* ob = (uint32_t*)out + wi * g.top_k;
        for (uint32_t i = 0; i < WW_N / 32; ++i) {
            const uint32_t j = 32 * i + lane;
            const uint64_t kw = keys[j], k = kw & ~WW_SIGN;
            const uint32_t beq = __ballot_sync(0xffffffffu, k == thr);
            const bool take = k > thr || (k == thr && eqseen + __popc(beq & lt) < need);
            const uint32_t bt = __ballot_sync(0xffffffffu, take);
            if (take) ob[pos + __popc(bt & lt)] = 2 * j + (uint32_t)(kw >> 63);
            pos += __popc(bt);
            eqseen += __popc(beq);
        }
        la = (uint16_t*)tmp;  // list parity back to the fixed regions
        lb = la + WW_N;
    }
}

// ------------------------------------------- one CTA per window, 32 x 64
// The same arithmetic as k_windows for the BASELINE geometry (32 x 64 images,
// <= 16 band rows) with far fewer instructions and barriers: fixed-tap
// resample weights (zero taps add exact zeros), the 2-D Haar as per-level
// 2 x 2 butterflies (row pass then column pass per block, the reference's
// operation order — thread per block, the low-low value handed to the next
// level; levels 4-6 in one warp by shuffles), coefficients rounded to f32 and
// turned into select keys once (|v'| bits + 1, 0 when ineligible, the sign in
// bit 63), a radix select over the stored keys with shrinking candidate
// lists, and the bits emitted in index order by per-warp ballots.
constexpr int WC_T = 256, WC_W = WC_T / 32;
constexpr uint32_t WC_N = 2048, WC_T64 = 64;
constexpr uint32_t WC_FT = 2, WC_TT = 3, WC_NWID = 3;
constexpr uint64_t WC_SIGN = 1ull << 63;
// shared layout (bytes): keys u64[2048] (band rows alias it before the Haar) |
// tmp f64[16][64] (the select histograms alias it after level 1) | ll1 f64[512] |
// ll2 f64[128] | level-3+ coefficients f32[128] | hist u32[256] | tables
constexpr size_t WC_OFF_TMP = WC_N * 8, WC_OFF_LL1 = WC_OFF_TMP + 64 * 16 * 8;
constexpr size_t WC_OFF_LL2 = WC_OFF_LL1 + 512 * 8, WC_OFF_LL3 = WC_OFF_LL2 + 128 * 8;
constexpr size_t WC_OFF_TAB = WC_OFF_LL3 + 64 * 8;
constexpr size_t WC_SMEM = WC_OFF_TAB + (32 * WC_FT + WC_NWID * 64 * WC_TT) * 12 + 64;

#ifndef WC_MINB
#define WC_MINB 4  // resident CTAs per SM asked of ptxas (A/B builds: make EXTRA=-DWC_MINB=5)
#endif
template <int MODE>
__global__ void __launch_bounds__(WC_T, WC_MINB) k_win_cta(
    const float* __restrict__ band, WinGeom g, const int64_t* __restrict__ widx,
    const int32_t* __restrict__ wf_off, const int32_t* __restrict__ wf_idx,
    const double* __restrict__ wf_val, const int32_t* __restrict__ wt_off,
    const int32_t* __restrict__ wt_idx, const double* __restrict__ wt_val,
    const double* __restrict__ med, const double* __restrict__ mad, void* __restrict__ out,
    uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) unsigned char csm[];
    uint64_t* keys = (uint64_t*)csm;
    float* gs = (float*)csm;
    double* tmp = (double*)(csm + WC_OFF_TMP);
    double* ll1 = (double*)(csm + WC_OFF_LL1);
    double* ll2 = (double*)(csm + WC_OFF_LL2);
    double* ll3 = (double*)(csm + WC_OFF_LL3);
    double* fv = (double*)(csm + WC_OFF_TAB);
    double* tv = fv + 32 * WC_FT;
    int32_t* fi = (int32_t*)(tv + WC_NWID * 64 * WC_TT);
    int32_t* ti = fi + 32 * WC_FT;
    __shared__ uint32_t s_nf, s_wcnt[WC_W], s_wcnt2[WC_W], s_ncur;
    __shared__ uint32_t s_dsel, s_ninel;
    __shared__ uint64_t s_kmax, s_kmin;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    const uint32_t nwid = g.wmax - g.wmin + 1, nb = g.nb;
    constexpr uint32_t mode = MODE;
    // ineligible coefficients (MAD == 0) have select key 0; the histogram
    // passes count them into digit 0 whenever the decided prefix is 0 and the
    // scan takes them back out (no per-key eligibility test)
    if (MODE == 3) {
        if (threadIdx.x == 0) s_ninel = 0;
        __syncthreads();
        uint32_t ni = 0;
        for (uint32_t j = threadIdx.x; j < WC_N; j += WC_T) ni += !(__ldg(mad + j) > 0.0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ni += __shfl_xor_sync(0xffffffffu, ni, o);
        if (lane == 0 && ni) atomicAdd(&s_ninel, ni);
    }
    for (uint32_t q = threadIdx.x; q < 32 * WC_FT; q += WC_T) {
        const uint32_t r = q / WC_FT, t = q - r * WC_FT;
        const int32_t e = wf_off[r] + (int32_t)t;
        const bool ok = e < wf_off[r + 1];
        fv[q] = ok ? wf_val[e] : 0.0;
        fi[q] = ok ? wf_idx[e] : 0;
    }
    for (uint32_t q = threadIdx.x; q < nwid * 64 * WC_TT; q += WC_T) {
        const uint32_t row = q / WC_TT, t = q - row * WC_TT;
        const uint32_t wd = row / 64, Ti = row - wd * 64;
        const int32_t* to = wt_off + (uint64_t)wd * 65;
        const int32_t e = to[Ti] + (int32_t)t;
        const bool ok = e < to[Ti + 1];
        tv[q] = ok ? wt_val[e] : 0.0;
        ti[q] = ok ? wt_idx[e] : 0;
    }
    const double s2 = 0.7071067811865475;  // 1.0 / math.sqrt(2.0), as the reference
    // window columns: c0 = ceil(idx * lag / hop), c1 = (idx * lag + win - frame) / hop + 1;
    // when hop divides lag (the BASELINE geometry) both are idx * (lag / hop) + constants
    const uint64_t lh = g.lag / g.hop;
    const bool lag_exact = lh * g.hop == g.lag;
    const uint64_t wfix = (g.win - g.frame) / g.hop + 1;
    for (uint64_t wi = blockIdx.x; wi < g.n_win; wi += gridDim.x) {
        const uint64_t idx = widx ? (uint64_t)widx[wi] : g.win0 + wi;
        uint64_t c0, c1;
        if (lag_exact) {
            c0 = idx * lh;
            c1 = c0 + wfix;
        } else {
            const uint64_t off = idx * g.lag;
            c0 = (off + g.hop - 1) / g.hop;
            c1 = (off + g.win - g.frame) / g.hop + 1;
        }
        const uint32_t width = (uint32_t)(c1 - c0);
        __syncthreads();
        if (threadIdx.x == 0) {
            s_nf = 0;
            s_kmax = 0;
            s_kmin = ~0ull;
        }
        for (uint32_t i = threadIdx.x; i < width * nb; i += WC_T) gs[i] = __ldg(band + c0 * nb + i);
        __syncthreads();
        // time resample (f64, CSR order; padded taps add exact zeros)
        const double* tvw = tv + (uint64_t)(width - g.wmin) * 64 * WC_TT;
        const int32_t* tiw = ti + (uint64_t)(width - g.wmin) * 64 * WC_TT;
        for (uint32_t i = threadIdx.x; i < 64 * nb; i += WC_T) {  // tmp[f][Ti], f-major
            const uint32_t Ti = i & 63, f = i >> 6;
            double acc = 0.0;
#pragma unroll
            for (uint32_t t = 0; t < WC_TT; ++t)
                acc = fma(tvw[Ti * WC_TT + t], (double)gs[tiw[Ti * WC_TT + t] * nb + f], acc);
            tmp[i] = acc;
        }
        __syncthreads();
        bool nonfinite = false;
        uint64_t kmax = 0, kmin = ~0ull;
        // md / me: the column's MAD and median (mode 3), loaded ahead by the caller
        auto emit_p = [&](uint32_t j, double v, double md, double me) {
            const float c = (float)v;  // coefficients are stored float32 (fingerprint.py:334)
            if (mode == 1) {
                ((float*)out)[wi * WC_N + j] = c;
            } else if (mode == 2) {
                ((float*)out)[(uint64_t)j * g.n_win + wi] = c;
            } else {
                const double cd = (double)c;
                if (!isfinite(cd)) nonfinite = true;
                uint64_t k = 0;
                if (md > 0.0) {
                    const double sc = __ddiv_rn(__dsub_rn(cd, me), md);
                    const uint64_t m = mag_key(sc) + 1;
                    kmax = m > kmax ? m : kmax;
                    kmin = m < kmin ? m : kmin;
                    k = m | (sc < 0.0 ? WC_SIGN : 0ull);
                }
                keys[j] = k;
            }
        };
        auto emit = [&](uint32_t j, double v) {
            if (mode == 3) emit_p(j, v, __ldg(mad + j), __ldg(med + j));
            else emit_p(j, v, 0.0, 0.0);
        };
        auto bfly = [&](double x00, double x01, double x10, double x11, uint32_t bi, uint32_t bj,
                        uint32_t h, uint32_t w) -> double {
            const double lo0 = __dmul_rn(__dadd_rn(x00, x01), s2), hi0 = __dmul_rn(__dsub_rn(x00, x01), s2);
            const double lo1 = __dmul_rn(__dadd_rn(x10, x11), s2), hi1 = __dmul_rn(__dsub_rn(x10, x11), s2);
            emit(bi * 64 + w / 2 + bj, __dmul_rn(__dadd_rn(hi0, hi1), s2));
            emit((h / 2 + bi) * 64 + bj, __dmul_rn(__dsub_rn(lo0, lo1), s2));
            emit((h / 2 + bi) * 64 + w / 2 + bj, __dmul_rn(__dsub_rn(hi0, hi1), s2));
            return __dmul_rn(__dadd_rn(lo0, lo1), s2);
        };
        // level 1 (32 x 64): block (bi, bj) = pixels rows 2bi, 2bi+1, cols 2bj, 2bj+1
        for (uint32_t bk = threadIdx.x; bk < 512; bk += WC_T) {
            const uint32_t bi = bk >> 5, bj = bk & 31;
            // the block's three detail coefficients: statistics loaded ahead
            const uint32_t j0 = bi * 64 + 32 + bj, j1 = (16 + bi) * 64 + bj, j2 = j1 + 32;
            double pmd[3] = {0.0, 0.0, 0.0}, pme[3] = {0.0, 0.0, 0.0};
            if (mode == 3) {
                pmd[0] = __ldg(mad + j0); pmd[1] = __ldg(mad + j1); pmd[2] = __ldg(mad + j2);
                pme[0] = __ldg(med + j0); pme[1] = __ldg(med + j1); pme[2] = __ldg(med + j2);
            }
            double x[2][2];
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const uint32_t r = 2 * bi + a;
                const double w0 = fv[r * WC_FT], w1 = fv[r * WC_FT + 1];
                const uint32_t i0 = fi[r * WC_FT], i1 = fi[r * WC_FT + 1];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t c = 2 * bj + b;
                    const double acc = fma(w1, tmp[i1 * 64 + c], fma(w0, tmp[i0 * 64 + c], 0.0));
                    x[a][b] = (double)(float)acc;  // images are float32 (fingerprint.py:239-241)
                }
            }
            const double lo0 = __dmul_rn(__dadd_rn(x[0][0], x[0][1]), s2);
            const double hi0 = __dmul_rn(__dsub_rn(x[0][0], x[0][1]), s2);
            const double lo1 = __dmul_rn(__dadd_rn(x[1][0], x[1][1]), s2);
            const double hi1 = __dmul_rn(__dsub_rn(x[1][0], x[1][1]), s2);
            emit_p(j0, __dmul_rn(__dadd_rn(hi0, hi1), s2), pmd[0], pme[0]);
            emit_p(j1, __dmul_rn(__dsub_rn(lo0, lo1), s2), pmd[1], pme[1]);
            emit_p(j2, __dmul_rn(__dsub_rn(hi0, hi1), s2), pmd[2], pme[2]);
            ll1[bk] = __dmul_rn(__dadd_rn(lo0, lo1), s2);
        }
        __syncthreads();
        if (threadIdx.x < 128) {  // level 2 (16 x 32)
            const uint32_t bi = threadIdx.x >> 4, bj = threadIdx.x & 15;
            ll2[threadIdx.x] = bfly(ll1[(2 * bi) * 32 + 2 * bj], ll1[(2 * bi) * 32 + 2 * bj + 1],
                                    ll1[(2 * bi + 1) * 32 + 2 * bj], ll1[(2 * bi + 1) * 32 + 2 * bj + 1],
                                    bi, bj, 16, 32);
        }
        __syncthreads();
        // levels 3-6 in one warp; their 128 coefficients (rows < 8, cols < 16)
        // go to a small f32 array (ll3 region) and are scored by 128 threads
        // after the barrier (the divisions stay off warp 0's critical path)
        float* c3 = (float*)ll3;  // [8][16]
        if (warp == 0) {
            auto emit3 = [&](uint32_t j, double v) {
                const float c = (float)v;
                if (mode == 1) ((float*)out)[wi * WC_N + j] = c;
                else if (mode == 2) ((float*)out)[(uint64_t)j * g.n_win + wi] = c;
                else c3[(j >> 6) * 16 + (j & 63)] = c;
            };
            auto bfly3 = [&](double x00, double x01, double x10, double x11, uint32_t bi, uint32_t bj,
                             uint32_t h, uint32_t w) -> double {
                const double lo0 = __dmul_rn(__dadd_rn(x00, x01), s2), hi0 = __dmul_rn(__dsub_rn(x00, x01), s2);
                const double lo1 = __dmul_rn(__dadd_rn(x10, x11), s2), hi1 = __dmul_rn(__dsub_rn(x10, x11), s2);
                emit3(bi * 64 + w / 2 + bj, __dmul_rn(__dadd_rn(hi0, hi1), s2));
                emit3((h / 2 + bi) * 64 + bj, __dmul_rn(__dsub_rn(lo0, lo1), s2));
                emit3((h / 2 + bi) * 64 + w / 2 + bj, __dmul_rn(__dsub_rn(hi0, hi1), s2));
                return __dmul_rn(__dadd_rn(lo0, lo1), s2);
            };
            const uint32_t tr = lane >> 3, tc = lane & 7;  // level-3 block (tr, tc) of 4 x 8
            const double l3 = bfly3(ll2[(2 * tr) * 16 + 2 * tc], ll2[(2 * tr) * 16 + 2 * tc + 1],
                                    ll2[(2 * tr + 1) * 16 + 2 * tc], ll2[(2 * tr + 1) * 16 + 2 * tc + 1],
                                    tr, tc, 8, 16);
            const double n01 = __shfl_down_sync(0xffffffffu, l3, 1);
            const double n10 = __shfl_down_sync(0xffffffffu, l3, 8);
            const double n11 = __shfl_down_sync(0xffffffffu, l3, 9);
            double l4 = 0.0;
            if (!(tr & 1) && !(tc & 1)) l4 = bfly3(l3, n01, n10, n11, tr / 2, tc / 2, 4, 8);
            const double m01 = __shfl_down_sync(0xffffffffu, l4, 2);
            const double m10 = __shfl_down_sync(0xffffffffu, l4, 16);
            const double m11 = __shfl_down_sync(0xffffffffu, l4, 18);
            double l5 = 0.0;
            if (lane == 0 || lane == 4) l5 = bfly3(l4, m01, m10, m11, 0, lane / 4, 2, 4);
            const double x1 = __shfl_down_sync(0xffffffffu, l5, 4);
            if (lane == 0) {
                emit3(0, __dmul_rn(__dadd_rn(l5, x1), s2));
                emit3(1, __dmul_rn(__dsub_rn(l5, x1), s2));
            }
        }
        if (mode != 3) continue;
        __syncthreads();
        if (threadIdx.x < 128) {
            const uint32_t j = (threadIdx.x >> 4) * 64 + (threadIdx.x & 15);
            emit(j, (double)c3[threadIdx.x]);
        }
        // select histograms (3 x (256 + a trash bin for keys off the decided
        // prefix), triple-buffered) and the <= 32-candidate list live in the
        // time-resample scratch, free after level 1
        constexpr uint32_t HS = 272;
        uint32_t* H = (uint32_t*)tmp;
        uint64_t* clist = (uint64_t*)(H + 3 * HS);
        const uint32_t n_inel = s_ninel;
        H[threadIdx.x] = 0;
        // CTA-wide non-finite flag, key range
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t a2 = __shfl_xor_sync(0xffffffffu, kmax, o);
            const uint64_t b2 = __shfl_xor_sync(0xffffffffu, kmin, o);
            kmax = a2 > kmax ? a2 : kmax;
            kmin = b2 < kmin ? b2 : kmin;
        }
        if (__any_sync(0xffffffffu, nonfinite) && lane == 0) s_nf = 1;
        if (lane == 0) {
            atomicMax((unsigned long long*)&s_kmax, (unsigned long long)kmax);
            atomicMin((unsigned long long*)&s_kmin, (unsigned long long)kmin);
        }
        __syncthreads();
        if (s_nf) {
            if (threadIdx.x == 0) atomicOr(flags, 1u);
            continue;
        }
        kmax = s_kmax;
        kmin = s_kmin;
        // each thread's 8 keys (j = 256 w + 32 q + lane) stay in registers for
        // the select passes and the emission
        uint64_t kr[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) kr[q] = keys[256 * warp + 32 * q + lane];
        // 8-bit digits starting at the highest bit where the eligible keys
        // differ (bits above it are common to all of them); the last digit may
        // overlap decided bits (constant over the candidates).  Pass p counts
        // into histogram p % 3 and clears histogram (p + 1) % 3, last read by
        // pass p - 2: one barrier per pass.  Once <= 32 candidates share the
        // decided prefix, one warp ranks them.
        const uint64_t dk = kmax ^ kmin;
        int shift = dk ? max(0, 63 - __clzll((long long)dk) - 7) : 0;
        uint64_t decided = shift + 8 < 64 ? ~0ull << (shift + 8) : 0ull;
        uint64_t prefix = kmax & decided;
        uint32_t krem = g.top_k, gt = 0;
        uint64_t thr = 0;
        for (uint32_t pass = 0;; ++pass) {
            uint32_t* hc = H + (pass % 3) * HS;
            uint32_t* hn = H + ((pass + 1) % 3) * HS;
            if (shift >= 32) {  // digit and decided bits in the high words
                // the sign (bit 31 of the high word) is masked out of dh; digits
                // stay below it (shift <= 55)
                const uint32_t dh = (uint32_t)(decided >> 32) & 0x7FFFFFFFu;
                const uint32_t ph = (uint32_t)(prefix >> 32);
                const uint32_t sh = (uint32_t)shift - 32;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t h = (uint32_t)(kr[q] >> 32);
                    atomicAdd(&hc[(h & dh) == ph ? (h >> sh) & 0xFFu : 256u], 1u);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint64_t k = kr[q] & ~WC_SIGN;
                    atomicAdd(&hc[(k & decided) == prefix ? (uint32_t)(k >> shift) & 0xFFu : 256u], 1u);
                }
            }
            hn[threadIdx.x] = 0;
            if (threadIdx.x == 0) s_ncur = 0;
            __syncthreads();
            // every warp finds the digit holding the krem-th largest
            uint32_t csel;
            {
                uint32_t c[8], sum = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e) c[e] = hc[8 * lane + e];
                if (lane == 0 && prefix == 0) c[0] -= n_inel;
#pragma unroll
                for (int e = 0; e < 8; ++e) sum += c[e];
                uint32_t x = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, x, o);
                    if (lane + o < 32) x += y;
                }
                const uint32_t above = x - sum;
                const bool mine = above < krem && krem <= x;
                uint32_t cum = above, dsel = 8 * lane, cs = 0;
                if (mine) {
#pragma unroll
                    for (int e = 7; e >= 0; --e) {
                        if (cum + c[e] >= krem) {
                            dsel = 8 * lane + e;
                            cs = c[e];
                            break;
                        }
                        cum += c[e];
                    }
                }
                const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
                dsel = __shfl_sync(0xffffffffu, dsel, owner);
                cum = __shfl_sync(0xffffffffu, cum, owner);
                csel = __shfl_sync(0xffffffffu, cs, owner);
                krem -= cum;
                gt += cum;
                prefix = (prefix & ~(0xFFull << shift)) | ((uint64_t)dsel << shift);
                decided |= 0xFFull << shift;
            }
            if (shift == 0) {
                thr = prefix;
                break;
            }
            shift = shift >= 8 ? shift - 8 : 0;
            if (csel <= 32) {  // the rest by ranks inside one warp
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint64_t k = kr[q] & ~WC_SIGN;
                    if (k && (k & decided) == prefix) clist[atomicAdd(&s_ncur, 1u)] = k;
                }
                __syncthreads();
                if (warp == 0) {
                    const uint32_t ncur = s_ncur;
                    const uint64_t k = lane < ncur ? clist[lane] : 0ull;
                    uint32_t greater = 0, geq = 0;
                    for (uint32_t mm = 0; mm < ncur; ++mm) {
                        const uint64_t km = __shfl_sync(0xffffffffu, k, mm);
                        greater += km > k;
                        geq += km >= k;
                    }
                    const bool hit = lane < ncur && greater < krem && krem <= geq;
                    const uint32_t own = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
                    if (lane == own) {
                        s_kmax = k;        // the threshold key
                        s_dsel = greater;  // candidates above it
                    }
                }
                __syncthreads();
                thr = s_kmax;
                gt += s_dsel;
                break;
            }
        }
        const uint32_t need = g.top_k - gt;
        // emission in index order: warp w owns key words 8w .. 8w + 7 (keys
        // 256 w .. 256 w + 255); per-warp counts of ties and takes, then prefixes
        uint32_t beqs[8], ntie = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint64_t k = kr[q] & ~WC_SIGN;
            beqs[q] = __ballot_sync(0xffffffffu, k == thr);
            ntie += __popc(beqs[q]);
        }
        if (lane == 0) s_wcnt[warp] = ntie;
        __syncthreads();
        uint32_t eqseen = 0;
        for (uint32_t w = 0; w < warp; ++w) eqseen += s_wcnt[w];
        uint32_t takes[8], ntake = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint64_t k = kr[q] & ~WC_SIGN;
            const bool take = k > thr || (k == thr && eqseen + __popc(beqs[q] & lt) < need);
            takes[q] = __ballot_sync(0xffffffffu, take);
            ntake += __popc(takes[q]);
            eqseen += __popc(beqs[q]);
        }
        if (lane == 0) s_wcnt2[warp] = ntake;
        __syncthreads();
        uint32_t pos = 0;
        for (uint32_t w = 0; w < warp; ++w) pos += s_wcnt2[w];
        // staged in the key array (the keys are in registers), then one
        // coalesced row store; the next window's band rows overwrite it only
        // after the loop-top barrier
        uint32_t* sb = (uint32_t*)keys;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t j = 256 * warp + 32 * q + lane;
            if ((takes[q] >> lane) & 1u)
                sb[pos + __popc(takes[q] & lt)] = 2 * j + (uint32_t)(kr[q] >> 63);
            pos += __popc(takes[q]);
        }
        __syncthreads();
        uint32_t* ob = (uint32_t*)out + wi * g.top_k;
        for (uint32_t i = threadIdx.x; i < g.top_k; i += WC_T) ob[i] = sb[i];
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

// Median / MAD of one column per CTA in few passes over the column: the
// order statistic k by 12-bit digits over the order-preserving 64-bit keys
// of the f64 values, starting at the highest bit where the column's min and
// max keys differ; once the bin holding rank k has <= MS_CAP members they
// are compacted into shared memory and ranked there (bitonic sort), so a
// column is read ~3 times instead of 8 per order statistic.  For an even
// count the upper middle value comes from one more pass (count <= v, min
// above v), then (a + b) / 2 in f64 as np.median.  mode 1: |x - center|.
constexpr int MS_T = 512;
constexpr uint32_t MS_CAP = 1024, MS_BINS = 4096;

__device__ __forceinline__ double ms_val(const float* c, uint64_t i, int mode, double ctr) {
    return mode ? fabs((double)c[i] - ctr) : (double)c[i];
}

__device__ uint64_t ms_reduce_u64(uint64_t v, bool is_max, uint64_t* red) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? (w > v ? w : v) : (w < v ? w : v);
    }
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = red[0];
    for (int w = 1; w < MS_T / 32; ++w) v = is_max ? (red[w] > v ? red[w] : v) : (red[w] < v ? red[w] : v);
    return v;
}

__global__ void __launch_bounds__(MS_T) k_col_median(const float* __restrict__ cols, uint64_t S,
                                                     int mode, const double* __restrict__ center,
                                                     double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char msm[];
    uint32_t* hist = (uint32_t*)msm;                               // [MS_BINS]
    uint64_t* lst = (uint64_t*)(msm + MS_BINS * 4);                 // [MS_CAP]
    __shared__ uint64_t red[MS_T / 32];
    __shared__ uint32_t s_cnt, s_bin, s_below;
    const uint32_t col = blockIdx.x;
    const float* c = cols + (uint64_t)col * S;
    const double ctr = mode ? center[col] : 0.0;
    uint64_t kmin = ~0ull, kmax = 0;
    for (uint64_t i = threadIdx.x; i < S; i += MS_T) {
        const uint64_t k = ord_key(ms_val(c, i, mode, ctr));
        kmin = k < kmin ? k : kmin;
        kmax = k > kmax ? k : kmax;
    }
    kmin = ms_reduce_u64(kmin, false, red);
    kmax = ms_reduce_u64(kmax, true, red);
    uint64_t rank = (S - 1) / 2;  // lower middle (the middle for odd S)
    const uint64_t dk = kmin ^ kmax;
    int shift = dk ? max(0, 63 - __clzll((long long)dk) - 11) : 0;
    uint64_t decided = shift + 12 < 64 ? ~0ull << (shift + 12) : 0ull;
    uint64_t prefix = kmin & decided;
    uint64_t v1key = 0;
    while (true) {
        for (uint32_t b = threadIdx.x; b < MS_BINS; b += MS_T) hist[b] = 0;
        __syncthreads();
        for (uint64_t i = threadIdx.x; i < S; i += MS_T) {
            const uint64_t k = ord_key(ms_val(c, i, mode, ctr));
            if ((k & decided) == prefix) atomicAdd(&hist[(k >> shift) & 0xFFF], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // the bin holding `rank` (ascending)
            uint64_t cum = 0;
            uint32_t b = 0;
            for (; b < MS_BINS; ++b) {
                if (cum + hist[b] > rank) break;
                cum += hist[b];
            }
            s_bin = b;
            s_below = (uint32_t)cum;
            s_cnt = hist[b];
        }
        __syncthreads();
        const uint32_t bin = s_bin, cnt = s_cnt;
        rank -= s_below;
        prefix = (prefix & ~(0xFFFull << shift)) | ((uint64_t)bin << shift);
        decided |= 0xFFFull << shift;
        if (cnt <= MS_CAP || shift == 0) {
            if (cnt > MS_CAP) {  // every remaining bit decided: the key itself
                v1key = prefix;
                break;
            }
            // compact the bin into shared memory and rank it there
            if (threadIdx.x == 0) s_cnt = 0;
            __syncthreads();
            for (uint64_t i = threadIdx.x; i < S; i += MS_T) {
                const uint64_t k = ord_key(ms_val(c, i, mode, ctr));
                if ((k & decided) == prefix) lst[atomicAdd(&s_cnt, 1u)] = k;
            }
            __syncthreads();
            const uint32_t L = s_cnt;
            uint32_t P = 1;
            while (P < L) P <<= 1;
            for (uint32_t i = L + threadIdx.x; i < P; i += MS_T) lst[i] = ~0ull;
            __syncthreads();
            for (uint32_t kk = 2; kk <= P; kk <<= 1)
                for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
                    for (uint32_t i = threadIdx.x; i < P; i += MS_T) {
                        const uint32_t l = i ^ j;
                        if (l > i) {
                            const uint64_t a = lst[i], b2 = lst[l];
                            const bool up = (i & kk) == 0;
                            if ((a > b2) == up) {
                                lst[i] = b2;
                                lst[l] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            v1key = lst[rank];
            break;
        }
        shift = shift >= 12 ? shift - 12 : 0;
    }
    double v = key_val(v1key);
    if (!(S & 1)) {
        // upper middle: v again when it repeats past the lower rank, else the
        // smallest value above it
        const uint64_t lower = (S - 1) / 2;
        uint64_t le = 0, above = ~0ull;
        for (uint64_t i = threadIdx.x; i < S; i += MS_T) {
            const uint64_t k = ord_key(ms_val(c, i, mode, ctr));
            le += k <= v1key;
            if (k > v1key && k < above) above = k;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) le += __shfl_xor_sync(0xffffffffu, le, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = le;
        __syncthreads();
        uint64_t tle = 0;
        for (int w = 0; w < MS_T / 32; ++w) tle += red[w];
        above = ms_reduce_u64(above, false, red);
        const double v2 = tle > lower + 1 ? v : key_val(above);
        v = (v + v2) / 2.0;  // np.median of an even count
    }
    if (threadIdx.x == 0) out[col] = v;
}

// (rows, cols) -> (cols, rows) through 32 x 33 shared-memory tiles; grid.x over
// row tiles (up to 2^31), grid.y over column tiles
__global__ void __launch_bounds__(256) k_transpose_f32(const float* __restrict__ src, uint64_t rows,
                                                       uint32_t cols, float* __restrict__ dst) {
    __shared__ float tile[32][33];
    const uint64_t r0 = (uint64_t)blockIdx.x * 32;
    const uint32_t c0 = blockIdx.y * 32;
    const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (uint32_t k = 0; k < 32; k += 8) {
        const uint64_t r = r0 + ty + k;
        if (r < rows && c0 + tx < cols) tile[ty + k][tx] = src[r * cols + c0 + tx];
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < 32; k += 8) {
        const uint32_t c = c0 + ty + k;
        if (c < cols && r0 + tx < rows) dst[(uint64_t)c * rows + r0 + tx] = tile[tx][ty + k];
    }
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
    // tensor-core path (default): bins in chunks of 16 (4 n-tiles), twiddles
    // for the whole frame + one slab of samples in shared memory
    static const char* sk = getenv("QS_STFT_KERNEL");
    const bool fma_path = sk && sk[0] == 'f';
    const uint32_t ksteps = (frame + 3) / 4;
    const size_t mma_smem = (size_t)ksteps * 4 * 32 * 8 + ((size_t)(SM_COLS - 1) * hop + ksteps * 4) * 8;
    if (!fma_path && mma_smem <= 200 * 1024) {
        const uint64_t slabs = (n_cols + SM_COLS - 1) / SM_COLS;
        const unsigned mgrid = (unsigned)(slabs < 148 * 2 * 8 ? slabs : 148 * 2 * 8);
        for (uint32_t b0 = 0; b0 < nb; b0 += 16) {
            const uint32_t nbc = min(16u, nb - b0);
            if (x_is_f32) {
                QS_CUDA(cudaFuncSetAttribute(k_band_stft_mma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mma_smem), "attr");
                k_band_stft_mma<float><<<mgrid, SM_WARPS * 32, mma_smem, st>>>(
                    (const float*)x_dev, n_samples, frame, hop, n_cols, nbc, tw_dev, out_dev, b0, nb);
            } else {
                QS_CUDA(cudaFuncSetAttribute(k_band_stft_mma<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mma_smem), "attr");
                k_band_stft_mma<double><<<mgrid, SM_WARPS * 32, mma_smem, st>>>(
                    (const double*)x_dev, n_samples, frame, hop, n_cols, nbc, tw_dev, out_dev, b0, nb);
            }
            QS_CHECK_LAUNCH("k_band_stft_mma");
        }
        return QS_OK;
    }
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

static int num_sms_fp() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
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
    WinGeom g{n_cols, lag, win, win0, n_win, frame, hop, nb, F, T, wmin, wmax, n_levels, top_k,
              (uint32_t)mode};
    // the BASELINE geometry (32 x 64 images, <= 16 band rows): one warp per window
    // kernel choice for the BASELINE geometry: QS_WIN_KERNEL = cta32 (default),
    // warp, generic (k_windows) — A/B measurements
    static const char* wk = getenv("QS_WIN_KERNEL");
    static const int kind = !wk ? 0 : (wk[0] == 'w' ? 1 : (wk[0] == 'g' ? 2 : 0));
    const bool cta_only = kind != 1;
    // padded resize tables: <= WW_FT taps per w_f row (nb <= 16 upsampled to 32
    // rows), <= WW_TT per w_t row (width <= 128 resampled to 64), <= WW_NWID widths
    const bool tabs_fit = nb <= 16 && wmax <= 128 && wmax - wmin + 1 <= WW_NWID;
    if (!cta_only && mode >= 1 && F == 32 && T == WW_T && nb <= WW_NBMAX && n_levels == 6 &&
        tabs_fit && (size_t)wmax * nb * 4 <= WW_N * 8) {
        const size_t wsmem = WW_TAB_BYTES + WW_WARP_BYTES * WW_WARPS;
        QS_CUDA(cudaFuncSetAttribute(k_win_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)wsmem), "attr");
        const uint64_t want = (n_win + WW_WARPS - 1) / WW_WARPS;
        const unsigned grid = (unsigned)(want < (uint64_t)num_sms_fp() ? want : (uint64_t)num_sms_fp());
        k_win_warp<<<grid, WW_WARPS * 32, wsmem, (cudaStream_t)stream>>>(
            band_dev, g, widx_dev, wf_off, wf_idx, wf_val, wt_off, wt_idx, wt_val, med_dev, mad_dev,
            out_dev, flags_dev);
        QS_CHECK_LAUNCH("k_win_warp");
        return QS_OK;
    }
    if (kind == 0 && mode >= 1 && F == 32 && T == WC_T64 && nb <= 16 && n_levels == 6 && wmax <= 128 &&
        wmax - wmin + 1 <= WC_NWID && (size_t)wmax * nb * 4 <= WC_N * 8) {
        auto kern = mode == 3 ? k_win_cta<3> : (mode == 2 ? k_win_cta<2> : k_win_cta<1>);
        QS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)WC_SMEM), "attr");
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WC_T, WC_SMEM);
        const uint64_t cap = (uint64_t)num_sms_fp() * (per_sm < 1 ? 1 : per_sm) * 4;
        const unsigned grid = (unsigned)(n_win < cap ? n_win : cap);
        kern<<<grid, WC_T, WC_SMEM, (cudaStream_t)stream>>>(
            band_dev, g, widx_dev, wf_off, wf_idx, wf_val, wt_off, wt_idx, wt_val, med_dev, mad_dev,
            out_dev, flags_dev);
        QS_CHECK_LAUNCH("k_win_cta");
        return QS_OK;
    }
    const size_t smem = win_smem(F, T, wmax, nb).bytes;
    QS_ARG(smem <= 200 * 1024, "spectral image too large for the window kernel");
    QS_CUDA(cudaFuncSetAttribute(k_windows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
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
    // QS_MAD_SELECT=radix: the round-1 8-pass radix select per order statistic
    static const bool radix = getenv("QS_MAD_SELECT") && getenv("QS_MAD_SELECT")[0] == 'r';
    if (!radix) {
        const size_t sm = (size_t)MS_BINS * 4 + (size_t)MS_CAP * 8;
        QS_CUDA(cudaFuncSetAttribute(k_col_median, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                "attr");
        k_col_median<<<n_coeffs, MS_T, sm, st>>>(cols_dev, S, 0, nullptr, med_dev);
        k_col_median<<<n_coeffs, MS_T, sm, st>>>(cols_dev, S, 1, med_dev, mad_dev);
        QS_CHECK_LAUNCH("qs_fp_mad");
        return QS_OK;
    }
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

int qs_fp_transpose_f32(const float* src_dev, uint64_t rows, uint32_t cols, float* dst_dev,
                        void* stream) {
    if (rows == 0 || cols == 0) return QS_OK;
    QS_ARG(src_dev && dst_dev && src_dev != dst_dev, "transpose needs two distinct buffers");
    QS_ARG(cols <= 65535u * 32u, "too many columns");
    const dim3 grid((unsigned)((rows + 31) / 32), (cols + 31) / 32);
    k_transpose_f32<<<grid, 256, 0, (cudaStream_t)stream>>>(src_dev, rows, cols, dst_dev);
    QS_CHECK_LAUNCH("k_transpose_f32");
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
