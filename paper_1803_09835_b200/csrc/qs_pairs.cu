// Candidate-pair enumeration with exact collision counting (sm_100a).
//
// Replaces the reference's per-query gather + (q << 32 | c) key materialisation
// + sort + run-length count (lsh_search.py:175-219) and the >= m threshold
// (:261, :281).  Work unit: a 32-member chunk of one bucket; lane i holds
// member a_i's bit-sliced tag planes in registers, the bucket's members are
// staged 32 at a time in shared memory (cp.async, double buffered: the next
// batch streams in while the current one is compared) and every lane compares
// its row with each staged row (broadcast shared-memory reads + LOP3).
//
// Exactness: each unordered pair is handled only in the bucket of its FIRST
// colliding table.  Tag-plane masks over-approximate the set of colliding
// tables (tags: false positives only), so every table a decision depends on
// is confirmed on the 64-bit keys (rkeys, row-major).  Confirmations are rare
// and divergent, so candidates are queued per warp in shared memory and
// drained 32 at a time with one candidate per lane (convergent, 32 independent
// key loads in flight).
//
// Modes (warp-uniform, compile time):
//   FULL      distinct-pair count + emission of sim >= m (no occurrence filter)
//   MATCHED   emission only (occurrence-filter pass 1): screen on 8 planes
//   DISTINCT  distinct-pair count only (pass 2 after the filter)
#include "qs_lsh.cuh"

namespace qs {

constexpr uint32_t GRAB = 8;
constexpr int QCAP = 64;
enum { MODE_FULL = 0, MODE_MATCHED = 1, MODE_DISTINCT = 2 };

template <int W, int MODE>
struct PairCfg {
    static constexpr int NP = MODE == MODE_MATCHED ? 8 : 16;    // planes staged / in registers
    static constexpr int WARPS = MODE == MODE_MATCHED ? 8 : 4;  // warps per CTA
    static constexpr int ROW = W * NP;                          // u32 per staged row
    // per-warp shared memory (u32 units): 2 row buffers + 2 id buffers + queue
    static constexpr int QWORDS = QCAP * (3 + W);
    static constexpr int PER_WARP = 2 * 32 * ROW + 2 * 32 + QWORDS;
};

// AND over np planes of ~(A ^ B) for 32-table word w; R is a staged row with NP planes/word
template <int W, int NP>
__device__ __forceinline__ uint32_t pmask(const uint32_t (&A)[W][NP], const uint32_t* R, int w,
                                          int np) {
    uint32_t x = 0xFFFFFFFFu;
    const uint4* r4 = (const uint4*)(R + w * NP);
#pragma unroll
    for (int q = 0; q < NP / 4; ++q) {
        if (q * 4 >= np) break;
        const uint4 v = r4[q];
        x &= ~(A[w][q * 4 + 0] ^ v.x);
        x &= ~(A[w][q * 4 + 1] ^ v.y);
        x &= ~(A[w][q * 4 + 2] ^ v.z);
        x &= ~(A[w][q * 4 + 3] ^ v.w);
    }
    return x;
}

// number of tables in `cand` (bit i = table wbase + i) whose keys agree;
// with stop_first, returns as soon as one agrees.
__device__ __forceinline__ uint32_t confirm(const uint64_t* __restrict__ rkeys, uint32_t t,
                                            uint32_t a, uint32_t b, uint32_t cand, uint32_t wbase,
                                            bool stop_first) {
    uint32_t hits = 0;
    const uint64_t* ra = rkeys + (uint64_t)a * t + wbase;
    const uint64_t* rb = rkeys + (uint64_t)b * t + wbase;
    while (cand) {
        uint32_t tt[4];
        bool v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = cand != 0;
            tt[k] = v[k] ? (uint32_t)(__ffs(cand) - 1) : 0u;
            cand &= cand - 1;
        }
        uint64_t ka[4], kb[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            ka[k] = v[k] ? __ldg(ra + tt[k]) : 0;
            kb[k] = v[k] ? __ldg(rb + tt[k]) : 1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) hits += (ka[k] == kb[k]);
        if (stop_first && hits) return hits;
    }
    return hits;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Queue entry flags (bits 8.. of qt; bits 0..7 = table & 0xFF, table >> 8 kept in bits 16..)
constexpr uint32_t QF_COUNT = 1u << 8;     // needs the confirmed count (emit if >= m)
constexpr uint32_t QF_DISTINCT = 1u << 9;  // count as a distinct pair when first

struct Queue {
    uint32_t* qa;
    uint32_t* qb;
    uint32_t* qt;
    uint32_t* qm;  // [QCAP][W]
};

// Drain `cnt` (<= 32) queued candidates, one per lane: first-table rule on
// the candidate bits below the table, confirmed count on the bits above.
template <int W>
__device__ __forceinline__ void drain(const Queue& q, uint32_t base, uint32_t cnt, uint32_t lane,
                                      const uint64_t* __restrict__ rkeys, uint32_t t, uint32_t m,
                                      uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim,
                                      uint64_t cap, unsigned long long* __restrict__ counters,
                                      unsigned long long& distinct) {
    if (lane < cnt) {
        const uint32_t e = (base + lane) & (QCAP - 1);
        const uint32_t a = q.qa[e], b = q.qb[e], f = q.qt[e];
        const uint32_t table = (f & 0xFFu) | ((f >> 16) << 8);
        const int wt = (int)(table >> 5);
        const uint32_t bt = table & 31, low = (1u << bt) - 1u;
        bool first = true;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w > wt || !first) break;
            const uint32_t mw = q.qm[e * W + w];
            const uint32_t ebits = (w < wt) ? mw : (mw & low);
            if (ebits && confirm(rkeys, t, a, b, ebits, w * 32, true)) first = false;
        }
        if (first) {
            if (f & QF_DISTINCT) ++distinct;
            if (f & QF_COUNT) {
                uint32_t exact = 1;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    if (w < wt) continue;
                    const uint32_t mw = q.qm[e * W + w];
                    const uint32_t x = (w == wt) ? (mw & ~((low << 1) | 1u)) : mw;
                    if (x) exact += confirm(rkeys, t, a, b, x, w * 32, false);
                }
                if (exact >= m) {
                    const unsigned long long pos = atomicAdd(counters + 1, 1ULL);
                    if (pos < cap) {
                        out_key[pos] = ((uint64_t)(b - a) << 32) | a;
                        out_sim[pos] = exact;
                    }
                }
            }
        }
    }
    __syncwarp();
}

template <int W, int MODE, bool HAS_E>
__global__ void __launch_bounds__(PairCfg<W, MODE>::WARPS * 32) k_pairs(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
    const uint64_t* __restrict__ chunk_off, uint64_t nb, const uint64_t* __restrict__ rkeys,
    const uint32_t* __restrict__ tags, uint32_t t, uint32_t m, uint64_t excl,
    const uint8_t* __restrict__ emask, const uint64_t* __restrict__ edges, uint32_t p,
    uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim, uint64_t cap,
    unsigned long long* __restrict__ counters, unsigned long long* __restrict__ work) {
    using C = PairCfg<W, MODE>;
    constexpr int NP = C::NP;
    extern __shared__ __align__(16) uint32_t psm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* wbase = psm + warp * C::PER_WARP;
    uint32_t* rows0 = wbase;                       // [2][32][ROW]
    uint32_t* rid0 = wbase + 2 * 32 * C::ROW;      // [2][32]
    Queue q;
    q.qa = rid0 + 64;
    q.qb = q.qa + QCAP;
    q.qt = q.qb + QCAP;
    q.qm = q.qt + QCAP;
    uint32_t qhead = 0, qn = 0;  // warp-uniform ring state
    const uint64_t total_chunks = chunk_off[nb];
    const uint32_t last_mask = (t & 31) ? ((1u << (t & 31)) - 1u) : 0xFFFFFFFFu;
    const uint32_t lt_mask = (1u << lane) - 1u;
    unsigned long long distinct = 0;

    while (true) {
        unsigned long long g0 = 0;
        if (lane == 0) g0 = atomicAdd(work, (unsigned long long)GRAB);
        g0 = __shfl_sync(0xffffffffu, g0, 0);
        if (g0 >= total_chunks) break;
        const uint64_t g1 = min((uint64_t)g0 + GRAB, total_chunks);
        uint64_t lo = 0, hi = nb;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (chunk_off[mid] <= g0) lo = mid;
            else hi = mid;
        }
        uint64_t b = lo;
        for (uint64_t g = g0; g < g1; ++g) {
            while (chunk_off[b + 1] <= g) ++b;
            const uint32_t c = (uint32_t)(g - chunk_off[b]);
            const uint64_t st = bstart[b];
            const uint32_t s = bsize[b];
            const uint32_t table = btab[b];
            const int wt = (int)(table >> 5);
            const uint32_t bt = table & 31, low = (1u << bt) - 1u;
            const uint32_t tflag = (table & 0xFFu) | ((table >> 8) << 16);
            const uint32_t i = c * 32 + lane;
            const bool active = i < s;
            const uint32_t a = active ? sids[st + i] : 0;
            // first staged batch (cp.async) overlaps the register loads of row a
            uint32_t jb = c * 32;
            int buf = 0;
            {
                const uint32_t jj = jb + lane;
                const uint32_t bid = jj < s ? sids[st + jj] : 0;
                rid0[lane] = bid;
                if (jj < s) {
                    uint32_t* dst = rows0 + lane * C::ROW;
#pragma unroll
                    for (int w = 0; w < W; ++w)
#pragma unroll
                        for (int qq = 0; qq < NP / 4; ++qq)
                            cp_async16(dst + w * NP + qq * 4, tags + ((uint64_t)bid * W + w) * 16 + qq * 4);
                }
                cp_async_commit();
            }
            uint32_t nxt = (jb + 32 + lane < s) ? sids[st + jb + 32 + lane] : 0;
            uint32_t A[W][NP];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint4* src = (const uint4*)(tags + ((uint64_t)a * W + w) * 16);
#pragma unroll
                for (int qq = 0; qq < NP / 4; ++qq) {
                    const uint4 v = active ? __ldg(src + qq) : make_uint4(0, 0, 0, 0);
                    A[w][qq * 4 + 0] = v.x; A[w][qq * 4 + 1] = v.y;
                    A[w][qq * 4 + 2] = v.z; A[w][qq * 4 + 3] = v.w;
                }
            }
            bool a_ok = active;
            uint32_t a_part = 0;
            if (HAS_E && active) {
                a_ok = emask[a] == 0;
                a_part = p > 1 ? part_of(edges, p, a) : 0;
            }
            for (; jb < s; jb += 32) {
                const bool more = jb + 32 < s;
                if (more) {
                    uint32_t* rows_n = rows0 + (buf ^ 1) * 32 * C::ROW;
                    rid0[(buf ^ 1) * 32 + lane] = nxt;
                    if (jb + 32 + lane < s) {
                        uint32_t* dst = rows_n + lane * C::ROW;
#pragma unroll
                        for (int w = 0; w < W; ++w)
#pragma unroll
                            for (int qq = 0; qq < NP / 4; ++qq)
                                cp_async16(dst + w * NP + qq * 4,
                                           tags + ((uint64_t)nxt * W + w) * 16 + qq * 4);
                    }
                    cp_async_commit();
                    nxt = (jb + 64 + lane < s) ? sids[st + jb + 64 + lane] : 0;
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncwarp();
                const uint32_t* rows = rows0 + buf * 32 * C::ROW;
                const uint32_t* rid = rid0 + buf * 32;
                const uint32_t un = min(32u, s - jb);
                const uint32_t u0 = (jb == c * 32) ? 1 : 0;
                for (uint32_t u = u0; u < un; ++u) {
                    const uint32_t bid = rid[u];
                    bool valid = a_ok && (jb + u > i);
                    const uint64_t dt = (uint64_t)bid - a;  // ids ascend within a bucket
                    valid = valid && dt > excl;
                    if (HAS_E && valid && emask[bid] && (p <= 1 || part_of(edges, p, bid) == a_part))
                        valid = false;
                    bool slow = false;
                    uint32_t qmask[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) qmask[w] = 0;
                    uint32_t flags = tflag;
                    if (valid) {
                        const uint32_t* R = rows + u * C::ROW;
                        if (MODE == MODE_MATCHED) {
                            uint32_t cnt = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                uint32_t s8 = pmask<W, NP>(A, R, w, 8);
                                if (w == W - 1) s8 &= last_mask;
                                qmask[w] = s8;
                                cnt += __popc(s8);
                            }
                            slow = cnt >= m;
                            flags |= QF_COUNT;
                        } else {
                            uint32_t early = 0, cnt = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                uint32_t x;
                                if (w <= wt) {
                                    x = pmask<W, NP>(A, R, w, 16);
                                    if (w == W - 1) x &= last_mask;
                                    early |= (w < wt) ? x : (x & low);
                                    if (w == wt) cnt += __popc(x & ~low);
                                } else if (MODE == MODE_FULL) {
                                    x = pmask<W, NP>(A, R, w, 8);
                                    if (w == W - 1) x &= last_mask;
                                    cnt += __popc(x);
                                } else {
                                    x = 0;
                                }
                                qmask[w] = x;
                            }
                            const bool need_count = (MODE == MODE_FULL) && cnt >= m;
                            if (early) {
                                slow = true;  // first-table rule needs confirmation
                                flags |= QF_DISTINCT | (need_count ? QF_COUNT : 0u);
                            } else {
                                ++distinct;
                                if (need_count) {
                                    slow = true;
                                    flags |= QF_COUNT;
                                }
                            }
                        }
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, slow);
                    if (bal) {
                        if (slow) {
                            const uint32_t e = (qhead + qn + __popc(bal & lt_mask)) & (QCAP - 1);
                            q.qa[e] = a;
                            q.qb[e] = bid;
                            q.qt[e] = flags;
#pragma unroll
                            for (int w = 0; w < W; ++w) q.qm[e * W + w] = qmask[w];
                        }
                        qn += __popc(bal);
                        if (qn >= 32) {
                            __syncwarp();
                            drain<W>(q, qhead, 32, lane, rkeys, t, m, out_key, out_sim, cap,
                                     counters, distinct);
                            qhead = (qhead + 32) & (QCAP - 1);
                            qn -= 32;
                        }
                    }
                }
                __syncwarp();
                buf ^= 1;
            }
        }
    }
    __syncwarp();
    if (qn) drain<W>(q, qhead, qn, lane, rkeys, t, m, out_key, out_sim, cap, counters, distinct);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, o);
    if (lane == 0 && distinct) atomicAdd(counters + 0, distinct);
}

// Generic path for t > 128 (any mode, no register caching): exact masks from
// the tag planes in global memory, confirmed on the keys.
__device__ __forceinline__ uint32_t gmask16(const uint32_t* __restrict__ tags, uint32_t W,
                                            uint32_t a, uint32_t b, int w) {
    const uint4* pa = (const uint4*)(tags + ((uint64_t)a * W + w) * 16);
    const uint4* pb = (const uint4*)(tags + ((uint64_t)b * W + w) * 16);
    uint32_t x = 0xFFFFFFFFu;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const uint4 u = __ldg(pa + qq), v = __ldg(pb + qq);
        x &= ~(u.x ^ v.x) & ~(u.y ^ v.y) & ~(u.z ^ v.z) & ~(u.w ^ v.w);
    }
    return x;
}

__global__ void __launch_bounds__(256) k_pairs_generic(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
    const uint64_t* __restrict__ chunk_off, uint64_t nb, const uint64_t* __restrict__ rkeys,
    const uint32_t* __restrict__ tags, uint32_t t, uint32_t m, uint64_t excl,
    const uint8_t* __restrict__ emask, const uint64_t* __restrict__ edges, uint32_t p, int mode,
    uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim, uint64_t cap,
    unsigned long long* __restrict__ counters) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t W = (t + 31) >> 5;
    const uint64_t total_chunks = chunk_off[nb];
    unsigned long long distinct = 0;
    for (uint64_t g = gwarp; g < total_chunks; g += nwarps) {
        uint64_t lo = 0, hi = nb;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (chunk_off[mid] <= g) lo = mid;
            else hi = mid;
        }
        const uint64_t b = lo, c = g - chunk_off[b], st = bstart[b];
        const uint32_t s = bsize[b], table = btab[b];
        const uint32_t i = (uint32_t)c * 32 + lane;
        if (i >= s) continue;
        const uint32_t a = sids[st + i];
        const bool a_ex = emask && emask[a];
        const uint32_t a_part = (emask && p > 1) ? part_of(edges, p, a) : 0;
        for (uint32_t j = i + 1; j < s; ++j) {
            const uint32_t bid = sids[st + j];
            const uint64_t dt = (uint64_t)bid - a;
            if (dt <= excl) continue;
            if (emask && (a_ex || (emask[bid] && (p <= 1 || part_of(edges, p, bid) == a_part)))) continue;
            bool first = true;
            uint32_t exact = 0;
            for (uint32_t w = 0; w < W; ++w) {
                uint32_t x = gmask16(tags, W, a, bid, (int)w);
                if (w == W - 1 && (t & 31)) x &= (1u << (t & 31)) - 1u;
                while (x) {
                    const uint32_t tt = w * 32 + __ffs(x) - 1;
                    x &= x - 1;
                    if (__ldg(rkeys + (uint64_t)a * t + tt) == __ldg(rkeys + (uint64_t)bid * t + tt)) {
                        if (tt < table) first = false;
                        ++exact;
                    }
                }
            }
            if (!first) continue;
            ++distinct;
            if (mode != MODE_DISTINCT && exact >= m) {
                const unsigned long long pos = atomicAdd(counters + 1, 1ULL);
                if (pos < cap) {
                    out_key[pos] = (dt << 32) | a;
                    out_sim[pos] = exact;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, o);
    if (lane == 0 && distinct && mode != MODE_MATCHED) atomicAdd(counters + 0, distinct);
}

__global__ void k_chunk_counts(const uint32_t* __restrict__ bsize, uint64_t nb,
                               uint64_t* __restrict__ off) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nb;
         i += (uint64_t)gridDim.x * blockDim.x)
        off[i] = i < nb ? (bsize[i] + 31) / 32 : 0;
}

template <int W, int MODE, bool HAS_E>
static int launch_pairs(const uint32_t* sids, const uint64_t* bstart, const uint32_t* bsize,
                        const uint32_t* btab, const uint64_t* off, uint64_t nb,
                        const uint64_t* rkeys, const uint32_t* tags, uint32_t t, uint32_t m,
                        uint64_t excl, const uint8_t* emask, const uint64_t* edges, uint32_t p,
                        uint64_t* out_key, uint32_t* out_sim, uint64_t cap,
                        unsigned long long* counters, unsigned long long* work, cudaStream_t st) {
    using C = PairCfg<W, MODE>;
    const size_t smem = (size_t)C::WARPS * C::PER_WARP * 4;
    auto kern = k_pairs<W, MODE, HAS_E>;
    QS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "smem attr");
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    kern<<<num_sms() * per_sm, C::WARPS * 32, smem, st>>>(sids, bstart, bsize, btab, off, nb, rkeys,
                                                         tags, t, m, excl, emask, edges, p, out_key,
                                                         out_sim, cap, counters, work);
    QS_CHECK_LAUNCH("k_pairs");
    return QS_OK;
}

template <int W>
static int dispatch_mode(int mode, bool has_e, const uint32_t* sids, const uint64_t* bstart,
                         const uint32_t* bsize, const uint32_t* btab, const uint64_t* off,
                         uint64_t nb, const uint64_t* rkeys, const uint32_t* tags, uint32_t t,
                         uint32_t m, uint64_t excl, const uint8_t* emask, const uint64_t* edges,
                         uint32_t p, uint64_t* ok, uint32_t* os, uint64_t cap,
                         unsigned long long* counters, unsigned long long* work, cudaStream_t st) {
#define QS_L(MM, EE) \
    launch_pairs<W, MM, EE>(sids, bstart, bsize, btab, off, nb, rkeys, tags, t, m, excl, emask, \
                            edges, p, ok, os, cap, counters, work, st)
    if (mode == MODE_FULL) return has_e ? QS_L(MODE_FULL, true) : QS_L(MODE_FULL, false);
    if (mode == MODE_MATCHED) return has_e ? QS_L(MODE_MATCHED, true) : QS_L(MODE_MATCHED, false);
    return has_e ? QS_L(MODE_DISTINCT, true) : QS_L(MODE_DISTINCT, false);
#undef QS_L
}

}  // namespace qs

using namespace qs;

extern "C" {

size_t qs_lsh_pairs_ws_bytes(uint64_t n_nonsingle) {
    return (size_t)(n_nonsingle + 2) * 8 + scan_ws_bytes(n_nonsingle + 1) + 512;
}

int qs_lsh_pairs(const uint32_t* sids_dev, const uint64_t* bstart_dev, const uint32_t* bsize_dev,
                 const uint32_t* btab_dev, uint64_t n_nonsingle, const uint64_t* rkeys_dev,
                 const uint32_t* tags_dev, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
                 const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p, int mode,
                 uint64_t* out_key_dev, uint32_t* out_sim_dev, uint64_t cap,
                 unsigned long long* counters_dev, void* ws_dev, size_t ws_bytes, void* stream) {
    (void)n;
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_pairs_ws_bytes(n_nonsingle), "pairs workspace too small");
    QS_ARG(m >= 1 && m <= t, "min_matches must be in [1, tables]");
    QS_ARG(mode >= 0 && mode <= 2, "mode must be 0 (full), 1 (matched) or 2 (distinct)");
    QS_ARG(t <= (1u << 24), "too many tables");
    if (n_nonsingle == 0) return QS_OK;
    uint64_t* off = (uint64_t*)ws_dev;
    unsigned long long* work = (unsigned long long*)(off + n_nonsingle + 1);
    void* sws = (void*)(((uintptr_t)(work + 1) + 63) & ~(uintptr_t)63);
    k_chunk_counts<<<qs_blocks(n_nonsingle + 1, 256), 256, 0, st>>>(bsize_dev, n_nonsingle, off);
    int rc = scan_u64(off, off, n_nonsingle + 1, nullptr, sws, st);
    if (rc) return rc;
    QS_CUDA(cudaMemsetAsync(work, 0, 8, st), "memset");
    const uint32_t W = (t + 31) >> 5;
    const bool has_e = excluded_dev != nullptr;
#define QS_D(WW)                                                                                  \
    dispatch_mode<WW>(mode, has_e, sids_dev, bstart_dev, bsize_dev, btab_dev, off, n_nonsingle,   \
                      rkeys_dev, tags_dev, t, m, excl, excluded_dev, edges_dev, p, out_key_dev,   \
                      out_sim_dev, cap, counters_dev, work, st)
    switch (W) {
        case 1: return QS_D(1);
        case 2: return QS_D(2);
        case 3: return QS_D(3);
        case 4: return QS_D(4);
        default:
            k_pairs_generic<<<num_sms() * 8, 256, 0, st>>>(
                sids_dev, bstart_dev, bsize_dev, btab_dev, off, n_nonsingle, rkeys_dev, tags_dev, t,
                m, excl, excluded_dev, edges_dev, p, mode, out_key_dev, out_sim_dev, cap,
                counters_dev);
            QS_CHECK_LAUNCH("k_pairs_generic");
            return QS_OK;
    }
#undef QS_D
}

}  // extern "C"
