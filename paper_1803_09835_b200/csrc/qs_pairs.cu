// Candidate-pair enumeration with exact collision counting (sm_100a).
//
// Replaces the reference's per-query gather + (q << 32 | c) key materialisation
// + sort + run-length count (lsh_search.py:175-219) and the >= m threshold
// (:261, :281).
//
// Work decomposition (persistent CTAs, warp-specialised producer/consumer):
//   * a work ITEM is a TILE of consecutive buckets of size <= L (<= 2L
//     members) or one (I, J) segment pair of a bigger bucket (L-member
//     segments); items are listed by a planning pass;
//   * one PRODUCER warp per CTA stages item k+1's member ids and bit-sliced
//     tag rows into the other half of a double-buffered shared-memory area
//     (cp.async, completion tracked by an mbarrier) while the CONSUMER warps
//     compare item k: each consumer warp takes 32-row x 64-row chunks, lane i
//     holds member a_i's tag planes in registers and compares them with the
//     later rows (broadcast shared-memory reads, 1 LOP3 per plane-word);
//   * consumers never wait for each other: a warp that runs out of chunks
//     releases the buffer (mbarrier arrive) and moves on to the next item, so
//     load latency and tail imbalance are both hidden.
//
// Exactness: each unordered pair is handled only in the bucket of its FIRST
// colliding table.  Tag-plane masks over-approximate the set of colliding
// tables (tags: false positives only), so every table a decision depends on
// is confirmed on the 64-bit keys (rkeys, row-major).  Confirmations are rare
// and divergent, so candidates are queued per warp in shared memory and
// drained 32 at a time with one candidate per lane.
//
// Tag layout: tags[2][n][W][8] uint32 (plane groups 0-7 / 8-15), W = ceil(t/32).
//
// Modes (warp-uniform, compile time):
//   FULL      distinct-pair count + emission of sim >= m (no occurrence filter)
//   MATCHED   emission only (occurrence-filter pass 1): screen on planes 0-7
//   DISTINCT  distinct-pair count only (pass 2 after the filter)
#include "qs_lsh.cuh"
#include <cstdlib>

namespace qs {

constexpr int QCAP = 64;
// Occupancy configuration (measured on B200 at cfg1, tools/sweep_pairs.py):
// 1 producer + 3 consumer warps per CTA; MATCHED rows (8 planes) run 5 CTAs/SM
// with two 16 KB staged buffers, the 16-plane modes 4 CTAs/SM with 21 KB.
#ifndef QS_CWARPS
#define QS_CWARPS 3
#endif
#ifndef QS_BUFKB_M
#define QS_BUFKB_M 16
#define QS_MINB_M 5
#endif
#ifndef QS_BUFKB
#define QS_BUFKB 21
#define QS_MINB 4
#endif
#ifndef QS_BUFKB_3
#define QS_BUFKB_3 21
#define QS_MINB_3 4
#endif
#ifndef QS_BUFKB_N
#define QS_BUFKB_N 14
#define QS_MINB_N 5
#endif
#ifndef QS_NBUF
#define QS_NBUF 2
#endif
constexpr int NBUF = QS_NBUF;          // staged items in flight per CTA (ring)
constexpr int CWARPS = QS_CWARPS;      // consumer warps per CTA (+1 producer warp)
#ifndef QS_NPROD
#define QS_NPROD 1
#endif
constexpr int NPROD = QS_NPROD;        // producer warps; producer p stages items k = p mod NPROD
static_assert(NPROD == 1 || NBUF % NPROD == 0, "each producer needs its own buffers");
constexpr int PTHREADS = (CWARPS + NPROD) * 32;
#ifndef QS_BPIECE
#define QS_BPIECE 16
#endif
constexpr uint32_t BPIECE = QS_BPIECE;  // B rows per chunk
constexpr uint32_t NCH_DONE = 0xFFFFFFFFu;
enum { MODE_FULL = 0, MODE_MATCHED = 1, MODE_DISTINCT = 2 };

#ifdef QS_PROF  // design instrumentation (not built by default)
__device__ unsigned long long g_prof[8];
#define PROF_DECL unsigned long long pr_acc[4] = {0, 0, 0, 0}; long long pr_t = 0;
#define PROF_START pr_t = clock64();
#define PROF_STOP(i) pr_acc[i] += (unsigned long long)(clock64() - pr_t);
#define PROF_FLUSH(base) if (lane == 0) for (int _i = 0; _i < 4; ++_i) atomicAdd(&g_prof[base + _i], pr_acc[_i]);
#else
#define PROF_DECL
#define PROF_START
#define PROF_STOP(i)
#define PROF_FLUSH(base)
#endif

// Staged row layout of a launch: tag planes kept per 32-table word.  MATCHED
// screens with planes 0-7 of every word; DISTINCT (one launch per table word
// WT, W = WT + 1) screens the words <= WT with planes 0-11 (a false early
// match, 1/4096 per table, only queues the pair for key confirmation); FULL
// (one launch per word WT) needs 16 planes of words <= WT (first-table test)
// and 8 of the later words (count screen).
constexpr int DISTINCT_PLANES = 12;
template <int MODE, int WT>
struct Layout {
    static constexpr int planes(int w) {
        return MODE == MODE_MATCHED ? 8
             : (MODE == MODE_DISTINCT ? DISTINCT_PLANES : (w <= WT ? 16 : 8));
    }
    static constexpr int off(int w) {  // closed form: folds to an immediate in unrolled loops
        return MODE == MODE_MATCHED ? 8 * w
             : (MODE == MODE_DISTINCT ? DISTINCT_PLANES * w
                : (w <= WT + 1 ? 16 * w : 16 * (WT + 1) + 8 * (w - WT - 1)));
    }
};

template <int W, int MODE, int WT>
struct TileCfg {
    using Lay = Layout<MODE, WT>;
    static constexpr int NP = MODE == MODE_MATCHED ? 8
                            : (MODE == MODE_DISTINCT ? DISTINCT_PLANES : 16);  // planes in registers
    static constexpr int ROW = Lay::off(W);                   // u32 per staged row
    // padded stride, an odd number of 16-byte units: row-parallel 16-byte
    // loads are conflict-free
    static constexpr int ROWP = ((ROW + 4) / 4) % 2 ? ROW + 4 : ROW + 8;
    // DISTINCT launches per table word with only words <= that word staged:
    // narrow rows (W <= 2) run more CTAs with smaller buffers
    static constexpr int BUFKB = MODE == MODE_MATCHED ? QS_BUFKB_M
                               : (ROW <= 32 ? QS_BUFKB_N : (ROW <= 48 ? QS_BUFKB_3 : QS_BUFKB));
    static constexpr int MINB = MODE == MODE_MATCHED ? QS_MINB_M
                              : (ROW <= 32 ? QS_MINB_N : (ROW <= 48 ? QS_MINB_3 : QS_MINB));
    static constexpr int CAP = (BUFKB * 1024) / (ROWP * 4);  // rows per buffer
    static constexpr int L = CAP / 2;                         // small-bucket / segment limit
    static constexpr int MAXCH = L + (2 * L / 32 + 1) * (2 * L / (int)BPIECE + 1) + 16;
    static constexpr int QWORDS = QCAP * (3 + W);
    // NBUF staged tag-row buffers + NMETA = NBUF + 1 item descriptors (member ids,
    // chunk list): the producer writes item k+1's descriptor while item k's rows
    // are in flight, so only one memory round trip separates "buffer free" from
    // "buffer full".
    static constexpr int NMETA = NBUF + NPROD;
    static constexpr size_t IDS_BYTES = ((size_t)CAP * 4 + 15) & ~(size_t)15;
    static constexpr size_t ROWBUF = ((size_t)CAP * ROWP * 4 + 127) & ~(size_t)127;
    static constexpr size_t META = ((IDS_BYTES + (size_t)MAXCH * 8) + 127) & ~(size_t)127;
    static constexpr size_t SMEM = NBUF * ROWBUF + NMETA * META + (size_t)CWARPS * QWORDS * 4 + 128;
};

// ------------------------------------------------------------ primitives
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
// expect `bytes` of bulk-copy transactions on the barrier and arrive once
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
// TMA-engine bulk copy global -> shared (16-byte aligned, size % 16 == 0),
// completion counted on the barrier's transaction count
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

// AND over np planes of ~(A ^ B) for 32-table word w of the staged row R
// (uniform across the warp: broadcast shared-memory reads, immediate offsets).
template <int W, int NP>
__device__ __forceinline__ uint32_t pmask(const uint32_t (&A)[W][NP], const uint32_t* R, int w,
                                          int np, int woff) {
    uint32_t x = 0xFFFFFFFFu;
    const uint4* r4 = (const uint4*)(R + woff);
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
    if (stop_first && cand) {
        // the lowest candidate alone first: for a pair that is not first in
        // this bucket it is usually a true collision, and the other three key
        // pairs of a batch would be wasted random reads
        const uint32_t t0 = (uint32_t)(__ffs(cand) - 1);
        if (__ldg(ra + t0) == __ldg(rb + t0)) return 1;
        cand &= cand - 1;
    }
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

// confirm() that stops once `need` tables agree: the tables it did not
// examine stay in `cand` (lazy counts, completed later for surviving pairs)
__device__ __forceinline__ uint32_t confirm_upto(const uint64_t* __restrict__ rkeys, uint32_t t,
                                                 uint32_t a, uint32_t b, uint32_t& cand,
                                                 uint32_t wbase, uint32_t need) {
    uint32_t hits = 0;
    const uint64_t* ra = rkeys + (uint64_t)a * t + wbase;
    const uint64_t* rb = rkeys + (uint64_t)b * t + wbase;
    while (cand && hits < need) {
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
    }
    return hits;
}

// Queue entry flags (bits 0..7 = table & 0xFF, bits 16.. = table >> 8)
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
// Every launch covers one table word (wt == WT), so the word loops have
// compile-time bounds; they stay rolled (one copy of each confirmation loop
// per call site instead of W: the kernel's code shrinks by half, and with it
// the instruction-fetch stalls of the warps that enter a drain), and the
// unexamined candidate words of a lazy count go back into the lane's own
// queue slot instead of a register array.
#ifndef QS_DRAIN_INLINE
#define QS_DRAIN_INLINE __forceinline__
#endif
template <int W, int WT>
__device__ QS_DRAIN_INLINE void drain(const Queue& q, uint32_t base, uint32_t cnt, uint32_t lane,
                                      const uint64_t* __restrict__ rkeys, uint32_t t, uint32_t m,
                                      uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim,
                                      uint32_t* __restrict__ out_rest,
                                      uint64_t cap, unsigned long long* __restrict__ counters,
                                      unsigned long long& distinct) {
    if (lane < cnt) {
        const uint32_t e = (base + lane) & (QCAP - 1);
        QS_DASSERT(e < QCAP);
        const uint32_t a = q.qa[e], b = q.qb[e], f = q.qt[e];
        QS_DASSERT(a < b);
        const uint32_t table = (f & 0xFFu) | ((f >> 16) << 8);
        QS_DASSERT((int)(table >> 5) == WT);
        const uint32_t bt = table & 31, low = (1u << bt) - 1u;
        uint32_t* qm = q.qm + e * W;
        bool first = true;
#pragma unroll 1
        for (int w = 0; w <= WT; ++w) {
            const uint32_t mw = qm[w];
            const uint32_t ebits = (w < WT) ? mw : (mw & low);
            if (ebits && confirm(rkeys, t, a, b, ebits, w * 32, true)) {
                first = false;
                break;
            }
        }
        if (first) {
            if (f & QF_DISTINCT) ++distinct;
            if (f & QF_COUNT) {
                // lazy (out_rest given, MATCHED): stop confirming once the pair
                // reaches m and keep the unexamined candidate tables, so the
                // exact count is completed only for pairs the filter keeps
                const bool lazy = out_rest != nullptr;
                uint32_t exact = 1;
#pragma unroll 1
                for (int w = WT; w < W; ++w) {
                    const uint32_t mw = qm[w];
                    uint32_t x = (w == WT) ? (mw & ~((low << 1) | 1u)) : mw;
                    if (lazy) {
                        if (x && exact < m) exact += confirm_upto(rkeys, t, a, b, x, w * 32, m - exact);
                        qm[w] = x;
                    } else if (x) {
                        exact += confirm(rkeys, t, a, b, x, w * 32, false);
                    }
                }
                if (exact >= m) {
                    const unsigned long long pos = atomicAdd(counters + 1, 1ULL);
                    if (pos < cap) {
                        out_key[pos] = ((uint64_t)(b - a) << 32) | a;
                        out_sim[pos] = exact;
                        if (lazy) {
#pragma unroll
                            for (int w = 0; w < W; ++w) out_rest[pos * W + w] = w < WT ? 0u : qm[w];
                        }
                    }
                }
            }
        }
    }
    __syncwarp();
}

// Items of a bucket of s > L members.  Up to 2L members fit one buffer as a
// single item (all rows, every pair).  A bigger bucket is cut into 32-row A
// groups g (rows [32g, 32g + 32)); each group pairs with the later rows
// [32(g+1), s) in balanced B pieces of <= 2L - 32 rows, item (g, J), and the
// group's first piece also carries its own triangle (a fold chunk).  Every
// rectangular step then has a full 32-row A group except in the last group
// (balanced I x J segments of <= L rows left lanes idle: 70 % lane use at cfg1).
//
// Core-first lists (MATCHED passes after the first table word, occurrence
// filter on): the bucket's nc members known to be core are listed first and
// pairs of two of them are skipped (they change no output: both endpoints are
// excluded whatever their count).  A group wholly inside the core prefix keeps
// only the B rows >= nc and no triangle; every other group is unchanged.
__host__ __device__ __forceinline__ uint32_t big_bmax(uint32_t L) { return 2 * L - 32; }
// first B row of A group g and whether its triangle is needed
__host__ __device__ __forceinline__ uint32_t g_blo(uint32_t s, uint32_t nc, uint32_t g, bool& tri) {
    const uint32_t a0 = 32 * g, acnt = s - a0 < 32 ? s - a0 : 32u;
    const bool full_core = a0 + acnt <= nc;
    tri = !full_core && acnt >= 2;
    const uint32_t b0 = a0 + acnt;
    return full_core ? (nc > b0 ? nc : b0) : b0;
}
__host__ __device__ __forceinline__ uint32_t g_pieces(uint32_t s, uint32_t nc, uint32_t g, uint32_t bmax) {
    bool tri;
    const uint32_t blo = g_blo(s, nc, g, tri);
    return s > blo ? (s - blo + bmax - 1) / bmax : (tri ? 1u : 0u);
}
__host__ __device__ __forceinline__ uint32_t big_groups(uint32_t s, uint32_t L) {
    return s <= 2 * L ? 1u : (s + 31) / 32;
}
__host__ __device__ __forceinline__ uint64_t big_items(uint32_t s, uint32_t nc, uint32_t L) {
    if (s <= 2 * L) return 1;
    uint64_t c = 0;
    for (uint32_t g = 0, ng = big_groups(s, L); g < ng; ++g) c += g_pieces(s, nc, g, big_bmax(L));
    return c;
}

// chunk descriptor: x = abase | bbeg << 16; y = bend | acnt << 16 | tri << 22 | table << 23
__device__ __forceinline__ uint2 make_chunk(uint32_t abase, uint32_t acnt, uint32_t bbeg,
                                            uint32_t bend, bool tri, uint32_t table) {
    return make_uint2(abase | (bbeg << 16),
                      bend | (acnt << 16) | ((tri ? 1u : 0u) << 22) | (table << 23));
}
__device__ __forceinline__ uint32_t n_pieces(uint32_t bb, uint32_t be) {
    return be > bb ? (be - bb + BPIECE - 1) / BPIECE : 0;
}
// all chunks of the rows [off, off + s) of one bucket (pairs j > i): per
// 32-row A group one FOLD chunk for the pairs inside the group (lane i meets
// row i + d mod acnt, d = 1 .. acnt / 2: the triangle in acnt / 2 steps with
// every lane busy) and rectangular pieces for the later rows
// (fold = false: triangle pieces from row i + 1 with per-lane validity, the
// MATCHED pass's choice — measured faster there, its broadcast row loads
// matter more than the idle lanes)
__device__ __forceinline__ uint32_t count_chunks_tri(uint32_t s, bool fold) {
    uint32_t n = 0;
    for (uint32_t c = 0; c * 32 < s; ++c) {
        const uint32_t acnt = min(32u, s - c * 32);
        n += fold ? (acnt >= 2 ? 1u : 0u) + n_pieces(c * 32 + acnt, s) : n_pieces(c * 32 + 1, s);
    }
    return n;
}
__device__ __forceinline__ void emit_chunks_tri(uint2* chunks, uint32_t base, uint32_t off,
                                                uint32_t s, uint32_t table, bool fold) {
    for (uint32_t c = 0; c * 32 < s; ++c) {
        const uint32_t ab = off + c * 32, acnt = min(32u, s - c * 32);
        if (fold && acnt >= 2) chunks[base++] = make_chunk(ab, acnt, 0, 0, true, table);
        QS_DASSERT(acnt >= 1 && acnt <= 32);
        const uint32_t first = fold ? acnt : 1;
        const uint32_t np = n_pieces(c * 32 + first, s);
        for (uint32_t k = 0; k < np; ++k) {
            const uint32_t b0 = ab + first + k * BPIECE;
            chunks[base++] = make_chunk(ab, acnt, b0, min(off + s, b0 + BPIECE), !fold, table);
        }
    }
}

// all chunks of a whole bucket of s rows whose first nc rows are core: per A
// group the triangle (unless wholly core) and the B rows from g_blo
__device__ __forceinline__ uint32_t chunks_nc(uint2* chunks, uint32_t s, uint32_t nc, uint32_t table,
                                              bool fold, bool emit) {
    uint32_t n = 0;
    for (uint32_t c = 0; c * 32 < s; ++c) {
        const uint32_t ab = c * 32, acnt = min(32u, s - ab);
        bool tri;
        const uint32_t blo = g_blo(s, nc, c, tri);
        if (tri) {
            if (fold) {
                if (emit) chunks[n] = make_chunk(ab, acnt, 0, 0, true, table);
                ++n;
            } else {
                const uint32_t np = n_pieces(ab + 1, ab + acnt);
                for (uint32_t k = 0; k < np; ++k) {
                    const uint32_t b0 = ab + 1 + k * BPIECE;
                    if (emit) chunks[n] = make_chunk(ab, acnt, b0, min(ab + acnt, b0 + BPIECE), true, table);
                    ++n;
                }
            }
        }
        const uint32_t np = n_pieces(blo, s);
        for (uint32_t k = 0; k < np; ++k) {
            const uint32_t b0 = blo + k * BPIECE;
            if (emit) chunks[n] = make_chunk(ab, acnt, b0, min(s, b0 + BPIECE), false, table);
            ++n;
        }
    }
    return n;
}

template <int W, class Lay, int ROWP>
__device__ __forceinline__ void stage_row(uint32_t* rows, uint32_t pos, const uint32_t* __restrict__ tags,
                                          uint64_t n, uint32_t id, uint32_t wg) {
    QS_DASSERT(id < n);
    uint4* dst = (uint4*)(rows + pos * ROWP);
#pragma unroll
    for (int w = 0; w < W; ++w)
#pragma unroll
        for (int qq = 0; qq < Lay::planes(w) / 4; ++qq) {
            const uint32_t grp = qq >> 1;  // plane group (0: planes 0-7, 1: planes 8-15)
            cp_async16(dst + (Lay::off(w) / 4 + qq),
                       tags + ((uint64_t)grp * n + id) * wg * 8 + w * 8 + (qq & 1) * 4);
        }
}

struct Plan {
    const uint64_t* mpre;        // exclusive prefix of small-bucket sizes (nb + 1)
    const uint64_t* tile_first;  // first bucket of each tile (n_tiles + 1)
    const uint64_t* bigitems;    // (bucket << 24) | (I << 12) | J per big item (if totals[5])
    const uint64_t* bigb;        // big bucket indices
    const uint64_t* bigoff;      // exclusive prefix of items per big bucket
    const uint64_t* totals;      // [0] small members, [1] n_big, [2] n_tiles, [3] n_bigitems,
                                 // [4] max segments per bucket, [5] item table valid
    const uint32_t* nc;          // core members per bucket, listed first (nullptr: none)
};

template <int W, int MODE, bool HAS_E, int WT, bool EX>
__global__ void __launch_bounds__(PTHREADS, TileCfg<W, MODE, WT>::MINB) k_pairs_pc(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab, Plan plan,
    const uint64_t* __restrict__ rkeys, const uint32_t* __restrict__ tags, uint64_t n, uint32_t t,
    uint32_t m, uint64_t excl, const uint8_t* __restrict__ emask, const uint64_t* __restrict__ edges,
    uint32_t p, uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim,
    uint32_t* __restrict__ out_rest, uint64_t cap, unsigned long long* __restrict__ counters,
    unsigned long long* __restrict__ work, uint32_t tmax, uint32_t wg) {
    // W = tag words staged per row (words 0..W-1); wg = words per row in `tags`;
    // WT = the launch's table word (DISTINCT / FULL are launched per word)
    using C = TileCfg<W, MODE, WT>;
    using Lay = typename C::Lay;
    constexpr int NP = C::NP;
    constexpr uint32_t L = C::L;
#ifndef QS_FOLD_MATCHED
#define QS_FOLD_MATCHED 1
#endif
#ifndef QS_FOLD_OFF
    constexpr bool FOLD = MODE != MODE_MATCHED || QS_FOLD_MATCHED;  // fold chunks for triangles
#else
    constexpr bool FOLD = false;
#endif
    extern __shared__ __align__(128) unsigned char psm[];
    __shared__ __align__(8) uint64_t full_bar[NBUF], empty_bar[NBUF];
    __shared__ uint32_t s_nch[C::NMETA], s_next[C::NMETA], s_nrows[C::NMETA];
    // producer scratch: tile bucket metadata, small-bucket offsets / member-list starts
    __shared__ uint64_t p_st_all[NPROD][L];
    __shared__ uint32_t p_off_all[NPROD][L + 1];
    // rows buffer b | item descriptor a: member ids, chunk descriptors
    auto rowsb = [&](int b) { return (uint32_t*)(psm + b * C::ROWBUF); };
    auto idsm = [&](int a) { return (uint32_t*)(psm + NBUF * C::ROWBUF + a * C::META); };
    auto chm = [&](int a) {
        return (uint2*)(psm + NBUF * C::ROWBUF + a * C::META + C::IDS_BYTES);
    };
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NBUF; ++i) {
            mbar_init(&full_bar[i], 64);
            mbar_init(&empty_bar[i], CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const uint64_t n_tiles = plan.totals[2], n_items = n_tiles + plan.totals[3];
    const bool use_table = plan.totals[5] != 0;

    if (warp >= CWARPS) {
        const uint32_t pw = warp - CWARPS;  // producer index
        uint64_t* p_st = p_st_all[pw];
        uint32_t* p_off = p_off_all[pw];
        // ================================================= producer warp
        PROF_DECL
        unsigned long long item_next = 0;
        if (lane == 0) item_next = atomicAdd(work, 1ULL);
        // item -> descriptor area ma: member ids and chunk descriptors (blocking:
        // bucket metadata and ids are two dependent round trips)
        auto stage_meta = [&](int ma) {
            // the next grab is issued one item ahead so its latency overlaps this item
            const unsigned long long item = __shfl_sync(0xffffffffu, item_next, 0);
            if (lane == 0 && item < n_items) item_next = atomicAdd(work, 1ULL);
            uint32_t* ids = idsm(ma);
            uint2* chunks = chm(ma);
            if (item >= n_items) {
                if (lane == 0) s_nch[ma] = NCH_DONE;
                __syncwarp();
                return;
            }
            if (lane == 0) {
                s_nch[ma] = 0;
                s_next[ma] = 0;
            }
            __syncwarp();
            if (item < n_tiles) {
                const uint64_t b0 = plan.tile_first[item], b1 = plan.tile_first[item + 1];
                const uint32_t cnt = (uint32_t)(b1 - b0);
                const uint64_t mbase = __ldg(plan.mpre + b0);
                // small buckets of the tile (positive entries of the member prefix;
                // big and left-out buckets count 0), order-preserving compaction with
                // one lane per bucket, and their chunk descriptors
                const uint32_t lt = (1u << lane) - 1u;
                uint32_t nsb = 0;
                for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
                    const uint32_t i = i0 + lane;
                    uint64_t mp0 = 0, mp1 = 0;
                    if (i < cnt) {
                        mp0 = __ldg(plan.mpre + b0 + i);
                        mp1 = __ldg(plan.mpre + b0 + i + 1);
                    }
                    const bool small = mp1 > mp0;
                    const uint32_t bal = __ballot_sync(0xffffffffu, small);
                    if (small) {
                        const uint32_t s = (uint32_t)(mp1 - mp0);
                        const uint32_t kk = nsb + __popc(bal & lt);
                        const uint32_t off = (uint32_t)(mp0 - mbase);
                        QS_DASSERT(kk < L);
                        p_off[kk] = off;
                        p_st[kk] = __ldg(bstart + b0 + i);
                        const uint32_t cb = atomicAdd(&s_nch[ma], count_chunks_tri(s, FOLD));
                        emit_chunks_tri(chunks, cb, off, s, __ldg(btab + b0 + i), FOLD);
                    }
                    nsb += __popc(bal);
                }
                const uint32_t tot = (uint32_t)(__ldg(plan.mpre + b1) - mbase);
                if (lane == 0) p_off[nsb] = tot;
                __syncwarp();
                // member ids, one lane per member (bucket found by binary search)
                for (uint32_t r = lane; r < tot; r += 32) {
                    uint32_t lo = 0, hi = nsb;
                    while (hi - lo > 1) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (p_off[mid] <= r) lo = mid;
                        else hi = mid;
                    }
                    QS_DASSERT(r < C::CAP && lo < nsb);
                    cp_async4(ids + r, sids + p_st[lo] + (r - p_off[lo]));
                }
                cp_async_wait_all();
                __syncwarp();
                if (lane == 0) s_nrows[ma] = tot;
            } else {
                uint64_t bk;
                uint32_t g, J;
                if (use_table) {
                    const uint64_t e = plan.bigitems[item - n_tiles];
                    bk = e >> 24;
                    g = (uint32_t)(e >> 12) & 0xFFFu;
                    J = (uint32_t)e & 0xFFFu;
                } else {  // giant buckets: decode (bucket, g, J) from the item prefix
                    const uint64_t idx = item - n_tiles;
                    uint64_t lo = 0, hi = plan.totals[1];
                    while (hi - lo > 1) {
                        const uint64_t mid = (lo + hi) >> 1;
                        if (plan.bigoff[mid] <= idx) lo = mid;
                        else hi = mid;
                    }
                    bk = plan.bigb[lo];
                    const uint32_t sb = bsize[bk], ncb = plan.nc ? plan.nc[bk] : 0u;
                    uint64_t rem = idx - plan.bigoff[lo];
                    uint32_t gg = 0;
                    if (sb > 2 * L) {
                        while (rem >= g_pieces(sb, ncb, gg, big_bmax(L))) {
                            rem -= g_pieces(sb, ncb, gg, big_bmax(L));
                            ++gg;
                        }
                    }
                    g = gg;
                    J = (uint32_t)rem;
                }
                const uint32_t s = bsize[bk];
                const uint32_t nc = plan.nc ? plan.nc[bk] : 0u;
                const uint64_t st = bstart[bk];
                uint32_t a0 = 0, nA = s, j0 = 0, nB = 0;  // s <= 2L: the whole bucket
                bool gtri = true;
                if (s > 2 * L) {
                    a0 = 32 * g;
                    nA = min(32u, s - a0);
                    const uint32_t blo = g_blo(s, nc, g, gtri), lb = s > blo ? s - blo : 0;
                    if (lb) {
                        const uint32_t np = g_pieces(s, nc, g, big_bmax(L)), pl = (lb + np - 1) / np;
                        j0 = blo + J * pl;
                        nB = min(pl, s - j0);
                    }
                }
                QS_DASSERT(nA + nB <= C::CAP);
                for (uint32_t r = lane; r < nA + nB; r += 32) {
                    QS_DASSERT(r < C::CAP);
                    cp_async4(ids + r, sids + st + (r < nA ? a0 + r : j0 + (r - nA)));
                }
                if (lane == 0) {
                    const uint32_t table = btab[bk];
                    uint32_t cbase = 0;
                    if (s <= 2 * L) {  // the whole bucket (pairs of two core rows left out)
                        cbase = chunks_nc(chunks, s, nc, table, FOLD, true);
                        nB = 0;
                    } else if (J == 0 && gtri) {  // group g's own triangle
                        emit_chunks_tri(chunks, 0, 0, nA, table, FOLD);
                        cbase = count_chunks_tri(nA, FOLD);
                    }
                    const uint32_t np = n_pieces(nA, nA + nB);
                    for (uint32_t kk = 0; kk < np; ++kk) {
                        const uint32_t bb = nA + kk * BPIECE;
                        chunks[cbase++] = make_chunk(0, nA, bb, min(nA + nB, bb + BPIECE), false, table);
                    }
                    QS_DASSERT(cbase <= C::MAXCH);
                    s_nch[ma] = cbase;
                }
                cp_async_wait_all();
                __syncwarp();
                if (lane == 0) s_nrows[ma] = nA + nB;
            }
            __syncwarp();
        };
        stage_meta(pw % C::NMETA);
        for (uint32_t k = pw;; k += NPROD) {
            const int b = k % NBUF, ma = k % C::NMETA;
            PROF_START
            if (k >= NBUF) mbar_wait(&empty_bar[b], ((k / NBUF) - 1) & 1);
            PROF_STOP(0)
            PROF_START
            // MATCHED rows are the first plane group of every word, contiguous in
            // `tags` ([2][n][W][8]): one TMA bulk copy per row, completion on the
            // barrier's transaction count; the other modes gather planes of
            // some words (per-thread 16-byte cp.async)
            const bool bulk = MODE == MODE_MATCHED && (uint32_t)W == wg;
            if (s_nch[ma] == NCH_DONE) {
                if (bulk) mbar_arrive(&full_bar[b]);
                else mbar_arrive_cp_async(&full_bar[b]);
                mbar_arrive(&full_bar[b]);
                break;
            }
            {
                uint32_t* rows = rowsb(b);
                const uint32_t* ids = idsm(ma);
                const uint32_t nrows = s_nrows[ma];
                if (bulk) {
                    constexpr uint32_t RB = (uint32_t)C::ROW * 4;
                    const uint32_t mine = nrows > lane ? (nrows - lane + 31) / 32 : 0;
                    mbar_arrive_expect_tx(&full_bar[b], mine * RB);
                    for (uint32_t r = lane; r < nrows; r += 32) {
                        QS_DASSERT(r < C::CAP && ids[r] < n);
                        bulk_g2s(rows + r * C::ROWP, tags + (uint64_t)ids[r] * wg * 8, RB, &full_bar[b]);
                    }
                } else {
                    for (uint32_t r = lane; r < nrows; r += 32)
                        stage_row<W, Lay, C::ROWP>(rows, r, tags, n, ids[r], wg);
                }
            }
            __syncwarp();
            if (!bulk) mbar_arrive_cp_async(&full_bar[b]);  // fires when this lane's row copies land
            mbar_arrive(&full_bar[b]);                       // releases the descriptor of item k
            // look ahead: the descriptor area of item k + NPROD belonged to item
            // k + NPROD - NMETA = k - NBUF, released by the empty wait above
            stage_meta((k + NPROD) % C::NMETA);
            PROF_STOP(1)
        }
        PROF_FLUSH(0)
        return;
    }

    // ===================================================== consumer warps
    PROF_DECL
    uint32_t* qbase = (uint32_t*)(psm + NBUF * C::ROWBUF + C::NMETA * C::META) + warp * C::QWORDS;
    Queue q;
    q.qa = qbase;
    q.qb = q.qa + QCAP;
    q.qt = q.qb + QCAP;
    q.qm = q.qt + QCAP;
    uint32_t qhead = 0, qn = 0;
    const uint32_t last_mask = (t & 31) ? ((1u << (t & 31)) - 1u) : 0xFFFFFFFFu;
    const uint32_t lt_mask = (1u << lane) - 1u;
    unsigned long long distinct = 0;

    uint32_t finished = 0;  // bit p: producer p has no more items
    for (uint32_t k = 0;; ++k) {
        const int bsel = k % NBUF, msel = k % C::NMETA;
        if (finished & (1u << (k % NPROD))) continue;
        PROF_START
        mbar_wait(&full_bar[bsel], (k / NBUF) & 1);
        PROF_STOP(0)
        PROF_START
        const uint32_t nch = s_nch[msel];
        if (nch == NCH_DONE) {
            finished |= 1u << (k % NPROD);
            if (finished == (1u << NPROD) - 1u) break;
            continue;
        }
        const uint32_t* rows = rowsb(bsel);
        const uint32_t* ids = idsm(msel);
        const uint2* chunks = chm(msel);
        while (true) {
            uint32_t ci = 0;
            if (lane == 0) ci = atomicAdd(&s_next[msel], 1u);
            ci = __shfl_sync(0xffffffffu, ci, 0);
            if (ci >= nch) break;
            QS_DASSERT(ci < C::MAXCH);
            const uint2 d = chunks[ci];
            const uint32_t abase = d.x & 0xFFFFu, bbeg = d.x >> 16;
            const uint32_t bend = d.y & 0xFFFFu, acnt = (d.y >> 16) & 63u;
            const bool tri = (d.y >> 22) & 1u;
            const uint32_t table = d.y >> 23;
            const int wt = (int)(table >> 5);
            const uint32_t bt = table & 31, low = (1u << bt) - 1u;
            const uint32_t tflag = (table & 0xFFu) | ((table >> 8) << 16);
            const bool active = lane < acnt;
            const uint32_t apos = abase + (active ? lane : 0);
            const uint32_t a = ids[apos];
            uint32_t A[W][NP];
            {
                const uint4* src = (const uint4*)(rows + apos * C::ROWP);
#pragma unroll
                for (int w = 0; w < W; ++w)
#pragma unroll
                    for (int qq = 0; qq < Lay::planes(w) / 4; ++qq) {
                        const uint4 v = src[Lay::off(w) / 4 + qq];
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
            constexpr bool excl_on = EX;  // exclusion windows (excl > 0) at compile time
            // evaluate the pair (a, row u): validity, tag-plane masks, queue decision.
            // Rectangular chunks: row u lies after every A row (its id is larger).
            // Fold chunks: row u may precede the lane's row, so the pair is taken
            // in canonical (smaller id, larger id) order.
            auto eval = [&](uint32_t u, const uint32_t* R, bool fold, bool fold_ok, bool& slow,
                            uint32_t& flags, uint32_t (&qmask)[W]) {
                bool valid;
                if (fold) {
                    valid = fold_ok;
                    if (excl_on || HAS_E) {
                        const uint32_t bid = ids[u];
                        const uint32_t c = min(a, bid), qv = max(a, bid);
                        if (excl_on) valid = valid && (uint64_t)(qv - c) > excl;
                        if (HAS_E && valid) {
                            if (emask[c]) valid = false;
                            else if (emask[qv] && (p <= 1 || part_of(edges, p, qv) ==
                                                                 part_of(edges, p, c)))
                                valid = false;
                        }
                    }
                } else {
                    valid = a_ok && u >= (tri ? apos + 1 : bbeg);  // tri: pairs j > i
                    if (excl_on || HAS_E) {
                        const uint32_t bid = ids[u];
                        // ids ascend in a bucket unless its list is core-first permuted
                        if (excl_on) valid = valid && (uint64_t)(max(a, bid) - min(a, bid)) > excl;
                        if (HAS_E && valid && emask[bid] &&
                            (p <= 1 || part_of(edges, p, bid) == a_part))
                            valid = false;
                    }
                }
                slow = false;
                flags = tflag;
                // masks are computed for every lane (no divergence); invalid lanes drop them
                if (MODE == MODE_MATCHED) {
                    // the bucket's table T must be the pair's first collision, so a
                    // pair with sim >= m collides in >= m - 1 tables after T: screen
                    // on those words only (earlier words are built in push())
                    uint32_t cnt = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        uint32_t s8 = 0;
                        if (w >= WT) {  // launches are per table word: wt == WT
                            s8 = pmask<W, NP>(A, R, w, 8, Lay::off(w));
                            if (w == (int)wg - 1) s8 &= last_mask;
                            cnt += __popc(w == WT ? (s8 & ~((low << 1) | 1u)) : s8);
                        }
                        qmask[w] = s8;
                    }
                    slow = valid && cnt + 1 >= m;
                    flags |= QF_COUNT;
                } else {
                    uint32_t early = 0, cnt = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        uint32_t x = 0;
                        if (w <= WT) {  // launches are per table word: wt == WT
                            x = pmask<W, NP>(A, R, w, Lay::planes(w), Lay::off(w));
                            if (w == (int)wg - 1) x &= last_mask;
                            early |= (w < WT) ? x : (x & low);
                            if (w == WT) cnt += __popc(x & ~low);
                        } else if (MODE == MODE_FULL) {
                            x = pmask<W, NP>(A, R, w, 8, Lay::off(w));
                            if (w == (int)wg - 1) x &= last_mask;
                            cnt += __popc(x);
                        }
                        qmask[w] = x;
                    }
                    const bool need_count = (MODE == MODE_FULL) && cnt >= m;
                    if (valid) {
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
            };
            // queue the warp's slow lanes; drain 32 once the queue holds 32
            auto push = [&](uint32_t u, const uint32_t* R, bool fold, bool slow, uint32_t flags,
                            uint32_t (&qmask)[W]) {
                const uint32_t bal = __ballot_sync(0xffffffffu, slow);
                if (bal) {
                    if (MODE == MODE_MATCHED) {
#pragma unroll
                        for (int w = 0; w < W; ++w)
                            if (w < WT) qmask[w] = pmask<W, NP>(A, R, w, 8, Lay::off(w));
                    }
                    if (slow) {
                        const uint32_t e = (qhead + qn + __popc(bal & lt_mask)) & (QCAP - 1);
                        const uint32_t bid = ids[u];
                        const uint32_t qa = min(a, bid), qb = max(a, bid);
                        QS_DASSERT(e < QCAP && qa < qb && qb < n);
                        q.qa[e] = qa;
                        q.qb[e] = qb;
                        q.qt[e] = flags;
#pragma unroll
                        for (int w = 0; w < W; ++w) q.qm[e * W + w] = qmask[w];
                    }
                    qn += __popc(bal);
                    if (qn >= 32) {
                        __syncwarp();
                        PROF_STOP(1)
                        PROF_START
                        drain<W, WT>(q, qhead, 32, lane, rkeys, t, m, out_key, out_sim, out_rest, cap,
                                 counters, distinct);
                        PROF_STOP(2)
                        PROF_START
                        qhead = (qhead + 32) & (QCAP - 1);
                        qn -= 32;
                    }
                }
            };
#ifndef QS_PAIR_MERGED
#define QS_PAIR_MERGED 0
#endif
            if (QS_PAIR_MERGED && FOLD && MODE != MODE_DISTINCT) {
                // one loop (one copy of eval / push / drain in the kernel) for fold
                // and rectangular chunks: the step's row is per-lane in a fold
                // chunk and the same for every lane otherwise
                const bool fold = tri;
                const uint32_t nst = fold ? (acnt >> 1) : (bend > bbeg ? bend - bbeg : 0u);
                for (uint32_t st = 0; st < nst; ++st) {
                    uint32_t u = bbeg + st;
                    bool ok = false;
                    if (fold) {
                        const uint32_t dd = st + 1;
                        uint32_t j = lane + dd;
                        if (j >= acnt) j -= acnt;
                        ok = active && (2 * dd != acnt || lane < dd);
                        u = abase + (active ? j : 0);
                    }
                    const uint32_t* R = rows + u * C::ROWP;
                    bool s0;
                    uint32_t f0, m0[W];
                    eval(u, R, fold, ok, s0, f0, m0);
                    push(u, R, fold, s0, f0, m0);
                }
            } else if (FOLD && tri) {
                // fold chunk: the pairs among the chunk's own acnt rows, lane i
                // against row i + dd (mod acnt); at dd = acnt / 2 (even acnt) the
                // lanes i < dd cover every pair once
                const uint32_t nst = acnt >> 1;
                for (uint32_t dd = 1; dd <= nst; ++dd) {
                    uint32_t j = lane + dd;
                    if (j >= acnt) j -= acnt;
                    const bool ok = active && (2 * dd != acnt || lane < dd);
                    const uint32_t u = abase + (active ? j : 0);
                    const uint32_t* R = rows + u * C::ROWP;
                    bool s0;
                    uint32_t f0, m0[W];
                    eval(u, R, true, ok, s0, f0, m0);
                    push(u, R, true, s0, f0, m0);
                }
            } else {
                uint32_t u = bbeg;
                const uint32_t* R = rows + bbeg * C::ROWP;
#ifndef QS_PAIR_UNROLL2
#define QS_PAIR_UNROLL2 1
#endif
#if QS_PAIR_UNROLL2
                // DISTINCT: two rows per iteration, their independent mask chains
                // interleave (-2 to -3 ms per bucket-size class at cfg1; the MATCHED
                // pass at its 96-register cap gets slower: 220 -> 294 ms)
#ifndef QS_UNROLL_MATCHED
#define QS_UNROLL_MATCHED 0
#endif
                if (MODE == MODE_DISTINCT || (MODE == MODE_MATCHED && QS_UNROLL_MATCHED))
                for (; u + 1 < bend; u += 2, R += 2 * C::ROWP) {
                    bool s0, s1;
                    uint32_t f0, f1, m0[W], m1[W];
                    eval(u, R, false, false, s0, f0, m0);
                    eval(u + 1, R + C::ROWP, false, false, s1, f1, m1);
                    push(u, R, false, s0, f0, m0);
                    push(u + 1, R + C::ROWP, false, s1, f1, m1);
                }
#endif
                for (; u < bend; ++u, R += C::ROWP) {
                    bool s0;
                    uint32_t f0, m0[W];
                    eval(u, R, false, false, s0, f0, m0);
                    push(u, R, false, s0, f0, m0);
                }
            }
        }
        __syncwarp();
        PROF_STOP(1)
        if (lane == 0) mbar_arrive(&empty_bar[bsel]);
    }
    __syncwarp();
    if (qn) drain<W, WT>(q, qhead, qn, lane, rkeys, t, m, out_key, out_sim, out_rest, cap, counters,
                     distinct);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, o);
    if (lane == 0 && distinct) atomicAdd(counters + 0, distinct);
    PROF_FLUSH(4)
}

// --------------------------------------------- small buckets (2 <= s <= 32)
// A bucket of s <= 32 members is one warp's work as a fold: lane r holds
// member r's tag planes in registers and meets member (r + d) mod s for
// d = 1 .. s/2 through register shuffles (every pair once; at d = s/2 of an
// even s only r < d).  Buckets are grouped by size class (planning below) so
// one warp task packs q = 32 / s buckets of the same size: lanes j*s .. j*s+s-1
// hold bucket j and every lane does useful work on every step.  The main
// kernel's tiles would spend a 32-lane broadcast step per member of such a
// bucket (cfg1: 60 ms of the MATCHED pass for 7 % of its pairs).
constexpr uint32_t SMALL_MAX = 32;
constexpr int SM_WARPS = 8;  // warps per CTA of k_pairs_small
constexpr int SM_CLS = 2 + 3 * 34;  // u32 words of the class table (see k_small_prefix)

// class table (u32): cnt[34] at 0, start[34] at 34 (bucket prefix by size),
// tpre[34] at 68 (task prefix by size), cursor[34] at 102
__global__ void k_small_count(const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                              uint32_t tmax, uint64_t nb, uint32_t smin, uint32_t smax,
                              uint32_t* __restrict__ cls, const uint32_t* __restrict__ nc) {
    __shared__ uint32_t h[34];
    if (threadIdx.x < 34) h[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = bsize[i];
        if (s >= smin && s <= smax && btab[i] <= tmax && !(nc && nc[i] >= s)) atomicAdd(&h[s], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 34 && h[threadIdx.x]) atomicAdd(&cls[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_small_prefix(uint32_t* __restrict__ cls) {
    if (threadIdx.x != 0) return;
    uint32_t acc = 0, tacc = 0;
    for (uint32_t s = 0; s < 34; ++s) {
        const uint32_t c = cls[s];
        cls[34 + s] = acc;
        cls[68 + s] = tacc;
        cls[102 + s] = 0;
        acc += c;
        tacc += s >= 2 && s <= SMALL_MAX ? (c + 32 / s - 1) / (32 / s) : 0;
    }
    cls[34 + 33] = acc;  // start[33]: total small buckets (cnt[33] is always 0)
    cls[68 + 33] = tacc;
}

// descriptor per small bucket, grouped by size: bstart | table << 48
constexpr int SM_SCAT = 4;  // buckets per thread
__global__ void __launch_bounds__(256) k_small_scatter(
    const uint64_t* __restrict__ bstart, const uint32_t* __restrict__ bsize,
    const uint32_t* __restrict__ btab, uint32_t tmax, uint64_t nb, uint32_t smin, uint32_t smax,
    uint32_t* __restrict__ cls, uint64_t* __restrict__ desc, const uint32_t* __restrict__ nc) {
    __shared__ uint32_t h[34], base[34];
    if (threadIdx.x < 34) h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t i0 = (uint64_t)blockIdx.x * 256 * SM_SCAT + threadIdx.x;
    uint32_t sz[SM_SCAT], rk[SM_SCAT];
#pragma unroll
    for (int k = 0; k < SM_SCAT; ++k) {
        const uint64_t i = i0 + (uint64_t)k * 256;
        sz[k] = 0;
        if (i < nb) {
            const uint32_t s = bsize[i];
            if (s >= smin && s <= smax && btab[i] <= tmax && !(nc && nc[i] >= s)) {
                sz[k] = s;
                rk[k] = atomicAdd(&h[s], 1u);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 34 && h[threadIdx.x]) base[threadIdx.x] = atomicAdd(&cls[102 + threadIdx.x], h[threadIdx.x]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SM_SCAT; ++k) {
        if (!sz[k]) continue;
        const uint64_t i = i0 + (uint64_t)k * 256;
        const uint32_t pos = cls[34 + sz[k]] + base[sz[k]] + rk[k];
        desc[pos] = bstart[i] | ((uint64_t)btab[i] << 48);
    }
}

template <int W, int MODE, int WT>
struct SmallCfg {  // tag-plane registers per lane -> CTAs per SM (register budget)
    static constexpr int AREGS = Layout<MODE, WT>::off(W);
    static constexpr int MINB = 2;
};

// Per warp, tasks k, k + nw, ...: while task k's tag rows are loaded and
// compared, the member ids of task k + nw and the descriptors of task k + 2nw
// are already in flight, so only the row load of the dependent chain
// descriptor -> member id -> tag row is exposed per task.
template <int W, int MODE, bool HAS_E, int WT, bool EX>
__global__ void __launch_bounds__(SM_WARPS * 32, (SmallCfg<W, MODE, WT>::MINB)) k_pairs_small(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ desc,
    const uint32_t* __restrict__ cls, const uint64_t* __restrict__ rkeys,
    const uint32_t* __restrict__ tags, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
    const uint8_t* __restrict__ emask, const uint64_t* __restrict__ edges, uint32_t p,
    uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim, uint32_t* __restrict__ out_rest,
    uint64_t cap, unsigned long long* __restrict__ counters, uint32_t wg) {
    using Lay = Layout<MODE, WT>;
    constexpr int NP = TileCfg<W, MODE, WT>::NP;
    constexpr int QW = QCAP * (3 + W);
    __shared__ uint32_t s_start[34], s_tpre[34], s_q[34];
    __shared__ uint16_t s_jr[34][32];  // (bucket j << 8 | member r) of lane l in class s
    __shared__ uint32_t qsm[SM_WARPS][QW];
    if (threadIdx.x < 34) {
        s_start[threadIdx.x] = cls[34 + threadIdx.x];
        s_tpre[threadIdx.x] = cls[68 + threadIdx.x];
        s_q[threadIdx.x] = threadIdx.x >= 2 ? 32u / threadIdx.x : 0u;
    }
    for (uint32_t i = threadIdx.x; i < 34 * 32; i += blockDim.x) {
        const uint32_t sc = i >> 5, l = i & 31;
        s_jr[sc][l] = sc >= 2 ? (uint16_t)(((l / sc) << 8) | (l % sc)) : 0;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ntask = s_tpre[33];
    const uint32_t nw = gridDim.x * SM_WARPS;
    Queue q;
    q.qa = qsm[warp];
    q.qb = q.qa + QCAP;
    q.qt = q.qb + QCAP;
    q.qm = q.qt + QCAP;
    uint32_t qhead = 0, qn = 0;
    const uint32_t last_mask = (t & 31) ? ((1u << (t & 31)) - 1u) : 0xFFFFFFFFu;
    const uint32_t lt_mask = (1u << lane) - 1u;
    unsigned long long distinct = 0;

    // task k -> packed geometry s | j << 6 | r << 11 | live << 16 (size class s,
    // the lane's bucket j in the task and member r) and its descriptor slot
    auto geom = [&](uint32_t k, uint32_t& pos) -> uint32_t {
        const bool hit = k < ntask && lane >= 2 && s_tpre[lane] <= k && k < s_tpre[lane + 1];
        const uint32_t hb = __ballot_sync(0xffffffffu, hit);
        const uint32_t s = hb ? (uint32_t)(__ffs(hb) - 1) : 32u;
        const uint32_t jr = s_jr[s][lane], j = jr >> 8, r = jr & 0xFF;
        pos = k < ntask ? s_start[s] + (k - s_tpre[s]) * s_q[s] + j : 0u;
        const bool live = k < ntask && j < s_q[s] && pos < s_start[s + 1];
        return s | (j << 6) | (r << 11) | ((live ? 1u : 0u) << 16);
    };
    auto load_desc = [&](uint32_t k, uint32_t& g) -> uint64_t {
        uint32_t pos;
        g = geom(k, pos);
        return (g >> 16) ? __ldg(desc + pos) : 0ull;
    };
    auto load_id = [&](uint32_t g, uint64_t d) -> uint32_t {
        return (g >> 16) ? __ldg(sids + (d & 0xFFFFFFFFFFFFull) + ((g >> 11) & 31)) : 0u;
    };

    // the lane's tag planes of member `id` (zeros for a dead lane)
    auto load_rows = [&](uint32_t (&X)[W][NP], uint32_t id, uint32_t g) {
#pragma unroll
        for (int w = 0; w < W; ++w)
#pragma unroll
            for (int qq = 0; qq < Lay::planes(w) / 4; ++qq) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (g >> 16)
                    v = __ldg((const uint4*)(tags + ((uint64_t)(qq >> 1) * n + id) * wg * 8 + w * 8 +
                                             (qq & 1) * 4));
                X[w][qq * 4 + 0] = v.x; X[w][qq * 4 + 1] = v.y;
                X[w][qq * 4 + 2] = v.z; X[w][qq * 4 + 3] = v.w;
            }
    };

    uint32_t k = blockIdx.x * SM_WARPS + warp;
    uint32_t g0, g1, g2;
    uint64_t d0 = load_desc(k, g0), d1 = load_desc(k + nw, g1);
    uint32_t a0 = load_id(g0, d0);
    uint32_t A[W][NP];
    load_rows(A, a0, g0);
    uint32_t a1 = load_id(g1, d1);
    uint64_t d2 = load_desc(k + 2 * nw, g2);
    for (; k < ntask; k += nw) {
        const uint32_t s = g0 & 63, j = (g0 >> 6) & 31, r = (g0 >> 11) & 31;
        const bool live = (g0 >> 16) != 0;
        const uint32_t a = a0;
        // the next task's rows, ids and descriptors are in flight while this
        // task's pairs are compared
        uint32_t An[W][NP];
        load_rows(An, a1, g1);
        const uint32_t a2 = load_id(g2, d2);
        uint32_t g3;
        const uint64_t d3 = load_desc(k + 3 * nw, g3);
        QS_DASSERT(!live || a < n);
        const uint32_t table = (uint32_t)(d0 >> 48);
        const uint32_t bt = table & 31, low = (1u << bt) - 1u;
        const uint32_t tflag = (table & 0xFFu) | ((table >> 8) << 16);
        const uint32_t half = s >> 1;
        for (uint32_t dd = 1; dd <= half; ++dd) {
            uint32_t rr = r + dd;
            if (rr >= s) rr -= s;
            const uint32_t src = live ? j * s + rr : lane;
            const uint32_t bid = __shfl_sync(0xffffffffu, a, src);
            // AND over np planes of ~(A ^ B) for word w, B = the partner's planes
            auto maskw = [&](int w, int np) {
                uint32_t x = 0xFFFFFFFFu;
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) {
                    if (pp >= np) break;
                    x &= ~(A[w][pp] ^ __shfl_sync(0xffffffffu, A[w][pp], src));
                }
                return x;
            };
            const uint32_t c = min(a, bid), qv = max(a, bid);
            bool valid = live && (2 * dd != s || r < dd);
            if (EX) valid = valid && (uint64_t)(qv - c) > excl;
            if (HAS_E && valid) {
                if (emask[c]) valid = false;
                else if (emask[qv] && (p <= 1 || part_of(edges, p, qv) == part_of(edges, p, c)))
                    valid = false;
            }
            bool slow = false;
            uint32_t flags = tflag;
            uint32_t qmask[W];
            if (MODE == MODE_MATCHED) {
                uint32_t cnt = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint32_t s8 = 0;
                    if (w >= WT) {
                        s8 = maskw(w, 8);
                        if (w == (int)wg - 1) s8 &= last_mask;
                        cnt += __popc(w == WT ? (s8 & ~((low << 1) | 1u)) : s8);
                    }
                    qmask[w] = s8;
                }
                slow = valid && cnt + 1 >= m;
                flags |= QF_COUNT;
            } else {
                uint32_t early = 0, cnt = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint32_t x = 0;
                    if (w <= WT) {
                        x = maskw(w, Lay::planes(w));
                        if (w == (int)wg - 1) x &= last_mask;
                        early |= (w < WT) ? x : (x & low);
                        if (w == WT) cnt += __popc(x & ~low);
                    } else if (MODE == MODE_FULL) {
                        x = maskw(w, 8);
                        if (w == (int)wg - 1) x &= last_mask;
                        cnt += __popc(x);
                    }
                    qmask[w] = x;
                }
                const bool need_count = (MODE == MODE_FULL) && cnt >= m;
                if (valid) {
                    if (early) {
                        slow = true;
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
                if (MODE == MODE_MATCHED) {
#pragma unroll
                    for (int w = 0; w < W; ++w)
                        if (w < WT) qmask[w] = maskw(w, 8);
                }
                if (slow) {
                    const uint32_t e = (qhead + qn + __popc(bal & lt_mask)) & (QCAP - 1);
                    QS_DASSERT(e < QCAP && c < qv && qv < n);
                    q.qa[e] = c;
                    q.qb[e] = qv;
                    q.qt[e] = flags;
#pragma unroll
                    for (int w = 0; w < W; ++w) q.qm[e * W + w] = qmask[w];
                }
                qn += __popc(bal);
                if (qn >= 32) {
                    __syncwarp();
                    drain<W, WT>(q, qhead, 32, lane, rkeys, t, m, out_key, out_sim, out_rest, cap,
                             counters, distinct);
                    qhead = (qhead + 32) & (QCAP - 1);
                    qn -= 32;
                }
            }
        }
#pragma unroll
        for (int w = 0; w < W; ++w)
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) A[w][pp] = An[w][pp];
        g0 = g1; g1 = g2; g2 = g3;
        d0 = d1; d1 = d2; d2 = d3;
        a0 = a1; a1 = a2;
    }
    __syncwarp();
    if (qn) drain<W, WT>(q, qhead, qn, lane, rkeys, t, m, out_key, out_sim, out_rest, cap, counters,
                     distinct);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, o);
    if (lane == 0 && distinct) atomicAdd(counters + 0, distinct);
}

// --------------------------------------------------------------- planning
// buckets of tables > tmax are left out (MATCHED: a pair with sim >= m has its
// first collision in a table <= t - m)
// (smin, smax: a bucket-size window, a design-measurement knob; 0, ~0 = all)
__global__ void k_plan_sizes(const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                             uint32_t tmax, uint64_t nb, uint32_t L,
                             uint64_t* __restrict__ small, uint64_t* __restrict__ bigflag,
                             uint32_t smin, uint32_t smax, const uint32_t* __restrict__ nc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nb;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = (i < nb && btab[i] <= tmax) ? bsize[i] : 0;
        if (s < smin || s > smax) s = 0;
        if (nc && i < nb && nc[i] >= s) s = 0;  // wholly core: nothing left to compare
        small[i] = (i < nb && s <= L) ? s : 0;
        bigflag[i] = (i < nb && s > L) ? 1 : 0;
    }
}

// per big bucket k: its item count (scan input) and bucket index
__global__ void k_plan_big(const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                           uint32_t tmax, uint64_t nb, uint32_t L,
                           const uint64_t* __restrict__ bigpos, uint64_t* __restrict__ bigb,
                           uint64_t* __restrict__ bigcnt, unsigned long long* __restrict__ maxnseg,
                           uint32_t smin, uint32_t smax, const uint32_t* __restrict__ nc) {
    uint32_t mx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = bsize[i], ncb = nc ? nc[i] : 0u;
        if (s <= L || btab[i] > tmax || s < smin || s > smax || ncb >= s) continue;
        const uint64_t k = bigpos[i];
        bigb[k] = i;
        bigcnt[k] = big_items(s, ncb, L);
        mx = max(mx, big_groups(s, L));
    }
    // one atomic per warp (a single contended address otherwise serialises)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxnseg, (unsigned long long)mx);
}

__global__ void k_plan_bigitems(const uint32_t* __restrict__ bsize, const uint64_t* __restrict__ bigb,
                                const uint64_t* __restrict__ bigoff, const uint64_t* __restrict__ totals,
                                uint32_t L, uint64_t* __restrict__ items, uint64_t items_cap,
                                const uint32_t* __restrict__ nc) {
    const uint64_t nbig = totals[1];
    if (totals[3] > items_cap || totals[4] > 4095) return;  // decoded on the fly instead
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nbig;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = bigb[k];
        const uint32_t sb = bsize[b], ng = big_groups(sb, L), ncb = nc ? nc[b] : 0u;
        uint64_t o = bigoff[k];
        for (uint32_t g = 0; g < ng; ++g) {
            const uint32_t np = sb > 2 * L ? g_pieces(sb, ncb, g, big_bmax(L)) : 1u;
            for (uint32_t J = 0; J < np; ++J) items[o++] = (b << 24) | ((uint64_t)g << 12) | J;
        }
    }
}

// totals[2] = n_tiles; tile_first[k] = lower_bound(mpre, k * L), tile_first[n_tiles] = nb
__global__ void k_plan_tiles(const uint64_t* __restrict__ mpre, uint64_t nb, uint32_t L,
                             uint64_t* __restrict__ totals, const uint64_t* __restrict__ bigoff,
                             uint64_t* __restrict__ tile_first, uint64_t items_cap) {
    const uint64_t n_tiles = (totals[0] + L - 1) / L;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        totals[2] = n_tiles;
        totals[3] = bigoff[totals[1]];
        totals[5] = (totals[3] <= items_cap && totals[4] <= 4095) ? 1 : 0;
    }
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= n_tiles;
         k += (uint64_t)gridDim.x * blockDim.x) {
        // the last tile ends after the last small bucket (trailing big or
        // left-out buckets belong to no tile)
        const uint64_t target = k == n_tiles ? totals[0] : k * L;
        uint64_t lo = 0, hi = nb;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (mpre[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        tile_first[k] = lo;
    }
}

// ------------------------------------------------ generic path (t > 128)
__device__ __forceinline__ uint32_t gmask16(const uint32_t* __restrict__ tags, uint64_t n,
                                            uint32_t W, uint32_t a, uint32_t b, int w) {
    uint32_t x = 0xFFFFFFFFu;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const uint4* pa = (const uint4*)(tags + ((uint64_t)g * n + a) * W * 8 + w * 8);
        const uint4* pb = (const uint4*)(tags + ((uint64_t)g * n + b) * W * 8 + w * 8);
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
            const uint4 u = __ldg(pa + qq), v = __ldg(pb + qq);
            x &= ~(u.x ^ v.x) & ~(u.y ^ v.y) & ~(u.z ^ v.z) & ~(u.w ^ v.w);
        }
    }
    return x;
}

__global__ void __launch_bounds__(256) k_pairs_generic(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
    const uint64_t* __restrict__ chunk_off, uint64_t nb, const uint64_t* __restrict__ rkeys,
    const uint32_t* __restrict__ tags, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
    const uint8_t* __restrict__ emask, const uint64_t* __restrict__ edges, uint32_t p, int mode,
    uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_sim,
    uint32_t* __restrict__ out_rest, uint64_t cap, unsigned long long* __restrict__ counters) {
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
                uint32_t x = gmask16(tags, n, W, a, bid, (int)w);
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
                    out_sim[pos] = exact;  // exact: nothing left to complete
                    if (out_rest)
                        for (uint32_t w = 0; w < W; ++w) out_rest[pos * W + w] = 0;
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

// ------------------------------------------------------------------ launch
template <int W, int MODE, bool HAS_E, int WT>
static int run_pc(const uint32_t* sids, const uint64_t* bstart, const uint32_t* bsize,
                  const uint32_t* btab, uint64_t nb, const uint64_t* rkeys, const uint32_t* tags,
                  uint64_t n, uint32_t t, uint32_t m, uint64_t excl, const uint8_t* emask,
                  const uint64_t* edges, uint32_t p, uint64_t* out_key, uint32_t* out_sim,
                  uint32_t* out_rest, uint64_t cap, unsigned long long* counters, uint64_t* ws,
                  void* sws, void* smws, cudaStream_t st, uint32_t wg, const uint32_t* nc) {
    using C = TileCfg<W, MODE, WT>;
    const uint32_t L = C::L;
    uint64_t* mpre = ws;                       // nb + 1
    uint64_t* bigpos = mpre + (nb + 1);        // nb + 1
    uint64_t* bigb = bigpos + (nb + 1);        // nb + 1
    uint64_t* bigoff = bigb + (nb + 1);        // nb + 1
    uint64_t* tile_first = bigoff + (nb + 1);  // nb + 1
    uint64_t* items = tile_first + (nb + 1);   // <= 8 (nb + 1)
    uint64_t* totals = items + (nb + 1) * 8;   // 6
    unsigned long long* work = (unsigned long long*)(totals + 6);
    const uint64_t items_cap = (nb + 1) * 8;
    const unsigned g = qs_blocks(nb + 1, 256);
    const uint32_t tmax = MODE == MODE_MATCHED ? t - m : t - 1;
    const uint32_t smin_env = getenv("QS_PAIRS_SMIN") ? (uint32_t)atoi(getenv("QS_PAIRS_SMIN")) : 0u;
    const uint32_t smax = getenv("QS_PAIRS_SMAX") ? (uint32_t)atoi(getenv("QS_PAIRS_SMAX")) : ~0u;
    // buckets of <= SMALL_MAX members go to k_pairs_small (QS_SMALL=0: all to k_pairs_pc)
    static const bool small_on = !getenv("QS_SMALL") || atoi(getenv("QS_SMALL")) != 0;
    uint32_t smin = smin_env;
    if (small_on) {
        uint32_t* cls = (uint32_t*)smws;
        uint64_t* desc = (uint64_t*)((char*)smws + 1024);
        const uint32_t lo = max(2u, smin_env), hi = min(SMALL_MAX, smax);
        smin = max(smin_env, SMALL_MAX + 1);
        if (lo <= hi) {
            QS_CUDA(cudaMemsetAsync(cls, 0, SM_CLS * 4, st), "memset");
            k_small_count<<<g, 256, 0, st>>>(bsize, btab, tmax, nb, lo, hi, cls, nc);
            k_small_prefix<<<1, 32, 0, st>>>(cls);
            k_small_scatter<<<(unsigned)((nb + 256 * SM_SCAT - 1) / (256 * SM_SCAT)), 256, 0, st>>>(
                bstart, bsize, btab, tmax, nb, lo, hi, cls, desc, nc);
            auto sk = excl > 0 ? k_pairs_small<W, MODE, HAS_E, WT, true>
                               : k_pairs_small<W, MODE, HAS_E, WT, false>;
            constexpr size_t ssm = 0;
            int per_sm_s = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, sk, SM_WARPS * 32, ssm);
            if (per_sm_s < 1) per_sm_s = 1;
            sk<<<num_sms() * per_sm_s, SM_WARPS * 32, ssm, st>>>(sids, desc, cls, rkeys, tags, n, t, m,
                                                             excl, emask, edges, p, out_key, out_sim,
                                                             out_rest, cap, counters, wg);
            QS_CHECK_LAUNCH("k_pairs_small");
        }
    }
    k_plan_sizes<<<g, 256, 0, st>>>(bsize, btab, tmax, nb, L, mpre, bigpos, smin, smax, nc);
    int rc = scan_u64(mpre, mpre, nb + 1, totals + 0, sws, st);
    if (rc) return rc;
    rc = scan_u64(bigpos, bigpos, nb + 1, totals + 1, sws, st);
    if (rc) return rc;
    QS_CUDA(cudaMemsetAsync(bigoff, 0, (nb + 1) * 8, st), "memset");
    QS_CUDA(cudaMemsetAsync(totals + 4, 0, 8, st), "memset");
    k_plan_big<<<g, 256, 0, st>>>(bsize, btab, tmax, nb, L, bigpos, bigb, bigoff,
                                  (unsigned long long*)(totals + 4), smin, smax, nc);
    rc = scan_u64(bigoff, bigoff, nb + 1, nullptr, sws, st);
    if (rc) return rc;
    k_plan_tiles<<<g, 256, 0, st>>>(mpre, nb, L, totals, bigoff, tile_first, items_cap);
    k_plan_bigitems<<<g, 256, 0, st>>>(bsize, bigb, bigoff, totals, L, items, items_cap, nc);
    QS_CUDA(cudaMemsetAsync(work, 0, 8, st), "memset");
    QS_CHECK_LAUNCH("plan");
    Plan plan{mpre, tile_first, items, bigb, bigoff, totals, nc};
    auto kern = excl > 0 ? k_pairs_pc<W, MODE, HAS_E, WT, true> : k_pairs_pc<W, MODE, HAS_E, WT, false>;
    QS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM),
            "smem attr");
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PTHREADS, C::SMEM);
    if (per_sm < 1) per_sm = 1;
    kern<<<num_sms() * per_sm, PTHREADS, C::SMEM, st>>>(sids, bstart, bsize, btab, plan, rkeys, tags,
                                                        n, t, m, excl, emask, edges, p, out_key,
                                                        out_sim, out_rest, cap, counters, work,
                                                        tmax, wg);
    QS_CHECK_LAUNCH("k_pairs_pc");
    return QS_OK;
}

// first bucket of each table word (btab is non-decreasing): bounds[w] for w <= W,
// then the first buckets of tables table_lo and table_hi (bounds[W + 1], [W + 2])
__global__ void k_word_bounds(const uint32_t* __restrict__ btab, uint64_t nb, uint32_t W,
                              uint32_t table_lo, uint32_t table_hi, uint64_t* __restrict__ bounds) {
    const uint32_t w = threadIdx.x;
    if (w > W + 2) return;
    uint64_t lo = 0, hi = nb;
    const uint32_t target = w <= W ? w * 32 : (w == W + 1 ? table_lo : table_hi);
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (btab[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    bounds[w] = w == W ? nb : lo;
}

// DISTINCT / FULL: one launch per table word w over that word's buckets.
// DISTINCT stages only words 0..w (16 planes); FULL stages words 0..w with 16
// planes and the later words with 8 (count screen).
template <int W, int MODE, bool HAS_E>
static int run_word_split(const uint32_t* sids, const uint64_t* bstart, const uint32_t* bsize,
                          const uint32_t* btab, uint64_t nb, const uint64_t* rkeys,
                          const uint32_t* tags, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
                          const uint8_t* emask, const uint64_t* edges, uint32_t p, uint64_t* ok,
                          uint32_t* os, uint32_t* orest, uint64_t cap,
                          unsigned long long* counters, uint64_t* ws, void* sws, void* smws,
                          cudaStream_t st, uint32_t t_lo, uint32_t t_hi, const uint32_t* nc) {
    uint64_t* dbounds = ws + (nb + 1) * 13;  // 8 spare words after the plan arrays
    k_word_bounds<<<1, 32, 0, st>>>(btab, nb, W, t_lo, t_hi, dbounds);
    uint64_t hb[7] = {0, 0, 0, 0, 0, 0, 0};
    QS_CUDA(cudaMemcpyAsync(hb, dbounds, (W + 3) * 8, cudaMemcpyDeviceToHost, st), "copy");
    QS_CUDA(cudaStreamSynchronize(st), "sync");
    const uint64_t ta = hb[W + 1], tb = t_hi >= t ? nb : hb[W + 2];  // buckets of [t_lo, t_hi)
    for (uint32_t w = 0; w < W; ++w) {
        const uint64_t a = max(hb[w], ta), b = min(hb[w + 1], tb);
        if (b <= a) continue;
        if (MODE == MODE_MATCHED && 32 * w > t - m) continue;  // no first collision there
#define QS_W(WW, WTT)                                                                             \
    run_pc<WW, MODE, HAS_E, WTT>(sids, bstart + a, bsize + a, btab + a, b - a, rkeys, tags, n, t, \
                                 m, excl, emask, edges, p, ok, os, orest, cap, counters, ws, sws, \
                                 smws, st, W, nc ? nc + a : nullptr)
        constexpr bool DI = MODE == MODE_DISTINCT;
        int rc = QS_OK;
        if (w == 0) {
            if constexpr (DI) rc = QS_W(1, 0); else rc = QS_W(W, 0);
        } else if (w == 1) {
            if constexpr (W >= 2) { if constexpr (DI) rc = QS_W(2, 1); else rc = QS_W(W, 1); }
        } else if (w == 2) {
            if constexpr (W >= 3) { if constexpr (DI) rc = QS_W(3, 2); else rc = QS_W(W, 2); }
        } else {
            if constexpr (W >= 4) { if constexpr (DI) rc = QS_W(4, 3); else rc = QS_W(W, 3); }
        }
#undef QS_W
        if (rc) return rc;
    }
    return QS_OK;
}

template <int W>
static int dispatch_mode(int mode, bool has_e, const uint32_t* sids, const uint64_t* bstart,
                         const uint32_t* bsize, const uint32_t* btab, uint64_t nb,
                         const uint64_t* rkeys, const uint32_t* tags, uint64_t n, uint32_t t,
                         uint32_t m, uint64_t excl, const uint8_t* emask, const uint64_t* edges,
                         uint32_t p, uint64_t* ok, uint32_t* os, uint32_t* orest, uint64_t cap,
                         unsigned long long* counters, uint64_t* ws, void* sws, void* smws,
                         cudaStream_t st, uint32_t w_lo, uint32_t w_hi, const uint32_t* nc) {
#define QS_D(MM, EE) \
    run_word_split<W, MM, EE>(sids, bstart, bsize, btab, nb, rkeys, tags, n, t, m, excl, emask, \
                              edges, p, ok, os, orest, cap, counters, ws, sws, smws, st, w_lo, \
                              w_hi, nc)
    if (mode != MODE_MATCHED) orest = nullptr;  // lazy counts: MATCHED only
    if (mode == MODE_FULL) return has_e ? QS_D(MODE_FULL, true) : QS_D(MODE_FULL, false);
    if (mode == MODE_MATCHED) return has_e ? QS_D(MODE_MATCHED, true) : QS_D(MODE_MATCHED, false);
    return has_e ? QS_D(MODE_DISTINCT, true) : QS_D(MODE_DISTINCT, false);
#undef QS_D
}

// Core-first member lists (buckets of tables >= table_lo): a stable partition of
// each bucket's ids, the members flagged in `core` first, and their count.
// Buckets of earlier tables get count 0 and are not copied.  A warp takes 32
// consecutive buckets: a lane partitions its own bucket when it has <= 32
// members (nearly all of them), the warp partitions the bigger ones together.
__global__ void k_core_first(const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
                             const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                             uint64_t nb, uint32_t table_lo, const uint8_t* __restrict__ core,
                             uint32_t* __restrict__ sids_out, uint32_t* __restrict__ nc) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t b0 = gw * 32; b0 < nb; b0 += nw * 32) {
        const uint64_t b = b0 + lane;
        bool mine = false, big = false;
        uint32_t s = 0;
        uint64_t st = 0;
        if (b < nb) {
            if (btab[b] < table_lo) {
                nc[b] = 0;
            } else {
                s = bsize[b];
                st = bstart[b];
                mine = s <= 32;
                big = !mine;
            }
        }
        if (mine) {
            uint32_t cm = 0;  // core bits of the members, in order
            for (uint32_t i = 0; i < s; ++i) cm |= (core[sids[st + i]] ? 1u : 0u) << i;
            const uint32_t ncore = __popc(cm);
            uint32_t pc = 0, pn = ncore;
            for (uint32_t i = 0; i < s; ++i) {
                const uint32_t id = sids[st + i];
                if ((cm >> i) & 1u) sids_out[st + pc++] = id;
                else sids_out[st + pn++] = id;
            }
            nc[b] = ncore;
        }
        uint32_t bigm = __ballot_sync(0xffffffffu, big);
        while (bigm) {
            const uint32_t src = __ffs(bigm) - 1;
            bigm &= bigm - 1;
            const uint32_t sb = __shfl_sync(0xffffffffu, s, src);
            const uint64_t sb0 = __shfl_sync(0xffffffffu, st, src);
            uint32_t ncore = 0;
            for (uint32_t i0 = 0; i0 < sb; i0 += 32) {
                const uint32_t i = i0 + lane;
                const bool c = i < sb && core[sids[sb0 + i]];
                ncore += __popc(__ballot_sync(0xffffffffu, c));
            }
            uint32_t pc = 0, pn = ncore;
            for (uint32_t i0 = 0; i0 < sb; i0 += 32) {
                const uint32_t i = i0 + lane;
                const uint32_t id = i < sb ? sids[sb0 + i] : 0u;
                const bool c = i < sb && core[id];
                const uint32_t bc = __ballot_sync(0xffffffffu, c);
                const uint32_t bn = __ballot_sync(0xffffffffu, i < sb && !c);
                if (c) sids_out[sb0 + pc + __popc(bc & lt)] = id;
                else if (i < sb) sids_out[sb0 + pn + __popc(bn & lt)] = id;
                pc += __popc(bc);
                pn += __popc(bn);
            }
            if (lane == src) nc[b] = ncore;
        }
    }
}

// Pairs of two core members the MATCHED pass over core-first lists leaves out
// (the planning rules of k_plan_sizes / g_blo / chunks_nc and the small-bucket
// planning): a wholly core bucket entirely; in a bucket of more than L members
// every pair (i, j), i < j < nc, whose row i lies in a wholly core A group.
__global__ void k_core_skipped(const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                               const uint32_t* __restrict__ nc, uint64_t nb, uint32_t table_lo,
                               uint32_t tmax, uint32_t L, unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t tb = btab[i];
        if (tb < table_lo || tb > tmax) continue;
        const uint64_t sz = bsize[i], c = nc[i];
        if (c >= sz) acc += sz * (sz - 1) / 2;
        else if (sz > L) {
            const uint64_t f = 32 * (c / 32);
            acc += f * (f - 1) / 2 + f * (c - f);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// exact counts of lazily counted pairs: the candidate tables the drain left
// unexamined (rest, W words per pair) are confirmed on the keys now
__global__ void k_complete_sims(const uint64_t* __restrict__ pk, uint32_t* __restrict__ ps,
                                const uint32_t* __restrict__ rest, uint64_t np,
                                const uint64_t* __restrict__ rkeys, uint32_t t, uint32_t W) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t add = 0;
        const uint64_t k = pk[i];
        const uint32_t a = (uint32_t)k, b = a + (uint32_t)(k >> 32);
        for (uint32_t w = 0; w < W; ++w) {
            const uint32_t x = rest[i * W + w];
            if (x) add += confirm(rkeys, t, a, b, x, w * 32, false);
        }
        if (add) ps[i] += add;
    }
}

}  // namespace qs

using namespace qs;

extern "C" {

#ifdef QS_PROF
int qs_prof_read(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, qs::g_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(qs::g_prof, z, sizeof(z));
    }
    return 0;
}
#endif

// big-bucket items: a bucket of s > L members gives nseg(nseg+1)/2 items with
// nseg = ceil(s / L) < 2s / L, i.e. fewer than 2 s^2 / L^2 items <= 8 per
// member-bucket slot for s <= 4L; larger buckets are bounded by the member
// count (s / L items per segment row), so 8 slots per bucket bound the table.
size_t qs_lsh_pairs_ws_bytes(uint64_t n_nonsingle) {
    // + the small-bucket class table (1 KB) and descriptors (8 B per bucket)
    return (size_t)(n_nonsingle + 1) * 8 * (5 + 8) + 64 + scan_ws_bytes(n_nonsingle + 1) + 512 +
           1024 + (size_t)(n_nonsingle + 1) * 8 + 64;
}

int qs_lsh_pairs_ex(const uint32_t* sids_dev, const uint64_t* bstart_dev, const uint32_t* bsize_dev,
                    const uint32_t* btab_dev, uint64_t n_nonsingle, const uint64_t* rkeys_dev,
                    const uint32_t* tags_dev, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
                    const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p, int mode,
                    uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev,
                    uint64_t cap, unsigned long long* counters_dev, void* ws_dev, size_t ws_bytes,
                    uint32_t table_lo, uint32_t table_hi, const uint32_t* core_count_dev,
                    void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(table_lo < table_hi, "empty table range");
    QS_ARG(core_count_dev == nullptr || mode == 1, "core-first lists are for the matched pass");
    QS_ARG(ws_bytes >= qs_lsh_pairs_ws_bytes(n_nonsingle), "pairs workspace too small");
    QS_ARG(m >= 1 && m <= t, "min_matches must be in [1, tables]");
    QS_ARG(mode >= 0 && mode <= 2, "mode must be 0 (full), 1 (matched) or 2 (distinct)");
    if (n_nonsingle == 0) return QS_OK;
    const uint64_t nb = n_nonsingle;
    uint64_t* ws = (uint64_t*)ws_dev;
    void* sws = (void*)(((uintptr_t)(ws + (nb + 1) * 13 + 8) + 63) & ~(uintptr_t)63);
    void* smws = (void*)(((uintptr_t)sws + scan_ws_bytes(nb + 1) + 63) & ~(uintptr_t)63);
    const uint32_t W = (t + 31) >> 5;
    const bool has_e = excluded_dev != nullptr;
#define QS_D(WW)                                                                                  \
    dispatch_mode<WW>(mode, has_e, sids_dev, bstart_dev, bsize_dev, btab_dev, nb, rkeys_dev,      \
                      tags_dev, n, t, m, excl, excluded_dev, edges_dev, p, out_key_dev,           \
                      out_sim_dev, out_rest_dev, cap, counters_dev, ws, sws, smws, st, table_lo,  \
                      table_hi, core_count_dev)
    switch (W) {
        case 1: return QS_D(1);
        case 2: return QS_D(2);
        case 3: return QS_D(3);
        case 4: return QS_D(4);
        default: {
            QS_ARG(table_lo == 0 && table_hi >= t && core_count_dev == nullptr,
                   "table ranges and core-first lists need t <= 128");
            uint64_t* off = ws;
            k_chunk_counts<<<qs_blocks(nb + 1, 256), 256, 0, st>>>(bsize_dev, nb, off);
            int rc = scan_u64(off, off, nb + 1, nullptr, sws, st);
            if (rc) return rc;
            k_pairs_generic<<<num_sms() * 8, 256, 0, st>>>(
                sids_dev, bstart_dev, bsize_dev, btab_dev, off, nb, rkeys_dev, tags_dev, n, t, m,
                excl, excluded_dev, edges_dev, p, mode, out_key_dev, out_sim_dev,
                mode == MODE_MATCHED ? out_rest_dev : nullptr, cap, counters_dev);
            QS_CHECK_LAUNCH("k_pairs_generic");
            return QS_OK;
        }
    }
#undef QS_D
}

int qs_lsh_pairs(const uint32_t* sids_dev, const uint64_t* bstart_dev, const uint32_t* bsize_dev,
                 const uint32_t* btab_dev, uint64_t n_nonsingle, const uint64_t* rkeys_dev,
                 const uint32_t* tags_dev, uint64_t n, uint32_t t, uint32_t m, uint64_t excl,
                 const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p, int mode,
                 uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev, uint64_t cap,
                 unsigned long long* counters_dev, void* ws_dev, size_t ws_bytes, void* stream) {
    return qs_lsh_pairs_ex(sids_dev, bstart_dev, bsize_dev, btab_dev, n_nonsingle, rkeys_dev,
                           tags_dev, n, t, m, excl, excluded_dev, edges_dev, p, mode, out_key_dev,
                           out_sim_dev, out_rest_dev, cap, counters_dev, ws_dev, ws_bytes, 0,
                           0xFFFFFFFFu, nullptr, stream);
}

int qs_lsh_core_first(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                      const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t n_nonsingle,
                      uint32_t table_lo, const uint8_t* core_dev, uint32_t* sids_out_dev,
                      uint32_t* core_count_dev, void* stream) {
    if (n_nonsingle == 0) return QS_OK;
    QS_ARG(core_dev != nullptr, "core mask required");
    k_core_first<<<num_sms() * 16, 256, 0, (cudaStream_t)stream>>>(
        sids_dev, bstart_dev, bsize_dev, btab_dev, n_nonsingle, table_lo, core_dev, sids_out_dev,
        core_count_dev);
    QS_CHECK_LAUNCH("k_core_first");
    return QS_OK;
}

int qs_lsh_core_skipped(const uint32_t* bsize_dev, const uint32_t* btab_dev,
                        const uint32_t* core_count_dev, uint64_t n_nonsingle, uint32_t t,
                        uint32_t m, uint32_t table_lo, unsigned long long* out_dev, void* stream) {
    if (n_nonsingle == 0) return QS_OK;
    QS_ARG(t >= 1 && t <= 128 && m >= 1 && m <= t, "bad t / m");
    const uint32_t W = (t + 31) >> 5;
    const uint32_t L = W == 1 ? TileCfg<1, MODE_MATCHED, 0>::L
                     : W == 2 ? TileCfg<2, MODE_MATCHED, 0>::L
                     : W == 3 ? TileCfg<3, MODE_MATCHED, 0>::L : TileCfg<4, MODE_MATCHED, 0>::L;
    k_core_skipped<<<qs_blocks(n_nonsingle, 256), 256, 0, (cudaStream_t)stream>>>(
        bsize_dev, btab_dev, core_count_dev, n_nonsingle, table_lo, t - m, L, out_dev);
    QS_CHECK_LAUNCH("k_core_skipped");
    return QS_OK;
}

int qs_lsh_complete_sims(const uint64_t* pair_key_dev, uint32_t* pair_sim_dev,
                         const uint32_t* rest_dev, uint64_t n_pairs, const uint64_t* rkeys_dev,
                         uint32_t t, void* stream) {
    if (n_pairs == 0) return QS_OK;
    QS_ARG(t >= 1, "t must be >= 1");
    k_complete_sims<<<qs_blocks(n_pairs, 256), 256, 0, (cudaStream_t)stream>>>(
        pair_key_dev, pair_sim_dev, rest_dev, n_pairs, rkeys_dev, t, (t + 31) >> 5);
    QS_CHECK_LAUNCH("k_complete_sims");
    return QS_OK;
}

}  // extern "C"
