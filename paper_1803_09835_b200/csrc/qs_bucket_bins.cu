// Bucket construction in two data passes: partition by key range, then sort
// each range in shared memory (lsh_search.py:157-172: per table, the member
// ids grouped by equal signature word, ids ascending inside a bucket — the
// stable argsort the reference runs per table).
//
//   pass 1  k_bb_hist + scan + k_bb_scatter: per table, a STABLE scatter of
//           (key, id) into 2^D bins by the key's top D bits (keys are
//           fmix64-mixed, so bins are even: ~2k members at D = ceil(log2(n /
//           2048))), reading the keys straight from the signature kernel's
//           (t, n) layout, ids implicit (= position);
//   pass 2  k_bb_bins: one CTA per bin sorts it in shared memory by the next
//           32 - D key bits (stable LSD, 7-bit digits) and writes the member
//           ids and the head/tail flag byte of every member (the listing's
//           input) — bins are whole buckets, so no work crosses a bin edge.
//           Bins whose 32-bit prefixes collide on different keys (~170 per
//           table at cfg1) re-sort on the full key; bins above the CTA's
//           capacity go to a larger-CTA kernel, the rare giant ones (one bucket
//           of > 16k members) to a single-CTA global-memory path.
//
// Bytes per (member, table): pass 1 reads 8 (histogram) + 8 and writes 12,
// pass 2 reads 12 and writes 5 — 45 B against the 143 B of the round-1
// LSD radix build (4 x (histogram + scatter) + fix-up + flag sweep).
#include <algorithm>

#include "qs_lsh.cuh"

namespace qs {

constexpr int BB_T1 = 256;                     // pass-1 threads
constexpr int BB_ITEMS = 16;                   // keys per thread per sub-tile
constexpr int BB_SUB = BB_T1 * BB_ITEMS;       // 4096-key sub-tiles
constexpr int BB_W1 = BB_T1 / 32;
constexpr uint32_t BB_DMAX = 12;               // <= 4096 bins per table
constexpr int BB_MAXTILES = 64;                // tiles per table (histogram size)
constexpr int BB_RBITS = 7, BB_RADIX = 1 << BB_RBITS;

__global__ void k_rs_scan(uint32_t* hist, uint64_t len);  // qs_sort.cu

struct BinGeo {
    uint32_t D, B, tiles;
    uint64_t tile;
};

static BinGeo bin_geo(uint64_t n) {
    BinGeo g;
    g.D = 0;
    while (g.D < BB_DMAX && (n >> g.D) > 2048) ++g.D;
    g.B = 1u << g.D;
    uint64_t tiles = std::min<uint64_t>(BB_MAXTILES, (n + BB_SUB - 1) / BB_SUB);
    if (tiles < 1) tiles = 1;
    g.tile = ((n + tiles - 1) / tiles + BB_SUB - 1) / BB_SUB * BB_SUB;
    g.tiles = (uint32_t)((n + g.tile - 1) / g.tile);
    return g;
}

__device__ __forceinline__ uint32_t bb_bin(uint64_t key, uint32_t D) {
    return D ? (uint32_t)(key >> (64 - D)) : 0u;
}

// ------------------------------------------------------------------ pass 1
// grid (tiles, t): per-(table, bin, tile) member counts, bin-major
__global__ void __launch_bounds__(BB_T1) k_bb_hist(const uint64_t* __restrict__ keys, uint64_t n,
                                                   uint32_t D, uint64_t tile_len, uint32_t tiles,
                                                   uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t bh[];
    const uint32_t B = 1u << D, tile = blockIdx.x, table = blockIdx.y;
    for (uint32_t i = threadIdx.x; i < B; i += BB_T1) bh[i] = 0;
    __syncthreads();
    const uint64_t* k = keys + (uint64_t)table * n;
    const uint64_t lo = (uint64_t)tile * tile_len, hi = min(n, lo + tile_len);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += BB_T1) atomicAdd(&bh[bb_bin(__ldcs(k + i), D)], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < B; b += BB_T1)
        counts[((uint64_t)table * B + b) * tiles + tile] = bh[b];
}

// grid (tiles, t): stable scatter of the tile's (key, position) pairs to the
// scanned (bin, tile) offsets; the tile is walked in 4096-key sub-tiles, each
// ranked per bin in input order (warp match_any + per-warp counters + a
// prefix over the earlier warps)
__global__ void __launch_bounds__(BB_T1, 2) k_bb_scatter(const uint64_t* __restrict__ keys, uint64_t n,
                                                         uint32_t D, uint64_t tile_len, uint32_t tiles,
                                                         const uint32_t* __restrict__ offs,
                                                         uint64_t* __restrict__ okeys,
                                                         uint32_t* __restrict__ oids) {
    extern __shared__ __align__(16) uint32_t bsm[];
    const uint32_t B = 1u << D, tile = blockIdx.x, table = blockIdx.y;
    uint32_t* goff = bsm;                                  // [B] running output offsets
    uint16_t* wcnt = (uint16_t*)(bsm + B);                 // [BB_W1][B] per-warp counts
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t b = threadIdx.x; b < B; b += BB_T1) {
        goff[b] = offs[((uint64_t)table * B + b) * tiles + tile];
#pragma unroll
        for (int w = 0; w < BB_W1; ++w) wcnt[w * B + b] = 0;
    }
    __syncthreads();
    const uint64_t* k = keys + (uint64_t)table * n;
    uint64_t* ok_out = okeys + (uint64_t)table * n;
    uint32_t* oi_out = oids + (uint64_t)table * n;
    const uint64_t lo = (uint64_t)tile * tile_len, hi = min(n, lo + tile_len);
    for (uint64_t sub = lo; sub < hi; sub += BB_SUB) {
        const uint64_t t0 = sub + (uint64_t)warp * (32 * BB_ITEMS);
        uint64_t kv[BB_ITEMS];
        uint32_t rank[BB_ITEMS];
#pragma unroll
        for (int r = 0; r < BB_ITEMS; ++r) {
            const uint64_t i = t0 + (uint64_t)r * 32 + lane;
            kv[r] = i < hi ? __ldcs(k + i) : 0;
        }
#pragma unroll
        for (int r = 0; r < BB_ITEMS; ++r) {
            const uint64_t i = t0 + (uint64_t)r * 32 + lane;
            const bool ok = i < hi;
            const uint32_t d = ok ? bb_bin(kv[r], D) : B;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t before = __popc(peers & lt);
            uint32_t c = 0;
            if (ok) c = wcnt[warp * B + d];
            rank[r] = c + before;
            __syncwarp();
            if (ok && before == 0) wcnt[warp * B + d] = (uint16_t)(c + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        uint32_t last = 0;  // bit r: this key is its warp's last of its bin
#pragma unroll
        for (int r = 0; r < BB_ITEMS; ++r) {
            const uint64_t i = t0 + (uint64_t)r * 32 + lane;
            if (i < hi) {
                const uint32_t d = bb_bin(kv[r], D);
                uint32_t base = goff[d];
                for (uint32_t w = 0; w < warp; ++w) base += wcnt[w * B + d];
                const uint32_t pos = base + rank[r];
                ok_out[pos] = kv[r];
                oi_out[pos] = (uint32_t)i;
                if (rank[r] + 1 == wcnt[warp * B + d]) last |= 1u << r;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < BB_ITEMS; ++r) {
            const uint64_t i = t0 + (uint64_t)r * 32 + lane;
            if (i < hi && ((last >> r) & 1u)) {
                const uint32_t d = bb_bin(kv[r], D);
                atomicAdd(&goff[d], rank[r] + 1);
                wcnt[warp * B + d] = 0;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ pass 2
// Stable LSD sort of E (digit source, index) pairs by `bits` bits starting at
// bit `lo` of the 32-bit values, with the block's warps each ranking one
// contiguous range (stable: range order = input order).  Arrays are shared or
// global memory; cnt is [nwarps][BB_RADIX] shared counters.
template <class IDX>
__device__ void bb_block_sort(uint32_t* va, IDX* ia, uint32_t* vb, IDX* ib, uint32_t E,
                              uint32_t lo, uint32_t bits, uint32_t* cnt, uint32_t*& vout,
                              IDX*& iout) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t C = ((E + W - 1) / W + 31) & ~31u;  // per-warp contiguous range
    const uint32_t r0 = min(E, warp * C), r1 = min(E, r0 + C);
    uint32_t *sv = va, *dv = vb;
    IDX *si = ia, *di = ib;
    for (uint32_t sh = lo; sh < lo + bits; sh += BB_RBITS) {
        const uint32_t nb = min((uint32_t)BB_RBITS, lo + bits - sh);
        const uint32_t mask = (1u << nb) - 1u;
        for (uint32_t i = threadIdx.x; i < W * BB_RADIX; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        for (uint32_t j0 = r0; j0 < r1; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool ok = j < r1;
            const uint32_t d = ok ? (sv[j] >> sh) & mask : BB_RADIX;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (ok && (peers & lt) == 0) cnt[warp * BB_RADIX + d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // exclusive prefix over (digit, warp): digits in order, warps in order
        if (threadIdx.x < BB_RADIX) {
            const uint32_t d = threadIdx.x;
            uint32_t tot = 0;
            for (uint32_t w = 0; w < W; ++w) tot += cnt[w * BB_RADIX + d];
            // block scan of the digit totals by warps 0..3
            uint32_t x = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            cnt[W * BB_RADIX + d] = x;  // inclusive within the warp (scratch row W)
        }
        __syncthreads();
        if (threadIdx.x < BB_RADIX) {
            const uint32_t d = threadIdx.x;
            uint32_t run = cnt[W * BB_RADIX + d];
            for (uint32_t q = 0; q < (d >> 5); ++q) run += cnt[W * BB_RADIX + q * 32 + 31];
            uint32_t tot = 0;
            for (uint32_t w = 0; w < W; ++w) tot += cnt[w * BB_RADIX + d];
            run -= tot;  // exclusive
            for (uint32_t w = 0; w < W; ++w) {
                const uint32_t c = cnt[w * BB_RADIX + d];
                cnt[w * BB_RADIX + d] = run;
                run += c;
            }
        }
        __syncthreads();
        for (uint32_t j0 = r0; j0 < r1; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool ok = j < r1;
            const uint32_t v = ok ? sv[j] : 0u;
            const uint32_t d = ok ? (v >> sh) & mask : BB_RADIX;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            uint32_t b = 0;
            if (ok) b = cnt[warp * BB_RADIX + d];
            __syncwarp();
            if (ok) {
                const uint32_t p = b + __popc(peers & lt);
                dv[p] = v;
                di[p] = si[j];
                if ((peers & lt) == 0) cnt[warp * BB_RADIX + d] = b + __popc(peers);
            }
            __syncwarp();
        }
        __syncthreads();
        uint32_t* tv = sv; sv = dv; dv = tv;
        IDX* ti = si; si = di; di = ti;
    }
    vout = sv;
    iout = si;
}

// Sort one bin [bstart, bstart + E) of a table and write ids + flags.  vals /
// idx: two buffers each of >= E entries (shared memory, or global scratch for
// the giant-bin path).
template <class IDX>
__device__ void bb_sort_bin(const uint64_t* __restrict__ okeys, const uint32_t* __restrict__ oids,
                            uint64_t bstart, uint32_t E, uint32_t D, uint32_t* va, uint32_t* vb,
                            IDX* ia, IDX* ib, uint64_t* kbuf, uint32_t* cnt,
                            uint32_t* __restrict__ sids, uint8_t* __restrict__ flags,
                            bool full_key) {
    const uint32_t pbits = 32 - D;  // prefix bits below the bin bits
    uint32_t* vs;
    IDX* is;
    if (!full_key) {
        for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) {
            va[j] = (uint32_t)(okeys[bstart + j] >> 32);
            ia[j] = (IDX)j;
        }
        __syncthreads();
        bb_block_sort<IDX>(va, ia, vb, ib, E, 0, pbits, cnt, vs, is);
    } else {
        // full 64-bit order: low 32 bits first, then the prefix (LSD)
        for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) {
            va[j] = (uint32_t)okeys[bstart + j];
            ia[j] = (IDX)j;
        }
        __syncthreads();
        bb_block_sort<IDX>(va, ia, vb, ib, E, 0, 32, cnt, vs, is);
        uint32_t* vo = vs == va ? vb : va;
        IDX* io = is == ia ? ib : ia;
        for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) {
            vo[j] = (uint32_t)(okeys[bstart + is[j]] >> 32);
            io[j] = is[j];
        }
        __syncthreads();
        bb_block_sort<IDX>(vo, io, vs, is, E, 0, pbits, cnt, vs, is);
    }
    // sorted keys + ids; flags from neighbouring full keys
    for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) {
        const uint32_t li = (uint32_t)is[j];
        kbuf[j] = okeys[bstart + li];
        sids[bstart + j] = oids[bstart + li];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) {
        const uint64_t key = kbuf[j];
        const bool head = j == 0 || kbuf[j - 1] != key;
        const bool tail = j + 1 == E || kbuf[j + 1] != key;
        flags[bstart + j] = (uint8_t)((head ? 1 : 0) | (tail ? 2 : 0));
    }
}

// true when two different keys share a 32-bit prefix somewhere in the sorted
// bin (then only the full-key sort gives the stable argsort order)
__device__ bool bb_prefix_collision(const uint64_t* kbuf, uint32_t E, uint32_t* flag) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (uint32_t j = 1 + threadIdx.x; j < E; j += blockDim.x)
        if ((kbuf[j] >> 32) == (kbuf[j - 1] >> 32) && kbuf[j] != kbuf[j - 1]) *flag = 1;
    __syncthreads();
    const bool r = *flag != 0;
    __syncthreads();
    return r;
}

constexpr uint32_t BB_CAP_S = 4096, BB_CAP_M = 16384;

__device__ __forceinline__ void bb_bin_bounds(const uint32_t* __restrict__ offs, uint64_t n,
                                              uint32_t B, uint32_t tiles, uint32_t table,
                                              uint32_t bin, uint64_t& s0, uint32_t& E) {
    s0 = offs[((uint64_t)table * B + bin) * tiles];
    const uint64_t s1 = bin + 1 < B ? offs[((uint64_t)table * B + bin + 1) * tiles] : n;
    E = (uint32_t)(s1 - s0);
}

template <uint32_t CAP>
__device__ void bb_one_bin(const uint64_t* __restrict__ okeys, const uint32_t* __restrict__ oids,
                           uint64_t bstart, uint32_t E, uint32_t D, unsigned char* bbs,
                           uint32_t* __restrict__ sids, uint8_t* __restrict__ flags) {
    uint64_t* kbuf = (uint64_t*)bbs;                      // [CAP] (aliases va/vb)
    uint32_t* va = (uint32_t*)bbs;                        // [CAP]
    uint32_t* vb = va + CAP;                              // [CAP]
    uint16_t* ia = (uint16_t*)(vb + CAP);                 // [CAP]
    uint16_t* ib = ia + CAP;                              // [CAP]
    uint32_t* cnt = (uint32_t*)(ib + CAP);                // [W + 1][RADIX] + flag
    if (E == 1) {
        if (threadIdx.x == 0) {
            sids[bstart] = oids[bstart];
            flags[bstart] = 3;
        }
        return;
    }
    bb_sort_bin<uint16_t>(okeys, oids, bstart, E, D, va, vb, ia, ib, kbuf, cnt, sids, flags, false);
    __syncthreads();
    if (bb_prefix_collision(kbuf, E, cnt + (blockDim.x / 32 + 1) * BB_RADIX))
        bb_sort_bin<uint16_t>(okeys, oids, bstart, E, D, va, vb, ia, ib, kbuf, cnt, sids, flags,
                              true);
    __syncthreads();
}

// one CTA per (bin, table) with E <= BB_CAP_S in shared memory; bigger bins
// are appended to the mid list [0, list_cap) or the giant list [list_cap, 2 list_cap)
__global__ void __launch_bounds__(256) k_bb_bins(const uint64_t* __restrict__ okeys,
                                                 const uint32_t* __restrict__ oids, uint64_t n,
                                                 uint32_t D, uint32_t tiles,
                                                 const uint32_t* __restrict__ offs,
                                                 uint32_t* __restrict__ sids,
                                                 uint8_t* __restrict__ flags,
                                                 uint64_t* __restrict__ lists,
                                                 unsigned long long* __restrict__ list_n,
                                                 uint64_t list_cap) {
    extern __shared__ __align__(16) unsigned char bbs[];
    const uint32_t B = 1u << D, bin = blockIdx.x, table = blockIdx.y;
    uint64_t s0;
    uint32_t E;
    bb_bin_bounds(offs, n, B, tiles, table, bin, s0, E);
    if (E == 0) return;
    if (E > BB_CAP_S) {
        if (threadIdx.x == 0) {
            const bool giant = E > BB_CAP_M;
            const unsigned long long k = atomicAdd(list_n + (giant ? 1 : 0), 1ull);
            if (k < list_cap) lists[(giant ? list_cap : 0) + k] = ((uint64_t)table << 32) | bin;
        }
        return;
    }
    bb_one_bin<BB_CAP_S>(okeys, oids, (uint64_t)table * n + s0, E, D, bbs, sids, flags);
}

// mid bins (BB_CAP_S < E <= BB_CAP_M): persistent CTAs over the list
__global__ void __launch_bounds__(1024) k_bb_mid(const uint64_t* __restrict__ okeys,
                                                 const uint32_t* __restrict__ oids, uint64_t n,
                                                 uint32_t D, uint32_t tiles,
                                                 const uint32_t* __restrict__ offs,
                                                 uint32_t* __restrict__ sids,
                                                 uint8_t* __restrict__ flags,
                                                 const uint64_t* __restrict__ lists,
                                                 unsigned long long* __restrict__ list_n,
                                                 uint64_t list_cap) {
    extern __shared__ __align__(16) unsigned char bbs[];
    __shared__ unsigned long long item;
    const uint32_t B = 1u << D;
    const uint64_t nl = min((unsigned long long)list_cap, list_n[0]);
    while (true) {
        if (threadIdx.x == 0) item = atomicAdd(list_n + 2, 1ull);
        __syncthreads();
        const uint64_t it = item;
        __syncthreads();
        if (it >= nl) break;
        const uint64_t e = lists[it];
        const uint32_t table = (uint32_t)(e >> 32), bin = (uint32_t)e;
        uint64_t s0;
        uint32_t E;
        bb_bin_bounds(offs, n, B, tiles, table, bin, s0, E);
        bb_one_bin<BB_CAP_M>(okeys, oids, (uint64_t)table * n + s0, E, D, bbs, sids, flags);
    }
}

// giant bins (> BB_CAP_M members): one CTA at a time, sorting in global scratch
__global__ void __launch_bounds__(1024) k_bb_giant(const uint64_t* __restrict__ okeys,
                                                   const uint32_t* __restrict__ oids, uint64_t n,
                                                   uint32_t D, uint32_t tiles,
                                                   const uint32_t* __restrict__ offs,
                                                   uint32_t* __restrict__ sids,
                                                   uint8_t* __restrict__ flags,
                                                   const uint64_t* __restrict__ lists,
                                                   const unsigned long long* __restrict__ list_n,
                                                   uint64_t list_cap, uint32_t* __restrict__ scratch) {
    __shared__ uint32_t cnt[(1024 / 32 + 1) * BB_RADIX + 4];
    const uint32_t B = 1u << D;
    const uint64_t ng = min((unsigned long long)list_cap, list_n[1]);
    for (uint64_t g = 0; g < ng; ++g) {
        const uint64_t e = lists[list_cap + g];
        const uint32_t table = (uint32_t)(e >> 32), bin = (uint32_t)e;
        uint64_t s0;
        uint32_t E;
        bb_bin_bounds(offs, n, B, tiles, table, bin, s0, E);
        const uint64_t bstart = (uint64_t)table * n + s0;
        uint32_t* va = scratch;
        uint32_t* vb = va + n;
        uint32_t* ia = vb + n;
        uint32_t* ib = ia + n;
        uint64_t* kbuf = (uint64_t*)(ib + n + (n & 1));
        // the full-key sort directly (giant bins are rare)
        bb_sort_bin<uint32_t>(okeys, oids, bstart, E, D, va, vb, ia, ib, kbuf, cnt, sids, flags,
                              true);
        __syncthreads();
    }
}

}  // namespace qs

using namespace qs;

namespace {

size_t bb_ws_layout(uint64_t n, uint32_t t, size_t* off_counts, size_t* off_okeys,
                    size_t* off_oids, size_t* off_lists, size_t* off_scratch, uint64_t* list_cap) {
    const BinGeo g = bin_geo(n);
    const uint64_t total = n * t;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = (o + 255) & ~(size_t)255;
        o = at + bytes;
        return at;
    };
    *list_cap = (uint64_t)g.B * t;
    *off_counts = take((size_t)t * g.B * g.tiles * 4);
    *off_okeys = take((size_t)total * 8);
    *off_oids = take((size_t)total * 4);
    *off_lists = take((size_t)(2 * *list_cap + 4) * 8);
    *off_scratch = take((size_t)n * 24 + 64);
    return o + 256;
}

}  // namespace

namespace qs {

size_t bucket_bins_ws_bytes(uint64_t n, uint32_t t) {
    size_t a, b, c, d, e;
    uint64_t lc;
    return bb_ws_layout(n, t, &a, &b, &c, &d, &e, &lc);
}

int bucket_bins_build(const uint64_t* keys, uint64_t n, uint32_t t, uint32_t* sids, uint8_t* flags,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n == 0 || t == 0) return QS_OK;
    QS_ARG(n < (1ull << 32), "more than 2**32 fingerprints are not supported");
    size_t oc, ok, oi, ol, os;
    uint64_t list_cap;
    const size_t need = bb_ws_layout(n, t, &oc, &ok, &oi, &ol, &os, &list_cap);
    QS_ARG(ws_bytes >= need, "bucket workspace too small");
    unsigned char* w = (unsigned char*)ws;
    uint32_t* counts = (uint32_t*)(w + oc);
    uint64_t* okeys = (uint64_t*)(w + ok);
    uint32_t* oids = (uint32_t*)(w + oi);
    unsigned long long* list_n = (unsigned long long*)(w + ol);
    uint64_t* lists = (uint64_t*)(list_n + 4);  // [0] mid count, [1] giant count, [2] mid cursor
    uint32_t* scratch = (uint32_t*)(w + os);
    const BinGeo g = bin_geo(n);
    const size_t hsm = (size_t)g.B * 4;
    const size_t ssm = (size_t)g.B * 4 + (size_t)BB_W1 * g.B * 2;
    QS_CUDA(cudaFuncSetAttribute(k_bb_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm),
            "smem attr");
    QS_CUDA(cudaFuncSetAttribute(k_bb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm),
            "smem attr");
    dim3 grid1(g.tiles, t);
    k_bb_hist<<<grid1, BB_T1, hsm, st>>>(keys, n, g.D, g.tile, g.tiles, counts);
    // per-table exclusive scan over (bin, tile)
    const uint64_t seg = (uint64_t)g.B * g.tiles;
    k_rs_scan<<<t, 1024, 0, st>>>(counts, seg);
    k_bb_scatter<<<grid1, BB_T1, ssm, st>>>(keys, n, g.D, g.tile, g.tiles, counts, okeys, oids);
    QS_CHECK_LAUNCH("bucket bins pass 1");
    QS_CUDA(cudaMemsetAsync(list_n, 0, 32, st), "memset");
    const int wS = 256, wM = 1024;
    const size_t smS = (size_t)BB_CAP_S * 12 + (size_t)(wS / 32 + 1) * BB_RADIX * 4 + 16;
    const size_t smM = (size_t)BB_CAP_M * 12 + (size_t)(wM / 32 + 1) * BB_RADIX * 4 + 16;
    QS_CUDA(cudaFuncSetAttribute(k_bb_bins, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smS),
            "smem attr");
    QS_CUDA(cudaFuncSetAttribute(k_bb_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smM),
            "smem attr");
    k_bb_bins<<<dim3(g.B, t), wS, smS, st>>>(okeys, oids, n, g.D, g.tiles, counts, sids, flags,
                                             lists, list_n, list_cap);
    k_bb_mid<<<num_sms(), wM, smM, st>>>(okeys, oids, n, g.D, g.tiles, counts, sids, flags, lists,
                                         list_n, list_cap);
    k_bb_giant<<<1, 1024, 0, st>>>(okeys, oids, n, g.D, g.tiles, counts, sids, flags, lists, list_n,
                                   list_cap, scratch);
    QS_CHECK_LAUNCH("bucket bins pass 2");
    return QS_OK;
}

}  // namespace qs
