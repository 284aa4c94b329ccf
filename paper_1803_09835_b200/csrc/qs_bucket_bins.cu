// Bucket construction: two 8-bit radix passes, then shared-memory sorts of
// whole key ranges (lsh_search.py:157-172: per table, the member ids grouped
// by equal signature word, ids ascending inside a bucket — the stable argsort
// the reference runs per table).
//
//   pass 1  two stable LSD radix passes (qs_sort.cu: histogram, scan,
//           coalesced tile scatter) on key bits 48-63, ids implicit (=
//           position), straight from the signature kernel's (t, n) keys: each
//           table is now ordered by its top 16 key bits (keys are fmix64-mixed,
//           so these 65536 ranges hold ~n/65536 members each);
//   pass 2  k_bb_ranges: one CTA per ~2048-member stretch, its ends moved to
//           the next top-16 boundary (whole buckets, no work crosses a CTA
//           edge), sorts the stretch in shared memory by the 32-bit key
//           prefix (stable LSD, 7-bit digits), and writes the member ids and
//           the head/tail flag byte of every member (the listing's input).
//           Stretches whose 32-bit prefixes collide on different keys re-sort
//           on the full key; longer stretches (a bucket of thousands of members)
//           go to a 1024-thread kernel, the rare giant ones (> 16384) to a
//           single-CTA global-memory path.
//
// Bytes per (member, table): pass 1 moves 2 x (8 histogram + 12 + 12) = 64,
// pass 2 reads 12 and writes 5 — 81 B against the 143 B of the round-1
// build (4 radix passes + fix-up sweeps + flag sweep).
//
// Measured and rejected (this round): a single stable scatter into 4096
// key-range bins per table (k_bb_scatter) — ~2 keys per (bin, 4096-key tile)
// means scattered 8-byte writes, and the partial-sector writes cost 38.6 GB of
// DRAM reads + 41 GB of writes per step (48 ms), against 5.9 ms per coalesced
// 8-bit pass.
#include <stdlib.h>

#include <algorithm>

#include "qs_lsh.cuh"

namespace qs {

constexpr int BB_RBITS = 7, BB_RADIX = 1 << BB_RBITS;
#ifndef QS_BB_R
#define QS_BB_R 2048
#define QS_BB_CAP 4096
#endif
constexpr uint32_t BB_R = QS_BB_R;                   // nominal members per pass-2 CTA
constexpr uint32_t BB_CAP_S = QS_BB_CAP, BB_CAP_M = 16384;
constexpr uint32_t BB_TOP = 16;                      // key bits ordered by pass 1

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


__device__ __forceinline__ uint32_t bb_top(uint64_t k) { return (uint32_t)(k >> (64 - BB_TOP)); }

// first position >= p (p <= n) where a new top-16 range begins (or n)
__device__ uint64_t bb_next_boundary(const uint64_t* __restrict__ k, uint64_t n, uint64_t p) {
    const uint32_t lane = threadIdx.x & 31;
    if (p == 0 || p >= n) return p >= n ? n : 0;
    uint32_t prev = bb_top(k[p - 1]);
    for (uint64_t q = p; q < n; q += 32) {
        const uint64_t i = q + lane;
        const bool bnd = i < n && bb_top(k[i]) != (i == q ? prev : bb_top(k[i - 1]));
        const uint32_t bal = __ballot_sync(0xffffffffu, bnd);
        if (bal) return q + __ffs(bal) - 1;
        prev = __shfl_sync(0xffffffffu, i < n ? bb_top(k[i]) : 0u, 31);
    }
    return n;
}

template <uint32_t CAP>
__device__ void bb_one_range(const uint64_t* __restrict__ okeys, const uint32_t* __restrict__ oids,
                             uint64_t bstart, uint32_t E, unsigned char* bbs,
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
    bb_sort_bin<uint16_t>(okeys, oids, bstart, E, 0, va, vb, ia, ib, kbuf, cnt, sids, flags, false);
    __syncthreads();
    if (bb_prefix_collision(kbuf, E, cnt + (blockDim.x / 32 + 1) * BB_RADIX))
        bb_sort_bin<uint16_t>(okeys, oids, bstart, E, 0, va, vb, ia, ib, kbuf, cnt, sids, flags,
                              true);
    __syncthreads();
}


// ------------------------------------------------- pass 2, one warp per bin
// The CTA stages its stretch (<= BB_CAP_S members) in shared memory as 16-bit
// sort keys (key bits 32-47: the top 16 are equal inside a top-16 bin) and
// local indices, finds the bin starts, and its warps take whole bins: two
// stable 8-bit LSD passes per bin with warp-private counters (no block
// barriers), then ids + head/tail flags written in order.  A bin whose sorted
// neighbours share the 32-bit prefix but not the key goes to the mid list
// (full-key sort there).
constexpr int BW_T = 256, BW_W = BW_T / 32;

__device__ __forceinline__ void bw_pass(const uint16_t* __restrict__ sk, const uint16_t* __restrict__ si,
                                        uint16_t* __restrict__ dk, uint16_t* __restrict__ di,
                                        uint32_t b0, uint32_t sz, uint32_t sh, uint16_t* cnt) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < 8; ++q) cnt[lane * 8 + q] = 0;
    __syncwarp();
    for (uint32_t j0 = 0; j0 < sz; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool ok = j < sz;
        const uint32_t d = ok ? (sk[b0 + j] >> sh) & 0xFFu : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (ok && (peers & lt) == 0) cnt[d] = (uint16_t)(cnt[d] + __popc(peers));
        __syncwarp();
    }
    // exclusive prefix of the 256 counters: 8 consecutive per lane
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        v[q] = cnt[lane * 8 + q];
        sum += v[q];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    uint32_t run = x - sum;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        cnt[lane * 8 + q] = (uint16_t)run;
        run += v[q];
    }
    __syncwarp();
    for (uint32_t j0 = 0; j0 < sz; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool ok = j < sz;
        const uint32_t kv = ok ? sk[b0 + j] : 0u;
        const uint32_t d = ok ? (kv >> sh) & 0xFFu : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t b = 0;
        if (ok) b = cnt[d];
        __syncwarp();
        if (ok) {
            const uint32_t r = b + __popc(peers & lt);
            dk[b0 + r] = (uint16_t)kv;
            di[b0 + r] = si[b0 + j];
            if ((peers & lt) == 0) cnt[d] = (uint16_t)(b + __popc(peers));
        }
        __syncwarp();
    }
}

constexpr uint32_t BW_CAP = 3072;  // stretch capacity of the warp-per-bin kernel

__global__ void __launch_bounds__(BW_T) k_bb_warpbins(const uint64_t* __restrict__ okeys,
                                                      const uint32_t* __restrict__ oids, uint64_t n,
                                                      uint32_t* __restrict__ sids,
                                                      uint8_t* __restrict__ flags,
                                                      uint64_t* __restrict__ lists,
                                                      unsigned long long* __restrict__ list_n,
                                                      uint64_t list_cap) {
    // sort keys (key bits 32-47), local indices, and the payload staged once:
    // member ids and the low key halves (flags and the prefix-collision test
    // rebuild full keys from shared memory, no global gathers)
    extern __shared__ __align__(16) unsigned char bws[];
    uint32_t* sid = (uint32_t*)bws;                       // [BW_CAP]
    uint32_t* slo = sid + BW_CAP;                         // [BW_CAP]
    uint16_t* ka = (uint16_t*)(slo + BW_CAP);             // [BW_CAP] x 5
    uint16_t* kb = ka + BW_CAP;
    uint16_t* ia = kb + BW_CAP;
    uint16_t* ib = ia + BW_CAP;
    uint16_t* binst = ib + BW_CAP;
    uint16_t (*cnt)[256] = (uint16_t (*)[256])(binst + BW_CAP);
    __shared__ uint32_t wtot[BW_W];
    __shared__ uint64_t se[2];
    __shared__ uint32_t next_bin;
    const uint32_t table = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t* k = okeys + (uint64_t)table * n;
    if (warp < 2) {
        const uint64_t p = min(n, ((uint64_t)blockIdx.x + warp) * BB_R);
        const uint64_t b = bb_next_boundary(k, n, p);
        if (lane == 0) se[warp] = b;
    }
    if (threadIdx.x == 0) next_bin = 0;
    __syncthreads();
    const uint64_t s = se[0], e = se[1];
    if (s >= e) return;
    const uint64_t E = e - s;
    if (E > BW_CAP) {
        if (threadIdx.x == 0) {
            const bool giant = E > BB_CAP_M;
            const unsigned long long q = atomicAdd(list_n + (giant ? 1 : 0), 1ull);
            if (q < list_cap) {
                uint64_t* L = lists + 2 * ((giant ? list_cap : 0) + q);
                L[0] = ((uint64_t)table << 32) | s;
                L[1] = e;
            }
        }
        return;
    }
    const uint64_t g0 = (uint64_t)table * n + s;  // global position of the stretch
    // stage; each warp compacts the bin starts of its own segment
    const uint32_t seg = ((uint32_t)E + BW_W * 32 - 1) / (BW_W * 32) * 32;
    const uint32_t j0w = warp * seg, j1w = min((uint32_t)E, j0w + seg);
    uint32_t nstart = 0;
    uint32_t prev_top = 0;
    if (j0w < j1w && j0w > 0) prev_top = bb_top(okeys[g0 + j0w - 1]);
    for (uint32_t j0 = j0w; j0 < j1w; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool ok = j < j1w;
        const uint64_t key = ok ? okeys[g0 + j] : 0;
        const uint32_t tp = bb_top(key);
        uint32_t up = __shfl_up_sync(0xffffffffu, tp, 1);
        if (lane == 0) up = prev_top;
        const bool bnd = ok && (j == 0 || up != tp);
        if (ok) {
            ka[j] = (uint16_t)(key >> 32);
            ia[j] = (uint16_t)j;
            slo[j] = (uint32_t)key;
            sid[j] = oids[g0 + j];
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, bnd);
        if (bnd) ib[j0w + nstart + __popc(bal & lt)] = (uint16_t)j;  // warp-local list
        nstart += __popc(bal);
        prev_top = __shfl_sync(0xffffffffu, tp, 31);
    }
    if (lane == 0) wtot[warp] = nstart;
    __syncthreads();
    uint32_t base = 0, nb = 0;
    for (uint32_t w = 0; w < BW_W; ++w) {
        if (w < warp) base += wtot[w];
        nb += wtot[w];
    }
    for (uint32_t q = lane; q < nstart; q += 32) binst[base + q] = ib[j0w + q];
    __syncthreads();
    uint16_t* wc = cnt[warp];
    while (true) {
        uint32_t bi = 0;
        if (lane == 0) bi = atomicAdd(&next_bin, 1u);
        bi = __shfl_sync(0xffffffffu, bi, 0);
        if (bi >= nb) break;
        const uint32_t b0 = binst[bi];
        const uint32_t b1 = bi + 1 < nb ? binst[bi + 1] : (uint32_t)E;
        const uint32_t sz = b1 - b0;
        if (sz > 1) {
            bw_pass(ka, ia, kb, ib, b0, sz, 0, wc);   // key bits 32-39
            bw_pass(kb, ib, ka, ia, b0, sz, 8, wc);   // key bits 40-47
        }
        // the bin's top 16 bits from its first member (all members share them)
        const uint64_t tb = (uint64_t)bb_top(okeys[g0 + b0]) << 48;
        bool collide = false;
        for (uint32_t j0 = 0; j0 < sz; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool ok = j < sz;
            uint64_t key = 0;
            if (ok) {
                const uint32_t li = ia[b0 + j];
                key = tb | ((uint64_t)ka[b0 + j] << 32) | slo[li];
                sids[g0 + b0 + j] = sid[li];
            }
            uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1);
            uint64_t next = __shfl_down_sync(0xffffffffu, key, 1);
            if (lane == 0 && ok && j > 0)
                prev = tb | ((uint64_t)ka[b0 + j - 1] << 32) | slo[ia[b0 + j - 1]];
            if (lane == 31 && j + 1 < sz)
                next = tb | ((uint64_t)ka[b0 + j + 1] << 32) | slo[ia[b0 + j + 1]];
            if (ok) {
                const bool head = j == 0 || prev != key;
                const bool tail = j + 1 == sz || next != key;
                flags[g0 + b0 + j] = (uint8_t)((head ? 1 : 0) | (tail ? 2 : 0));
                if (j > 0 && prev != key && (prev >> 32) == (key >> 32)) collide = true;
            }
        }
        if (__any_sync(0xffffffffu, collide) && lane == 0) {
            const unsigned long long q = atomicAdd(list_n + 0, 1ull);
            if (q < list_cap) {
                uint64_t* L = lists + 2 * q;
                L[0] = ((uint64_t)table << 32) | (s + b0);
                L[1] = s + b1;
            }
        }
        __syncwarp();
    }
}

// grid (ceil(n / BB_R), t): the stretch [c R, (c + 1) R) moved to range
// boundaries; stretches above BB_CAP_S go to the mid list [0, cap) or the
// giant list [cap, 2 cap) as (table << 32 | start, end) pairs
__global__ void __launch_bounds__(256) k_bb_ranges(const uint64_t* __restrict__ okeys,
                                                   const uint32_t* __restrict__ oids, uint64_t n,
                                                   uint32_t* __restrict__ sids,
                                                   uint8_t* __restrict__ flags,
                                                   uint64_t* __restrict__ lists,
                                                   unsigned long long* __restrict__ list_n,
                                                   uint64_t list_cap) {
    extern __shared__ __align__(16) unsigned char bbs[];
    __shared__ uint64_t se[2];
    const uint32_t table = blockIdx.y, warp = threadIdx.x >> 5;
    const uint64_t* k = okeys + (uint64_t)table * n;
    if (warp < 2) {
        const uint64_t p = min(n, ((uint64_t)blockIdx.x + warp) * BB_R);
        const uint64_t b = bb_next_boundary(k, n, p);
        if ((threadIdx.x & 31) == 0) se[warp] = b;
    }
    __syncthreads();
    const uint64_t s = se[0], e = se[1];
    if (s >= e) return;
    const uint64_t E = e - s;
    if (E > BB_CAP_S) {
        if (threadIdx.x == 0) {
            const bool giant = E > BB_CAP_M;
            const unsigned long long q = atomicAdd(list_n + (giant ? 1 : 0), 1ull);
            if (q < list_cap) {
                uint64_t* L = lists + 2 * ((giant ? list_cap : 0) + q);
                L[0] = ((uint64_t)table << 32) | s;
                L[1] = e;
            }
        }
        return;
    }
    bb_one_range<BB_CAP_S>(okeys, oids, (uint64_t)table * n + s, (uint32_t)E, bbs, sids, flags);
}

// mid stretches (BB_CAP_S < E <= BB_CAP_M): persistent CTAs over the list
__global__ void __launch_bounds__(1024) k_bb_mid(const uint64_t* __restrict__ okeys,
                                                 const uint32_t* __restrict__ oids, uint64_t n,
                                                 uint32_t* __restrict__ sids,
                                                 uint8_t* __restrict__ flags,
                                                 const uint64_t* __restrict__ lists,
                                                 unsigned long long* __restrict__ list_n,
                                                 uint64_t list_cap) {
    extern __shared__ __align__(16) unsigned char bbs[];
    __shared__ unsigned long long item;
    const uint64_t nl = min((unsigned long long)list_cap, list_n[0]);
    while (true) {
        if (threadIdx.x == 0) item = atomicAdd(list_n + 2, 1ull);
        __syncthreads();
        const uint64_t it = item;
        __syncthreads();
        if (it >= nl) break;
        const uint64_t a = lists[2 * it], e = lists[2 * it + 1];
        const uint32_t table = (uint32_t)(a >> 32);
        const uint64_t s = (uint32_t)a;
        bb_one_range<BB_CAP_M>(okeys, oids, (uint64_t)table * n + s, (uint32_t)(e - s), bbs, sids,
                               flags);
    }
}

// giant stretches (> BB_CAP_M members): one CTA, sorting in global scratch
__global__ void __launch_bounds__(1024) k_bb_giant(const uint64_t* __restrict__ okeys,
                                                   const uint32_t* __restrict__ oids, uint64_t n,
                                                   uint32_t* __restrict__ sids,
                                                   uint8_t* __restrict__ flags,
                                                   const uint64_t* __restrict__ lists,
                                                   const unsigned long long* __restrict__ list_n,
                                                   uint64_t list_cap, uint32_t* __restrict__ scratch) {
    __shared__ uint32_t cnt[(1024 / 32 + 1) * BB_RADIX + 4];
    const uint64_t ng = min((unsigned long long)list_cap, list_n[1]);
    for (uint64_t g = 0; g < ng; ++g) {
        const uint64_t a = lists[2 * (list_cap + g)], e = lists[2 * (list_cap + g) + 1];
        const uint32_t table = (uint32_t)(a >> 32);
        const uint64_t s = (uint32_t)a;
        const uint32_t E = (uint32_t)(e - s);
        uint32_t* va = scratch;
        uint32_t* vb = va + n;
        uint32_t* ia = vb + n;
        uint32_t* ib = ia + n;
        uint64_t* kbuf = (uint64_t*)(ib + n + (n & 1));
        bb_sort_bin<uint32_t>(okeys, oids, (uint64_t)table * n + s, E, 0, va, vb, ia, ib, kbuf, cnt,
                              sids, flags, true);
        __syncthreads();
    }
}

}  // namespace qs

using namespace qs;

namespace {

struct BbLayout {
    size_t okeys, oids, altk, altv, rws, lists, scratch, total;
    uint64_t list_cap;
};

BbLayout bb_layout(uint64_t n, uint32_t t) {
    BbLayout L;
    const uint64_t total = n * t;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = (o + 255) & ~(size_t)255;
        o = at + bytes;
        return at;
    };
    L.list_cap = ((n + BB_R - 1) / BB_R) * t + 1;
    L.okeys = take((size_t)total * 8);
    L.oids = take((size_t)total * 4);
    L.altk = take((size_t)total * 8);
    L.altv = take((size_t)total * 4);
    L.rws = take(radix_ws_bytes(n, t));
    L.lists = take((size_t)(4 * L.list_cap + 4) * 8);
    L.scratch = take((size_t)n * 24 + 64);
    L.total = o + 256;
    return L;
}

}  // namespace

namespace qs {

size_t bucket_bins_ws_bytes(uint64_t n, uint32_t t) {
    if (n == 0 || t == 0) return 256;
    return bb_layout(n, t).total;
}

int bucket_bins_build(const uint64_t* keys, uint64_t n, uint32_t t, uint32_t* sids, uint8_t* flags,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n == 0 || t == 0) return QS_OK;
    QS_ARG(n < (1ull << 32), "more than 2**32 fingerprints are not supported");
    const BbLayout L = bb_layout(n, t);
    QS_ARG(ws_bytes >= L.total, "bucket workspace too small");
    unsigned char* w = (unsigned char*)ws;
    uint64_t* okeys = (uint64_t*)(w + L.okeys);
    uint32_t* oids = (uint32_t*)(w + L.oids);
    unsigned long long* list_n = (unsigned long long*)(w + L.lists);
    uint64_t* lists = (uint64_t*)(list_n + 4);  // after [0] mid count, [1] giant count, [2] cursor
    uint32_t* scratch = (uint32_t*)(w + L.scratch);
    // pass 1: stable order by the top 16 key bits (two coalesced 8-bit passes)
    int rc = radix_sort_pairs_to(keys, nullptr, n, t, 64 - BB_TOP, 64, okeys, oids,
                                 (uint64_t*)(w + L.altk), (uint32_t*)(w + L.altv), w + L.rws,
                                 radix_ws_bytes(n, t), st);
    if (rc) return rc;
    // pass 2: shared-memory sorts of whole top-16 ranges
    QS_CUDA(cudaMemsetAsync(list_n, 0, 32, st), "memset");
    const int wS = 256, wM = 1024;
    const size_t smS = (size_t)BB_CAP_S * 12 + (size_t)(wS / 32 + 1) * BB_RADIX * 4 + 16;
    const size_t smM = (size_t)BB_CAP_M * 12 + (size_t)(wM / 32 + 1) * BB_RADIX * 4 + 16;
    QS_CUDA(cudaFuncSetAttribute(k_bb_ranges, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smS),
            "smem attr");
    static const bool block_ranges = getenv("QS_BB_BLOCK") && getenv("QS_BB_BLOCK")[0] == '1';
    const size_t smW = (size_t)BW_CAP * 18 + (size_t)BW_W * 256 * 2;
    QS_CUDA(cudaFuncSetAttribute(k_bb_warpbins, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smW), "smem attr");
    QS_CUDA(cudaFuncSetAttribute(k_bb_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smM),
            "smem attr");
    const uint64_t ctas = (n + BB_R - 1) / BB_R;
    QS_ARG(ctas < (1ull << 31) && t <= 65535, "table too large for the bucket build");
    if (block_ranges)
        k_bb_ranges<<<dim3((unsigned)ctas, t), wS, smS, st>>>(okeys, oids, n, sids, flags, lists,
                                                              list_n, L.list_cap);
    else
        k_bb_warpbins<<<dim3((unsigned)ctas, t), BW_T, smW, st>>>(okeys, oids, n, sids, flags,
                                                                  lists, list_n, L.list_cap);
    k_bb_mid<<<num_sms(), wM, smM, st>>>(okeys, oids, n, sids, flags, lists, list_n, L.list_cap);
    k_bb_giant<<<1, 1024, 0, st>>>(okeys, oids, n, sids, flags, lists, list_n, L.list_cap, scratch);
    QS_CHECK_LAUNCH("bucket build pass 2");
    return QS_OK;
}

}  // namespace qs
