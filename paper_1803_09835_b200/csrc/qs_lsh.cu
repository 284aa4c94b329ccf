// LSH search stages on sm_100a (integer / byte work, HBM- and ALU-bound).
//
// Reference: lsh_search.py:157-303.  The reference builds per-table sorted
// columns, then for every query gathers all equal-signature members of every
// table, materialises one 8-byte (q, c) key per (pair, table) hit, sorts all
// keys and run-length counts them (lsh_search.py:175-219).
//
// B200 design:
//   * keys (t, n) = mix64(signature word) (a bijection, so bucket equality is
//     exactly the reference's) + bit-sliced 16-bit tags (n, 16, W) per row;
//   * buckets = per-table stable (key, id) sort, ids ascending in a bucket;
//   * pair enumeration inside buckets, each unordered pair handled ONLY in
//     the bucket of its first colliding table: earlier tables are screened by
//     64 LOP3s on the tag planes and confirmed on the 64-bit keys, the total
//     collision count is the popcount of the tag-match mask (confirmed on the
//     keys only when it could reach m).  No (pair, table) key is ever
//     materialised and no global hash table is needed: HBM traffic is O(n*t)
//     while the per-hit work is register/shared-memory ALU work.
#include "qs_common.cuh"

namespace qs {

int radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t seg_len, uint32_t segments,
                     uint32_t key_bits, uint64_t* keys_alt, uint32_t* vals_alt, void* ws,
                     size_t ws_bytes, int* in_alt, cudaStream_t st);
size_t radix_ws_bytes(uint64_t seg_len, uint32_t segments);

__device__ __forceinline__ uint64_t mix_key(uint64_t s) { return fmix64(s ^ GOLDEN64); }

// partition index of fingerprint i: edges[k] <= i < edges[k+1]
__device__ __forceinline__ uint32_t part_of(const uint64_t* __restrict__ edges, uint32_t p,
                                            uint64_t i) {
    uint32_t lo = 0, hi = p;  // invariant edges[lo] <= i < edges[hi]
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(edges + mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------------- prep
// Row-major signatures -> table-major keys + bit-sliced tags (one warp per row).
__global__ void __launch_bounds__(256) k_prep(const uint64_t* __restrict__ sigs, uint64_t n,
                                              uint32_t t, uint64_t* __restrict__ keys,
                                              uint32_t* __restrict__ tags) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t W = (t + 31) >> 5;
    for (uint64_t row = gwarp; row < n; row += nwarps) {
        for (uint32_t wr = 0; wr < W; ++wr) {
            const uint32_t i = wr * 32 + lane;
            uint64_t key = 0;
            if (i < t) {
                key = mix_key(sigs[row * t + i]);
                keys[(uint64_t)i * n + row] = key;
            }
            const uint32_t tag = (uint32_t)key & 0xFFFFu;
            uint32_t plane = 0;
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                uint32_t word = __ballot_sync(0xffffffffu, (i < t) && ((tag >> b) & 1u));
                if (lane == (uint32_t)b) plane = word;
            }
            if (lane < 16) tags[(row * 16 + lane) * W + wr] = plane;
        }
    }
}

__global__ void k_iota_segments(uint32_t* __restrict__ ids, uint64_t n, uint32_t t) {
    uint64_t total = n * t;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        ids[i] = (uint32_t)(i % n);
}

// --------------------------------------------------------------- listing
// Ordered compaction of bucket heads/tails over the sorted (t, n) key array.
// kind 0: heads of non-singleton buckets, kind 1: tails of non-singleton
// buckets, kind 2: all heads (count only).
__device__ __forceinline__ bool list_flag(const uint64_t* __restrict__ k, uint64_t n,
                                          uint64_t g, int kind) {
    const uint64_t pos = g % n;
    const uint64_t key = k[g];
    const bool head = pos == 0 || k[g - 1] != key;
    const bool tail = pos == n - 1 || k[g + 1] != key;
    if (kind == 0) return head && !tail;
    if (kind == 1) return tail && !head;
    return head;
}

constexpr int LIST_THREADS = 512;

__global__ void __launch_bounds__(LIST_THREADS) k_list_count(const uint64_t* __restrict__ k,
                                                             uint64_t n, uint64_t total,
                                                             uint64_t chunk, int kind,
                                                             uint64_t* __restrict__ counts) {
    __shared__ uint32_t red[LIST_THREADS / 32];
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    uint32_t c = 0;
    for (uint64_t g = lo + threadIdx.x; g < hi; g += LIST_THREADS) c += list_flag(k, n, g, kind);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t s = 0;
        for (int w = 0; w < LIST_THREADS / 32; ++w) s += red[w];
        counts[blockIdx.x] = s;
    }
}

// single-CTA exclusive scan of `len` uint64 values in place; total to *total
__global__ void __launch_bounds__(1024) k_scan_u64(uint64_t* __restrict__ a, uint64_t len,
                                                   uint64_t* __restrict__ total) {
    __shared__ uint64_t ws[32];
    __shared__ uint64_t carry;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < len; b0 += 1024) {
        const uint64_t i = b0 + threadIdx.x;
        const uint64_t v = i < len ? a[i] : 0;
        uint64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint64_t w = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= (uint32_t)o) w += y;
            }
            ws[lane] = w;
        }
        __syncthreads();
        const uint64_t incl = carry + (warp ? ws[warp - 1] : 0) + x;
        if (i < len) a[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// kind 0 writes global positions (uint64) of non-singleton heads; kind 1
// writes in-table positions (uint32) of non-singleton tails.
__global__ void __launch_bounds__(LIST_THREADS) k_list_write(const uint64_t* __restrict__ k,
                                                             uint64_t n, uint64_t total,
                                                             uint64_t chunk, int kind,
                                                             const uint64_t* __restrict__ offs,
                                                             uint64_t* __restrict__ out64,
                                                             uint32_t* __restrict__ out32) {
    __shared__ uint32_t wsum[LIST_THREADS / 32];
    __shared__ uint64_t base;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    if (threadIdx.x == 0) base = offs[blockIdx.x];
    __syncthreads();
    for (uint64_t g0 = lo; g0 < hi; g0 += LIST_THREADS) {
        const uint64_t g = g0 + threadIdx.x;
        const bool f = g < hi && list_flag(k, n, g, kind);
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        uint64_t wb = base;
        uint32_t tot = 0;
        for (int w = 0; w < LIST_THREADS / 32; ++w) {
            if (w < (int)warp) wb += wsum[w];
            tot += wsum[w];
        }
        if (f) {
            const uint64_t o = wb + __popc(bal & ((1u << lane) - 1u));
            if (kind == 0) out64[o] = g;
            else out32[o] = (uint32_t)(g % n);
        }
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
}

// bsize holds in-table tail positions on entry, bucket sizes on exit
__global__ void k_make_sizes(const uint64_t* __restrict__ heads, const uint64_t* __restrict__ nbp,
                             uint64_t n, uint32_t* __restrict__ bsize) {
    const uint64_t nb = *nbp;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x)
        bsize[i] = (uint32_t)(bsize[i] - heads[i] % n + 1);
}

// ----------------------------------------------------------------- stats
// One thread per non-singleton bucket: partition split, lookups, size histogram.
__global__ void k_bucket_stats(const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
                               const uint32_t* __restrict__ bsize, uint64_t nb,
                               const uint8_t* __restrict__ excl_mask,
                               const uint64_t* __restrict__ edges, uint32_t p,
                               unsigned long long* __restrict__ hist, uint32_t hist_len,
                               uint32_t* __restrict__ big, uint64_t big_cap,
                               unsigned long long* __restrict__ out) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t st = bstart[b];
        const uint64_t s = bsize[b];
        unsigned long long looks = 0, pieces = 0, mx = 0;
        uint64_t cum_e = 0, e_tot = 0;
        uint64_t j = 0;
        while (j < s) {
            const uint64_t id = sids[st + j];
            const uint32_t P = p > 1 ? part_of(edges, p, id) : 0;
            const uint64_t end = p > 1 ? edges[P + 1] : ~0ULL;
            uint64_t nP = 0, eP = 0;
            while (j < s) {
                const uint64_t x = sids[st + j];
                if (x >= end) break;
                ++nP;
                if (excl_mask && excl_mask[x]) ++eP;
                ++j;
            }
            cum_e += eP;
            e_tot += eP;
            looks += nP * (s - cum_e);
            ++pieces;
            if (nP > mx) mx = nP;
            if (nP < hist_len) atomicAdd(hist + nP, 1ULL);
            else {
                unsigned long long k = atomicAdd(out + 2, 1ULL);
                if (k < big_cap) big[k] = (uint32_t)nP;
            }
        }
        looks -= (s - e_tot);
        atomicAdd(out + 0, looks);
        atomicAdd(out + 1, pieces);
        atomicMax(out + 3, mx);
    }
}

// ----------------------------------------------------------------- pairs
constexpr int PAIR_WARPS = 4;
constexpr uint32_t GRAB = 16;

__device__ __forceinline__ bool keys_equal(const uint64_t* __restrict__ keys, uint64_t n,
                                           uint32_t tt, uint64_t a, uint64_t b) {
    return __ldg(keys + (uint64_t)tt * n + a) == __ldg(keys + (uint64_t)tt * n + b);
}

// W = 32-table words per tag plane (compile-time, 1..4).
template <int W>
__global__ void __launch_bounds__(PAIR_WARPS * 32) k_pairs(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint64_t* __restrict__ chunk_off, uint64_t nb,
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ tags, uint64_t n, uint32_t t,
    uint32_t m, uint64_t excl, const uint8_t* __restrict__ emask,
    const uint64_t* __restrict__ edges, uint32_t p, uint64_t* __restrict__ out_key,
    uint32_t* __restrict__ out_sim, uint64_t cap, unsigned long long* __restrict__ counters,
    unsigned long long* __restrict__ work) {
    __shared__ __align__(16) uint32_t rows[PAIR_WARPS][32][16 * W];
    __shared__ uint32_t rid[PAIR_WARPS][32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t total_chunks = chunk_off[nb];
    const uint32_t last_mask = (t & 31) ? ((1u << (t & 31)) - 1u) : 0xFFFFFFFFu;
    unsigned long long distinct = 0;

    while (true) {
        unsigned long long g0 = 0;
        if (lane == 0) g0 = atomicAdd(work, (unsigned long long)GRAB);
        g0 = __shfl_sync(0xffffffffu, g0, 0);
        if (g0 >= total_chunks) break;
        const uint64_t g1 = min((uint64_t)g0 + GRAB, total_chunks);
        // bucket of chunk g0: largest b with chunk_off[b] <= g0
        uint64_t lo = 0, hi = nb;
        while (hi - lo > 1) {
            uint64_t mid = (lo + hi) >> 1;
            if (chunk_off[mid] <= g0) lo = mid;
            else hi = mid;
        }
        uint64_t b = lo;
        for (uint64_t g = g0; g < g1; ++g) {
            while (chunk_off[b + 1] <= g) ++b;
            const uint64_t c = g - chunk_off[b];
            const uint64_t st = bstart[b];
            const uint32_t s = bsize[b];
            const uint32_t table = (uint32_t)(st / n);
            const uint32_t wt = table >> 5, bt = table & 31;
            const uint32_t i = (uint32_t)c * 32 + lane;
            const bool active = i < s;
            const uint32_t a = active ? sids[st + i] : 0;
            uint32_t A[16][W];
            if (active) {
                const uint4* src = (const uint4*)(tags + (uint64_t)a * 16 * W);
                if (W == 4) {
#pragma unroll
                    for (int pl = 0; pl < 16; ++pl) {
                        uint4 v = __ldg(src + pl);
                        A[pl][0] = v.x; A[pl][1 % W] = v.y; A[pl][2 % W] = v.z; A[pl][3 % W] = v.w;
                    }
                } else {
#pragma unroll
                    for (int pl = 0; pl < 16; ++pl)
#pragma unroll
                        for (int w = 0; w < W; ++w) A[pl][w] = __ldg(tags + ((uint64_t)a * 16 + pl) * W + w);
                }
            } else {
#pragma unroll
                for (int pl = 0; pl < 16; ++pl)
#pragma unroll
                    for (int w = 0; w < W; ++w) A[pl][w] = 0;
            }
            const bool a_ex = emask && active && emask[a];
            const uint32_t a_part = (emask && p > 1 && active) ? part_of(edges, p, a) : 0;
            for (uint32_t jb = (uint32_t)c * 32; jb < s; jb += 32) {
                const uint32_t jj = jb + lane;
                __syncwarp();
                if (jj < s) {
                    const uint32_t bid = sids[st + jj];
                    rid[warp][lane] = bid;
                    const uint4* src = (const uint4*)(tags + (uint64_t)bid * 16 * W);
                    uint4* dst = (uint4*)&rows[warp][lane][0];
#pragma unroll
                    for (int q = 0; q < 4 * W; ++q) dst[q] = __ldg(src + q);
                }
                __syncwarp();
                const uint32_t un = min(32u, s - jb);
                for (uint32_t u = 0; u < un; ++u) {
                    const uint32_t j = jb + u;
                    if (!(active && j > i)) continue;
                    const uint32_t bid = rid[warp][u];
                    const uint64_t dt = (uint64_t)bid - a;  // ids ascend within a bucket
                    if (dt <= excl) continue;
                    if (emask) {
                        if (a_ex) continue;
                        if (emask[bid] && (p <= 1 || part_of(edges, p, bid) == a_part)) continue;
                    }
                    uint32_t M[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) M[w] = 0xFFFFFFFFu;
                    const uint4* rb = (const uint4*)&rows[warp][u][0];
                    if (W == 4) {
#pragma unroll
                        for (int pl = 0; pl < 16; ++pl) {
                            const uint4 v = rb[pl];
                            M[0] &= ~(A[pl][0] ^ v.x);
                            M[1 % W] &= ~(A[pl][1 % W] ^ v.y);
                            M[2 % W] &= ~(A[pl][2 % W] ^ v.z);
                            M[3 % W] &= ~(A[pl][3 % W] ^ v.w);
                        }
                    } else {
                        const uint32_t* rw = &rows[warp][u][0];
#pragma unroll
                        for (int pl = 0; pl < 16; ++pl)
#pragma unroll
                            for (int w = 0; w < W; ++w) M[w] &= ~(A[pl][w] ^ rw[pl * W + w]);
                    }
                    M[W - 1] &= last_mask;
                    // earlier tables (first-colliding-table rule)
                    bool first = true;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        if ((uint32_t)w > wt) break;
                        uint32_t e = (uint32_t)w < wt ? M[w] : (M[w] & ((1u << bt) - 1u));
                        while (e && first) {
                            const uint32_t tt = w * 32 + __ffs(e) - 1;
                            e &= e - 1;
                            if (keys_equal(keys, n, tt, a, bid)) first = false;
                        }
                    }
                    if (!first) continue;
                    ++distinct;
                    uint32_t tot = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) tot += __popc(M[w]);
                    if (tot < m) continue;
                    uint32_t exact = 1;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        uint32_t e = M[w];
                        if ((uint32_t)w == wt) e &= ~(1u << bt);
                        while (e) {
                            const uint32_t tt = w * 32 + __ffs(e) - 1;
                            e &= e - 1;
                            exact += keys_equal(keys, n, tt, a, bid);
                        }
                    }
                    if (exact >= m) {
                        const unsigned long long pos = atomicAdd(counters + 1, 1ULL);
                        if (pos < cap) {
                            out_key[pos] = (dt << 32) | a;
                            out_sim[pos] = exact;
                        }
                    }
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, o);
    if (lane == 0 && distinct) atomicAdd(counters + 0, distinct);
}

// Generic path for t > 128: tag words read from global memory per pair.
__global__ void __launch_bounds__(256) k_pairs_generic(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, const uint64_t* __restrict__ chunk_off, uint64_t nb,
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ tags, uint64_t n, uint32_t t,
    uint32_t m, uint64_t excl, const uint8_t* __restrict__ emask,
    const uint64_t* __restrict__ edges, uint32_t p, uint64_t* __restrict__ out_key,
    uint32_t* __restrict__ out_sim, uint64_t cap, unsigned long long* __restrict__ counters) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t W = (t + 31) >> 5;
    const uint64_t total_chunks = chunk_off[nb];
    unsigned long long distinct = 0;
    for (uint64_t g = gwarp; g < total_chunks; g += nwarps) {
        uint64_t lo = 0, hi = nb;
        while (hi - lo > 1) {
            uint64_t mid = (lo + hi) >> 1;
            if (chunk_off[mid] <= g) lo = mid;
            else hi = mid;
        }
        const uint64_t b = lo, c = g - chunk_off[b], st = bstart[b];
        const uint32_t s = bsize[b], table = (uint32_t)(st / n);
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
            uint32_t tot = 0, exact = 0;
            for (uint32_t w = 0; w < W; ++w) {
                uint32_t M = 0xFFFFFFFFu;
                for (int pl = 0; pl < 16; ++pl)
                    M &= ~(tags[((uint64_t)a * 16 + pl) * W + w] ^ tags[((uint64_t)bid * 16 + pl) * W + w]);
                if (w == W - 1 && (t & 31)) M &= (1u << (t & 31)) - 1u;
                uint32_t e = M;
                while (e) {
                    const uint32_t tt = w * 32 + __ffs(e) - 1;
                    e &= e - 1;
                    if (keys_equal(keys, n, tt, a, bid)) {
                        if (tt < table) first = false;
                        ++exact;
                    }
                }
                tot += __popc(M);
            }
            (void)tot;
            if (!first) continue;
            ++distinct;
            if (exact >= m) {
                const unsigned long long pos = atomicAdd(counters + 1, 1ULL);
                if (pos < cap) {
                    out_key[pos] = (dt << 32) | a;
                    out_sim[pos] = exact;
                }
            }
        }
    }
    atomicAdd(counters + 0, distinct);
}

__global__ void k_chunk_counts(const uint32_t* __restrict__ bsize, uint64_t nb,
                               uint64_t* __restrict__ off) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x)
        off[i] = (bsize[i] + 31) / 32;
}

// ------------------------------------------------------------ occurrence
__global__ void k_occ_degree(const uint64_t* __restrict__ pk, uint64_t np,
                             const uint64_t* __restrict__ edges, uint32_t p,
                             uint32_t* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = pk[i] & 0xFFFFFFFFull, q = c + (pk[i] >> 32);
        if (p > 1 && part_of(edges, p, c) != part_of(edges, p, q)) continue;
        atomicAdd(deg + c, 1u);
        atomicAdd(deg + q, 1u);
    }
}

__global__ void k_occ_core(const uint32_t* __restrict__ deg, uint64_t n, double thr,
                           const uint64_t* __restrict__ edges, uint32_t p,
                           uint8_t* __restrict__ ex) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t P = p > 1 ? part_of(edges, p, i) : 0;
        const double size = (double)(edges[P + 1] - edges[P]);
        ex[i] = ((double)deg[i] > thr * size) ? 2 : 0;  // 2 = core
    }
}

__global__ void k_occ_touch(const uint64_t* __restrict__ pk, uint64_t np,
                            const uint64_t* __restrict__ edges, uint32_t p,
                            uint8_t* __restrict__ ex) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = pk[i] & 0xFFFFFFFFull, q = c + (pk[i] >> 32);
        if (p > 1 && part_of(edges, p, c) != part_of(edges, p, q)) continue;
        if (ex[c] == 2 || ex[q] == 2) {
            if (ex[c] == 0) ex[c] = 1;
            if (ex[q] == 0) ex[q] = 1;
        }
    }
}

__global__ void k_occ_finish(uint8_t* __restrict__ ex, uint64_t n,
                             unsigned long long* __restrict__ count) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t v = ex[i] ? 1 : 0;
        ex[i] = v;
        c += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// -------------------------------------------------------------- finalize
__global__ void k_pack_triplets(const uint64_t* __restrict__ key, const uint32_t* __restrict__ sim,
                                uint64_t np, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[i];
        const uint64_t dt = k >> 32, idx1 = k & 0xFFFFFFFFull;
        uint32_t* r = out + i * 5;  // <u8 dt, <u8 idx1, <u4 sim (20 bytes, little endian)
        r[0] = (uint32_t)dt;
        r[1] = (uint32_t)(dt >> 32);
        r[2] = (uint32_t)idx1;
        r[3] = 0;
        r[4] = sim[i];
    }
}

}  // namespace qs

using namespace qs;

extern "C" {

int qs_lsh_prep(const uint64_t* sigs_dev, uint64_t n, uint32_t t, uint64_t* keys_dev,
                uint32_t* tags_dev, void* stream) {
    QS_ARG(t >= 1, "tables must be >= 1");
    if (n == 0) return QS_OK;
    k_prep<<<qs_blocks(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(sigs_dev, n, t, keys_dev, tags_dev);
    QS_CHECK_LAUNCH("k_prep");
    return QS_OK;
}

size_t qs_lsh_bucket_ws_bytes(uint64_t n, uint32_t t) {
    return (size_t)n * t * (sizeof(uint64_t) + sizeof(uint32_t)) + radix_ws_bytes(n, t) + 512;
}

int qs_lsh_build_buckets(const uint64_t* keys_dev, uint64_t n, uint32_t t, uint64_t* keys_out_dev,
                         uint32_t* ids_out_dev, void* ws_dev, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0 || t == 0) return QS_OK;
    QS_ARG(n < (1ull << 32), "more than 2**32 fingerprints are not supported");
    QS_ARG(ws_bytes >= qs_lsh_bucket_ws_bytes(n, t), "bucket workspace too small");
    const uint64_t total = n * t;
    unsigned char* w = (unsigned char*)ws_dev;
    uint64_t* alt_k = (uint64_t*)w;
    uint32_t* alt_v = (uint32_t*)(w + total * 8);
    void* rws = (void*)(((uintptr_t)(w + total * 12) + 255) & ~(uintptr_t)255);
    if (keys_out_dev != keys_dev)
        QS_CUDA(cudaMemcpyAsync(keys_out_dev, keys_dev, total * 8, cudaMemcpyDeviceToDevice, st), "copy keys");
    k_iota_segments<<<qs_blocks(total, 256), 256, 0, st>>>(ids_out_dev, n, t);
    QS_CHECK_LAUNCH("k_iota_segments");
    int in_alt = 0;
    int rc = radix_sort_pairs(keys_out_dev, ids_out_dev, n, t, 64, alt_k, alt_v, rws,
                              radix_ws_bytes(n, t), &in_alt, st);
    if (rc) return rc;
    if (in_alt) {
        QS_CUDA(cudaMemcpyAsync(keys_out_dev, alt_k, total * 8, cudaMemcpyDeviceToDevice, st), "copy");
        QS_CUDA(cudaMemcpyAsync(ids_out_dev, alt_v, total * 4, cudaMemcpyDeviceToDevice, st), "copy");
    }
    return QS_OK;
}

static uint64_t list_blocks(uint64_t total) {
    uint64_t b = (total + 65535) / 65536;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return b;
}

size_t qs_lsh_list_ws_bytes(uint64_t n, uint32_t t) {
    uint64_t b = list_blocks(n * t);
    return (size_t)(b + 1) * 8 * 3 + 256;
}

int qs_lsh_list_buckets(const uint64_t* skeys_dev, uint64_t n, uint32_t t, uint64_t* bstart_dev,
                        uint32_t* bsize_dev, uint64_t* counts_dev, void* ws_dev, size_t ws_bytes,
                        void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_list_ws_bytes(n, t), "list workspace too small");
    const uint64_t total = n * t;
    if (total == 0) {
        QS_CUDA(cudaMemsetAsync(counts_dev, 0, 16, st), "memset");
        return QS_OK;
    }
    const uint64_t B = list_blocks(total);
    const uint64_t chunk = (total + B - 1) / B;
    uint64_t* cnt = (uint64_t*)ws_dev;
    if (bstart_dev == nullptr) {
        k_list_count<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, 0, cnt);
        k_scan_u64<<<1, 1024, 0, st>>>(cnt, B, counts_dev + 0);
        k_list_count<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, 2, cnt);
        k_scan_u64<<<1, 1024, 0, st>>>(cnt, B, counts_dev + 1);
        QS_CHECK_LAUNCH("list count");
        return QS_OK;
    }
    for (int kind = 0; kind < 2; ++kind) {
        k_list_count<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, kind, cnt);
        k_scan_u64<<<1, 1024, 0, st>>>(cnt, B, kind == 0 ? counts_dev : nullptr);
        k_list_write<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, kind, cnt, bstart_dev,
                                                 bsize_dev);
    }
    k_make_sizes<<<148 * 8, 256, 0, st>>>(bstart_dev, counts_dev, n, bsize_dev);
    QS_CHECK_LAUNCH("list buckets");
    return QS_OK;
}

int qs_lsh_bucket_stats(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                        const uint32_t* bsize_dev, uint64_t n_nonsingle,
                        const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p,
                        uint64_t* hist_dev, uint32_t hist_len, uint32_t* big_dev, uint64_t big_cap,
                        uint64_t* out_dev, void* stream) {
    if (n_nonsingle == 0) return QS_OK;
    k_bucket_stats<<<qs_blocks(n_nonsingle, 128), 128, 0, (cudaStream_t)stream>>>(
        sids_dev, bstart_dev, bsize_dev, n_nonsingle, excluded_dev, edges_dev, p,
        (unsigned long long*)hist_dev, hist_len, big_dev, big_cap, (unsigned long long*)out_dev);
    QS_CHECK_LAUNCH("k_bucket_stats");
    return QS_OK;
}

size_t qs_lsh_pairs_ws_bytes(uint64_t n_nonsingle) {
    return (size_t)(n_nonsingle + 1) * 8 + (qs_lsh_list_ws_bytes(n_nonsingle, 1)) + 512;
}

int qs_lsh_pairs(const uint32_t* sids_dev, const uint64_t* bstart_dev, const uint32_t* bsize_dev,
                 uint64_t n_nonsingle, const uint64_t* keys_dev, const uint32_t* tags_dev,
                 uint64_t n, uint32_t t, uint32_t m, uint64_t excl, const uint8_t* excluded_dev,
                 const uint64_t* edges_dev, uint32_t p, uint64_t* out_key_dev,
                 uint32_t* out_sim_dev, uint64_t cap, unsigned long long* counters_dev,
                 void* ws_dev, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_pairs_ws_bytes(n_nonsingle), "pairs workspace too small");
    QS_ARG(m >= 1 && m <= t, "min_matches must be in [1, tables]");
    if (n_nonsingle == 0) return QS_OK;
    uint64_t* off = (uint64_t*)ws_dev;
    unsigned long long* work = (unsigned long long*)(off + n_nonsingle + 1);
    k_chunk_counts<<<qs_blocks(n_nonsingle, 256), 256, 0, st>>>(bsize_dev, n_nonsingle, off);
    k_scan_u64<<<1, 1024, 0, st>>>(off, n_nonsingle + 1, nullptr);
    QS_CUDA(cudaMemsetAsync(work, 0, 8, st), "memset");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t W = (t + 31) >> 5;
#define QS_PAIRS(WW)                                                                              \
    k_pairs<WW><<<sms * 8, PAIR_WARPS * 32, 0, st>>>(sids_dev, bstart_dev, bsize_dev, off,        \
                                                    n_nonsingle, keys_dev, tags_dev, n, t, m, excl, \
                                                    excluded_dev, edges_dev, p, out_key_dev,     \
                                                    out_sim_dev, cap, counters_dev, work)
    switch (W) {
        case 1: QS_PAIRS(1); break;
        case 2: QS_PAIRS(2); break;
        case 3: QS_PAIRS(3); break;
        case 4: QS_PAIRS(4); break;
        default:
            k_pairs_generic<<<sms * 8, 256, 0, st>>>(sids_dev, bstart_dev, bsize_dev, off, n_nonsingle,
                                                   keys_dev, tags_dev, n, t, m, excl, excluded_dev,
                                                   edges_dev, p, out_key_dev, out_sim_dev, cap,
                                                   counters_dev);
    }
#undef QS_PAIRS
    QS_CHECK_LAUNCH("k_pairs");
    return QS_OK;
}

int qs_lsh_occurrence_filter(const uint64_t* pair_key_dev, const uint32_t* pair_sim_dev,
                             uint64_t n_pairs, uint64_t n, double threshold,
                             const uint64_t* edges_dev, uint32_t p, uint8_t* excluded_dev,
                             unsigned long long* counters_dev, void* ws_dev, void* stream) {
    (void)pair_sim_dev;
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return QS_OK;
    uint32_t* deg = (uint32_t*)ws_dev;
    QS_CUDA(cudaMemsetAsync(deg, 0, n * 4, st), "memset");
    if (n_pairs)
        k_occ_degree<<<qs_blocks(n_pairs, 256), 256, 0, st>>>(pair_key_dev, n_pairs, edges_dev, p, deg);
    k_occ_core<<<qs_blocks(n, 256), 256, 0, st>>>(deg, n, threshold, edges_dev, p, excluded_dev);
    if (n_pairs)
        k_occ_touch<<<qs_blocks(n_pairs, 256), 256, 0, st>>>(pair_key_dev, n_pairs, edges_dev, p, excluded_dev);
    k_occ_finish<<<qs_blocks(n, 256), 256, 0, st>>>(excluded_dev, n, counters_dev);
    QS_CHECK_LAUNCH("occurrence filter");
    return QS_OK;
}

size_t qs_sort_pairs_ws_bytes(uint64_t n) {
    return (size_t)n * 12 + radix_ws_bytes(n, 1) + 512;
}

int qs_lsh_finalize(uint64_t* pair_key_dev, uint32_t* pair_sim_dev, uint64_t n_pairs,
                    uint32_t key_bits, uint8_t* triplets_dev, void* ws_dev, size_t ws_bytes,
                    void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_pairs == 0) return QS_OK;
    QS_ARG(ws_bytes >= qs_sort_pairs_ws_bytes(n_pairs), "finalize workspace too small");
    unsigned char* w = (unsigned char*)ws_dev;
    uint64_t* ak = (uint64_t*)w;
    uint32_t* av = (uint32_t*)(w + n_pairs * 8);
    void* rws = (void*)(((uintptr_t)(w + n_pairs * 12) + 255) & ~(uintptr_t)255);
    int in_alt = 0;
    int rc = radix_sort_pairs(pair_key_dev, pair_sim_dev, n_pairs, 1, key_bits, ak, av, rws,
                              radix_ws_bytes(n_pairs, 1), &in_alt, st);
    if (rc) return rc;
    const uint64_t* k = in_alt ? ak : pair_key_dev;
    const uint32_t* v = in_alt ? av : pair_sim_dev;
    k_pack_triplets<<<qs_blocks(n_pairs, 256), 256, 0, st>>>(k, v, n_pairs, (uint32_t*)triplets_dev);
    QS_CHECK_LAUNCH("k_pack_triplets");
    return QS_OK;
}

}  // extern "C"
