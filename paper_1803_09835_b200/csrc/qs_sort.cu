// Stable LSD radix sort of (uint64 key, uint32 value) pairs, batched over
// equal-length independent segments (one segment per LSH table).
//
// Per 8-bit digit pass: (1) per-tile digit histograms, (2) per-segment
// exclusive scan over (digit, tile), (3) stable scatter: each tile ranks its
// keys per digit in input order (warp match_any + per-warp counters, then a
// cross-warp prefix), so equal digits keep their relative order.
#include "qs_common.cuh"

namespace qs {

#ifndef QS_RS_THREADS
#define QS_RS_THREADS 256
#endif
constexpr int RS_THREADS = QS_RS_THREADS;
#ifndef QS_RS_ITEMS
#define QS_RS_ITEMS 16
#endif
constexpr int RS_ITEMS = QS_RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 keys per tile
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_RADIX = 256;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint64_t* __restrict__ keys,
                                                        uint64_t seg_len, uint32_t tiles,
                                                        uint32_t shift,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[RS_RADIX];
    const uint32_t tile = blockIdx.x, seg = blockIdx.y;
    for (int i = threadIdx.x; i < RS_RADIX; i += RS_THREADS) h[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)seg * seg_len;
    const uint64_t lo = (uint64_t)tile * RS_TILE;
    const uint64_t hi = min(seg_len, lo + RS_TILE);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += RS_THREADS)
        atomicAdd(&h[(keys[base + i] >> shift) & 0xFF], 1u);
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < RS_RADIX; dgt += RS_THREADS)
        hist[((uint64_t)seg * RS_RADIX + dgt) * tiles + tile] = h[dgt];
}

// One CTA per segment: exclusive scan (in place) of RS_RADIX * tiles counts.
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* __restrict__ hist, uint64_t len) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    uint32_t* a = hist + (uint64_t)blockIdx.x * len;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t b0 = 0; b0 < len; b0 += 1024 * 4) {
        uint32_t v[4], s = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint64_t i = b0 + threadIdx.x * 4 + e;
            v[e] = i < len ? a[i] : 0;
            s += v[e];
        }
        uint32_t x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= (uint32_t)o) w += y;
            }
            warp_sums[lane] = w;
        }
        __syncthreads();
        uint32_t excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - s;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint64_t i = b0 + threadIdx.x * 4 + e;
            if (i < len) a[i] = excl;
            excl += v[e];
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl;
        __syncthreads();
    }
}

// Multi-block exclusive scan of one long uint32 histogram (single-segment
// sorts: a lone CTA would walk 256 x tiles entries serially).
constexpr int RSC_T = 512, RSC_I = 8;
constexpr uint64_t RSC_TILE = (uint64_t)RSC_T * RSC_I;

__device__ __forceinline__ uint64_t rs_block_excl(uint64_t v, uint64_t* wsum) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < (blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const uint64_t r = (warp ? wsum[warp - 1] : 0) + x - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(RSC_T) k_rs_scan_reduce(const uint32_t* __restrict__ a, uint64_t len,
                                                          uint64_t* __restrict__ part) {
    __shared__ uint64_t red[RSC_T / 32];
    const uint64_t base = blockIdx.x * RSC_TILE;
    uint64_t s = 0;
    for (int e = 0; e < RSC_I; ++e) {
        const uint64_t i = base + (uint64_t)e * RSC_T + threadIdx.x;
        if (i < len) s += a[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < RSC_T / 32; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_rs_scan_top(uint64_t* __restrict__ part, uint64_t nb) {
    __shared__ uint64_t ws[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < nb; b0 += 1024) {
        const uint64_t i = b0 + threadIdx.x;
        const uint64_t v = i < nb ? part[i] : 0;
        const uint64_t ex = rs_block_excl(v, ws);
        const uint64_t tot = ws[31];
        if (i < nb) part[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(RSC_T) k_rs_scan_down(uint32_t* __restrict__ a, uint64_t len,
                                                        const uint64_t* __restrict__ part) {
    __shared__ uint64_t ws[32];
    const uint64_t base = blockIdx.x * RSC_TILE + (uint64_t)threadIdx.x * RSC_I;
    uint32_t v[RSC_I];
    uint64_t s = 0;
#pragma unroll
    for (int e = 0; e < RSC_I; ++e) {
        v[e] = (base + e < len) ? a[base + e] : 0u;
        s += v[e];
    }
    uint64_t ex = rs_block_excl(s, ws) + part[blockIdx.x];
#pragma unroll
    for (int e = 0; e < RSC_I; ++e) {
        if (base + e < len) a[base + e] = (uint32_t)ex;
        ex += v[e];
    }
}

// Stable scatter of one tile: rank in input order per digit, stage the tile in
// shared memory in (digit, input) order, then write each digit's run to its
// global slot with consecutive threads on consecutive addresses (coalesced).
#ifndef QS_RS_MINB
#define QS_RS_MINB 2
#endif
__global__ void __launch_bounds__(RS_THREADS, QS_RS_MINB) k_rs_scatter(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t seg_len,
    uint32_t tiles, uint32_t shift, const uint32_t* __restrict__ offs,
    uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals) {
    extern __shared__ __align__(16) unsigned char rs_smem[];
    uint64_t* sk = (uint64_t*)rs_smem;                  // [RS_TILE]
    uint32_t* sv = (uint32_t*)(sk + RS_TILE);           // [RS_TILE]
    __shared__ uint32_t wcnt[RS_WARPS][RS_RADIX];
    __shared__ uint32_t dstart[RS_RADIX];   // digit run start inside the tile
    __shared__ uint32_t goff[RS_RADIX];     // digit run start in the output segment
    const uint32_t tile = blockIdx.x, seg = blockIdx.y;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    for (int dgt = threadIdx.x; dgt < RS_RADIX; dgt += RS_THREADS)
        goff[dgt] = offs[((uint64_t)seg * RS_RADIX + dgt) * tiles + tile];
    __syncthreads();
    const uint64_t base = (uint64_t)seg * seg_len;
    const uint64_t tile0 = (uint64_t)tile * RS_TILE;
    const uint32_t tile_n = (uint32_t)min((uint64_t)RS_TILE, seg_len - tile0);
    const uint64_t t0 = tile0 + (uint64_t)warp * (32 * RS_ITEMS);
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    const uint32_t lt = (1u << lane) - 1u;
    // all loads in flight before the ranking (its warp syncs would serialise them)
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint64_t i = t0 + (uint64_t)r * 32 + lane;
        const bool ok = i < seg_len;
        k[r] = ok ? __ldcs(keys + base + i) : 0;
        v[r] = ok ? (vals ? __ldcs(vals + base + i) : (uint32_t)i) : 0;  // no vals: position
    }
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint64_t i = t0 + (uint64_t)r * 32 + lane;
        const bool ok = i < seg_len;
        const uint32_t dgt = ok ? (uint32_t)((k[r] >> shift) & 0xFF) : 0x100u;
#ifndef QS_RS_MATCH
        uint32_t peers = 0xffffffffu;  // lanes with the same digit, from 9 ballots
#pragma unroll
        for (int b = 0; b < 9; ++b) {
            const bool bit = (dgt >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
#else
        const uint32_t peers = __match_any_sync(0xffffffffu, dgt);
#endif
        const uint32_t cnt = __popc(peers);
        const uint32_t before = __popc(peers & lt);
        uint32_t b = 0;
        if (ok) b = wcnt[warp][dgt];
        rank[r] = b + before;
        __syncwarp();
        if (ok && before == 0) wcnt[warp][dgt] = b + cnt;
        __syncwarp();
    }
    __syncthreads();
    // per digit: tile-local run start and per-warp offsets inside the run
    if (threadIdx.x < RS_RADIX) {
        const uint32_t dgt = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t c = wcnt[w][dgt];
            wcnt[w][dgt] = run;
            run += c;
        }
        dstart[dgt] = run;  // digit total for now
    }
    __syncthreads();
    // exclusive scan of digit totals (256 entries) by warp 0
    if (warp == 0) {
        uint32_t tot[8], s = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            tot[e] = dstart[lane * 8 + e];
            s += tot[e];
        }
        uint32_t x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        uint32_t ex = x - s;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            dstart[lane * 8 + e] = ex;
            ex += tot[e];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint64_t i = t0 + (uint64_t)r * 32 + lane;
        if (i < seg_len) {
            const uint32_t dgt = (uint32_t)((k[r] >> shift) & 0xFF);
            const uint32_t lp = dstart[dgt] + wcnt[warp][dgt] + rank[r];
            QS_DASSERT(lp < tile_n);
            sk[lp] = k[r];
            sv[lp] = v[r];
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tile_n; j += RS_THREADS) {
        const uint64_t key = sk[j];
        const uint32_t dgt = (uint32_t)((key >> shift) & 0xFF);
        const uint64_t pos = base + goff[dgt] + (j - dstart[dgt]);
        QS_DASSERT(pos < base + seg_len && j >= dstart[dgt]);
        okeys[pos] = key;
        ovals[pos] = sv[j];
    }
}

static uint32_t rs_tiles(uint64_t seg_len) { return (uint32_t)((seg_len + RS_TILE - 1) / RS_TILE); }

size_t radix_ws_bytes(uint64_t seg_len, uint32_t segments) {
    const uint64_t hist = (uint64_t)rs_tiles(seg_len) * RS_RADIX * segments;
    return (size_t)hist * sizeof(uint32_t) + ((hist + RSC_TILE - 1) / RSC_TILE + 1) * 8 + 512;
}

// per-segment exclusive scans of the digit histograms
static void rs_scan(uint32_t* hist, uint64_t seg_hist, uint32_t segments, void* ws,
                    cudaStream_t st) {
    if (segments > 1 || seg_hist < (1u << 18)) {
        k_rs_scan<<<segments, 1024, 0, st>>>(hist, seg_hist);
        return;
    }
    const uint64_t nb = (seg_hist + RSC_TILE - 1) / RSC_TILE;
    uint64_t* part = (uint64_t*)(((uintptr_t)(hist + seg_hist) + 15) & ~(uintptr_t)15);
    (void)ws;
    k_rs_scan_reduce<<<(unsigned)nb, RSC_T, 0, st>>>(hist, seg_hist, part);
    k_rs_scan_top<<<1, 1024, 0, st>>>(part, nb);
    k_rs_scan_down<<<(unsigned)nb, RSC_T, 0, st>>>(hist, seg_hist, part);
}

int radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t seg_len, uint32_t segments,
                     uint32_t key_bits, uint64_t* keys_alt, uint32_t* vals_alt, void* ws,
                     size_t ws_bytes, int* in_alt, cudaStream_t st, uint32_t bit_lo,
                     uint32_t lo_bits) {
    *in_alt = 0;
    if (seg_len == 0 || segments == 0 || key_bits == 0) return QS_OK;
    QS_ARG(seg_len < (1ull << 32), "radix sort segment longer than 2^32");
    QS_ARG(ws_bytes >= radix_ws_bytes(seg_len, segments), "radix sort workspace too small");
    const uint32_t tiles = rs_tiles(seg_len);
    QS_ARG(tiles <= 65535u * 64u, "too many tiles");
    uint32_t* hist = (uint32_t*)ws;
    QS_CUDA(cudaFuncSetAttribute(k_rs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 RS_TILE * 12), "smem attr");
    uint64_t *src_k = keys, *dst_k = keys_alt;
    uint32_t *src_v = vals, *dst_v = vals_alt;
    // lo_bits < 32: the low 32-bit half only uses its lowest lo_bits bits (a
    // (dt << 32 | idx1) pair key): its always-zero digits are skipped
    for (uint32_t shift = bit_lo; shift < key_bits; shift += 8) {
        if (shift < 32 && shift >= lo_bits) continue;
        dim3 grid(tiles, segments);
        k_rs_hist<<<grid, RS_THREADS, 0, st>>>(src_k, seg_len, tiles, shift, hist);
        rs_scan(hist, (uint64_t)RS_RADIX * tiles, segments, ws, st);
        k_rs_scatter<<<grid, RS_THREADS, RS_TILE * 12, st>>>(src_k, src_v, seg_len, tiles, shift,
                                                             hist, dst_k, dst_v);
        QS_CHECK_LAUNCH("radix sort pass");
        uint64_t* tk = src_k; src_k = dst_k; dst_k = tk;
        uint32_t* tv = src_v; src_v = dst_v; dst_v = tv;
        *in_alt ^= 1;
    }
    return QS_OK;
}

// Same sort with separate input / output buffers: the first pass reads
// keys_in (left untouched) and vals_in (NULL: each value is its in-segment
// position), passes alternate between out and alt so the last lands in out.
int radix_sort_pairs_to(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t seg_len,
                        uint32_t segments, uint32_t bit_lo, uint32_t key_bits, uint64_t* keys_out,
                        uint32_t* vals_out, uint64_t* keys_alt, uint32_t* vals_alt, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
    if (seg_len == 0 || segments == 0) return QS_OK;
    QS_ARG(seg_len < (1ull << 32), "radix sort segment longer than 2^32");
    QS_ARG(ws_bytes >= radix_ws_bytes(seg_len, segments), "radix sort workspace too small");
    QS_ARG(key_bits > bit_lo && (key_bits - bit_lo) % 8 == 0, "whole 8-bit digits only");
    const uint32_t tiles = rs_tiles(seg_len);
    QS_ARG(tiles <= 65535u * 64u, "too many tiles");
    uint32_t* hist = (uint32_t*)ws;
    QS_CUDA(cudaFuncSetAttribute(k_rs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 RS_TILE * 12), "smem attr");
    const uint32_t passes = (key_bits - bit_lo) / 8;
    const uint64_t* src_k = keys_in;
    const uint32_t* src_v = vals_in;
    for (uint32_t ps = 0; ps < passes; ++ps) {
        const uint32_t shift = bit_lo + 8 * ps;
        const bool to_out = ((passes - 1 - ps) & 1) == 0;
        uint64_t* dst_k = to_out ? keys_out : keys_alt;
        uint32_t* dst_v = to_out ? vals_out : vals_alt;
        dim3 grid(tiles, segments);
        k_rs_hist<<<grid, RS_THREADS, 0, st>>>(src_k, seg_len, tiles, shift, hist);
        rs_scan(hist, (uint64_t)RS_RADIX * tiles, segments, ws, st);
        k_rs_scatter<<<grid, RS_THREADS, RS_TILE * 12, st>>>(src_k, src_v, seg_len, tiles, shift,
                                                             hist, dst_k, dst_v);
        QS_CHECK_LAUNCH("radix sort pass");
        src_k = dst_k;
        src_v = dst_v;
    }
    return QS_OK;
}

}  // namespace qs

extern "C" {

size_t qs_radix_sort_ws_bytes(uint64_t seg_len, uint32_t segments) {
    return qs::radix_ws_bytes(seg_len, segments);
}

int qs_radix_sort_pairs(uint64_t* keys_dev, uint32_t* vals_dev, uint64_t seg_len,
                        uint32_t segments, uint32_t key_bits, uint64_t* keys_alt_dev,
                        uint32_t* vals_alt_dev, void* ws_dev, size_t ws_bytes,
                        int* result_in_alt, void* stream) {
    QS_ARG(key_bits <= 64, "key_bits must be <= 64");
    return qs::radix_sort_pairs(keys_dev, vals_dev, seg_len, segments, key_bits, keys_alt_dev,
                                vals_alt_dev, ws_dev, ws_bytes, result_in_alt,
                                (cudaStream_t)stream, 0, 32);
}

}  // extern "C"
