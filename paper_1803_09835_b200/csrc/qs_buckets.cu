// Bucket head/tail flags and the bucket listing built on them.
//
// The search consumes buckets (lsh_search.py:157-172 run lengths) as member
// ids grouped by key plus the bounds of every non-singleton bucket.  The
// bucket build (qs_lsh_build_buckets: stable LSD radix sort of (key, id) per
// table) leaves a sorted-key array of 8 bytes per member; one sweep turns it
// into one flag byte per member (bit 0: first member of its bucket, bit 1:
// last), and the listing then reads 1 byte per member instead of comparing
// neighbouring 8-byte keys (7.6 -> 2.7 ms at cfg1).
//
// Measured and rejected (round 1): a binned build — key-range bins of ~2k
// members scattered in one pass, each bin sorted in shared memory by id-rank
// + key sub-bin counting — came to 56 ms against the radix path's 50 ms: the
// per-bin sort is instruction-bound (~30 warp instructions per member).
#include <stdlib.h>

#include "qs_lsh.cuh"

namespace qs {

// sorted keys -> flags (adjacent key comparisons); grid (blocks, t)
__global__ void k_flags_from_keys(const uint64_t* __restrict__ sk, uint64_t n,
                                  uint8_t* __restrict__ flags) {
    const uint64_t* k = sk + (uint64_t)blockIdx.y * n;
    uint8_t* f = flags + (uint64_t)blockIdx.y * n;
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < n;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = k[pos];
        const bool head = pos == 0 || k[pos - 1] != key;
        const bool tail = pos == n - 1 || k[pos + 1] != key;
        f[pos] = (uint8_t)((head ? 1 : 0) | (tail ? 2 : 0));
    }
}

// ------------------------------------------------------ listing from flags
constexpr int LF_T = 512;

static uint64_t lf_blocks(uint64_t total) {
    uint64_t b = (total + 262143) / 262144;
    if (b < 1) b = 1;
    if (b > 148 * 8) b = 148 * 8;
    return b;
}

__global__ void __launch_bounds__(LF_T) k_listf_count(const uint8_t* __restrict__ f, uint64_t total,
                                                      uint64_t chunk, uint64_t nblk,
                                                      uint64_t* __restrict__ counts) {
    __shared__ uint32_t red[2][LF_T / 32];
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    uint32_t c0 = 0, c1 = 0;
    // 4 flags per thread step (chunk is a multiple of 4)
    for (uint64_t g = lo + threadIdx.x * 4ull; g < hi; g += LF_T * 4ull) {
        uint32_t w;
        if (g + 4 <= hi) w = *(const uint32_t*)(f + g);
        else {
            w = 0;
            for (uint64_t e = g; e < hi; ++e) w |= (uint32_t)f[e] << (8 * (e - g));
        }
        // byte b: head = bit 0, tail = bit 1; non-singleton head = head & !tail
        const uint32_t hd = w & 0x01010101u, tl = (w >> 1) & 0x01010101u;
        c0 += __popc(hd & ~tl);
        c1 += __popc(hd);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c0 += __shfl_down_sync(0xffffffffu, c0, o);
        c1 += __shfl_down_sync(0xffffffffu, c1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = c0;
        red[1][threadIdx.x >> 5] = c1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t s0 = 0, s1 = 0;
        for (int w = 0; w < LF_T / 32; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        counts[blockIdx.x] = s0;
        counts[nblk + blockIdx.x] = s1;
    }
}

// heads write their global position to bstart[i], tails their in-table
// position to bsize[i] (k_make_sizes turns those into sizes)
__global__ void __launch_bounds__(LF_T) k_listf_write(const uint8_t* __restrict__ f, uint64_t n,
                                                      uint64_t total, uint64_t chunk,
                                                      const uint64_t* __restrict__ offs,
                                                      uint64_t* __restrict__ out64,
                                                      uint32_t* __restrict__ out32) {
    __shared__ uint32_t wsum[LF_T / 32];
    __shared__ uint64_t base;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    if (threadIdx.x == 0) base = offs[blockIdx.x];
    __syncthreads();
    for (uint64_t g0 = lo; g0 < hi; g0 += LF_T * 8ull) {
        const uint64_t gt = g0 + (uint64_t)threadIdx.x * 8;
        uint64_t w = 0;
        if (gt + 8 <= hi) w = *(const uint64_t*)(f + gt);
        else
            for (uint64_t e = gt; e < hi; ++e) w |= (uint64_t)f[e] << (8 * (e - gt));
        const uint64_t hd = w & 0x0101010101010101ull, tl = (w >> 1) & 0x0101010101010101ull;
        const uint64_t H = hd & ~tl, T = tl & ~hd;
        const uint32_t c = __popcll(H);
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint64_t wb = base;
        uint32_t tot = 0;
        for (int q = 0; q < LF_T / 32; ++q) {
            if (q < (int)warp) wb += wsum[q];
            tot += wsum[q];
        }
        uint64_t incl = wb + x - c;
        if (H | T) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool h = (H >> (8 * e)) & 1, tt = (T >> (8 * e)) & 1;
                incl += h;
                if (h) out64[incl - 1] = gt + e;
                if (tt) out32[incl - 1] = (uint32_t)((gt + e) % n);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
}

}  // namespace qs

using namespace qs;

extern "C" {

// QS_BUCKET_BINS=1 selects the two-pass build of qs_bucket_bins.cu (2 radix
// passes + shared-memory range sorts): 81 instead of 143 B per (member,
// table) but measured 32-36 ms against this path's 31.7 ms at cfg1 — the
// range sorts are latency-bound
static bool use_radix_build() {
    const char* e = getenv("QS_BUCKET_BINS");
    return !(e && e[0] == '1');
}

size_t qs_lsh_bucket_flags_ws_bytes(uint64_t n, uint32_t t) {
    if (!use_radix_build()) return bucket_bins_ws_bytes(n, t);
    // sorted keys + the radix build's own workspace
    return (size_t)n * t * 8 + 256 + qs_lsh_bucket_ws_bytes(n, t);
}

int qs_lsh_build_bucket_flags(const uint64_t* keys_dev, uint64_t n, uint32_t t,
                              uint32_t* ids_out_dev, uint8_t* flags_out_dev, void* ws_dev,
                              size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0 || t == 0) return QS_OK;
    QS_ARG(ws_bytes >= qs_lsh_bucket_flags_ws_bytes(n, t), "bucket workspace too small");
    if (!use_radix_build())
        return bucket_bins_build(keys_dev, n, t, ids_out_dev, flags_out_dev, ws_dev, ws_bytes, st);
    const uint64_t total = n * t;
    uint64_t* skeys = (uint64_t*)ws_dev;
    void* rws = (void*)(((uintptr_t)(skeys + total) + 255) & ~(uintptr_t)255);
    int rc = qs_lsh_build_buckets(keys_dev, n, t, skeys, ids_out_dev, rws,
                                  qs_lsh_bucket_ws_bytes(n, t), stream);
    if (rc) return rc;
    k_flags_from_keys<<<dim3(qs_blocks(n, 256, 1184), t), 256, 0, st>>>(skeys, n, flags_out_dev);
    QS_CHECK_LAUNCH("flags from keys");
    return QS_OK;
}

size_t qs_lsh_list_flags_ws_bytes(uint64_t n, uint32_t t) {
    const uint64_t b = lf_blocks(n * t);
    return (size_t)(2 * b + 1) * 8 + scan_ws_bytes(b) + 256;
}

int qs_lsh_list_buckets_flags(const uint8_t* flags_dev, uint64_t n, uint32_t t,
                              uint64_t* bstart_dev, uint32_t* bsize_dev, uint32_t* btab_dev,
                              const uint32_t* table_ids_dev, uint64_t* counts_dev, void* ws_dev,
                              size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_list_flags_ws_bytes(n, t), "list workspace too small");
    const uint64_t total = n * t;
    if (total == 0) {
        QS_CUDA(cudaMemsetAsync(counts_dev, 0, 16, st), "memset");
        return QS_OK;
    }
    const uint64_t B = lf_blocks(total);
    const uint64_t chunk = ((total + B - 1) / B + 7) & ~7ull;
    uint64_t* cnt = (uint64_t*)ws_dev;
    void* sws = (void*)(((uintptr_t)(cnt + 2 * B + 1) + 63) & ~(uintptr_t)63);
    k_listf_count<<<B, LF_T, 0, st>>>(flags_dev, total, chunk, B, cnt);
    int rc = scan_u64(cnt, cnt, B, counts_dev + 0, sws, st);
    if (rc) return rc;
    rc = scan_u64(cnt + B, cnt + B, B, counts_dev + 1, sws, st);
    if (rc) return rc;
    if (bstart_dev != nullptr) {
        k_listf_write<<<B, LF_T, 0, st>>>(flags_dev, n, total, chunk, cnt, bstart_dev, bsize_dev);
        rc = make_bucket_sizes(bstart_dev, counts_dev, n, bsize_dev, btab_dev, table_ids_dev, st);
        if (rc) return rc;
    }
    QS_CHECK_LAUNCH("list buckets (flags)");
    return QS_OK;
}

}  // extern "C"
