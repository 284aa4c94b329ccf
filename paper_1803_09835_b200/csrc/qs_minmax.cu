// Min-Max hash signatures on sm_100a (integer ALU; no tensor-core shape).
//
// Reference: minmax_hash.py:73-128 (mapping, row split) and _sigcore.pyx:32-85
// (element-major kernel: running min/max over all t*k/2 mapping columns for
// every set bit, K*t*k/2 64-bit compare-selects per fingerprint).
//
// B200 design — probe MinHash: the plan stores, per hash column f, the element
// indices in ascending mapping-value order.  For a fingerprint held as a d-bit
// bitmap in shared memory, min_x V[x, f] is the value of the FIRST element of
// that order present in the bitmap, and the max is the last one.  With K of d
// bits set the expected number of probes per column is d/K (≈10 at cfg1)
// instead of K compare-selects (400): the same outputs, bit for bit, because
// the plan is built from the mapping values themselves (ties share a value).
#include <mutex>

#include "qs_common.cuh"

namespace qs {

// -------------------------------------------------------------- mapping
__global__ void k_gen_mapping(uint64_t* __restrict__ v, uint32_t d, uint32_t F, uint64_t seed) {
    uint64_t total = (uint64_t)d * F;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = i / F, j = i - x * F;
        v[i] = fmix64(((x + 1ULL) * GOLDEN64) ^ (seed + j));
    }
}

// ----------------------------------------------------------------- plan
constexpr uint32_t PLAN_MAX_D = 16384;  // smem bitonic sort capacity (192 KB)

// Plan layout, probe-sequence-major so one probe sequence walks consecutive
// addresses (L1-resident prefixes): order[side][f][r], svals[side][f][r] with
// side 0 = ascending value order (minimum probes), side 1 = descending (maximum);
// svals holds fmix64(value), the only form the combine step uses.
static inline size_t plan_order_bytes(uint32_t d, uint32_t F) {
    return (((size_t)2 * d * F * sizeof(uint16_t)) + 255) & ~(size_t)255;
}
// The first PLAN_BLK ranks of every probe sequence again, rank-block-major:
// blk[b][seq] = ranks 8b .. 8b + 7 of sequence seq (16 bytes).  Lanes of a warp
// mostly sit in the first blocks of neighbouring sequences, so these loads
// coalesce where the sequence-major rows scatter over 32 lines.
constexpr uint32_t PLAN_BLK = 32;
static inline size_t plan_blk_offset(uint32_t d, uint32_t F) {
    return plan_order_bytes(d, F) + (size_t)2 * d * F * sizeof(uint64_t);
}

// One CTA per hash column: bitonic sort of (value, element) in shared memory,
// then write both probe directions of the column into the plan.
__global__ void __launch_bounds__(1024) k_plan(const uint64_t* __restrict__ v, uint32_t d,
                                               uint32_t F, uint32_t dpad,
                                               uint16_t* __restrict__ order,
                                               uint64_t* __restrict__ svals,
                                               uint16_t* __restrict__ blk) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* key = (uint64_t*)smem;
    uint32_t* idx = (uint32_t*)(key + dpad);
    const uint32_t f = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < dpad; i += blockDim.x) {
        if (i < d) {
            key[i] = v[(uint64_t)i * F + f];
            idx[i] = i;
        } else {
            key[i] = ~0ULL;
            idx[i] = 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    for (uint32_t k = 2; k <= dpad; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < dpad; i += blockDim.x) {
                uint32_t l = i ^ j;
                if (l > i) {
                    bool up = (i & k) == 0;
                    uint64_t a = key[i], b = key[l];
                    uint32_t ia = idx[i], ib = idx[l];
                    bool gt = (a > b) || (a == b && ia > ib);
                    if (gt == up) {
                        key[i] = b; key[l] = a;
                        idx[i] = ib; idx[l] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (blk != nullptr)
        for (uint32_t r = threadIdx.x; r < PLAN_BLK && r < d; r += blockDim.x) {
            blk[((uint64_t)(r >> 3) * 2 * F + f) * 8 + (r & 7)] = (uint16_t)idx[r];
            blk[((uint64_t)(r >> 3) * 2 * F + F + f) * 8 + (r & 7)] = (uint16_t)idx[d - 1 - r];
        }
    for (uint32_t r = threadIdx.x; r < d; r += blockDim.x) {
        const uint64_t up = (uint64_t)f * d + r, down = ((uint64_t)F + f) * d + r;
        // the combine step only ever uses fmix64(value): store it pre-mixed
        order[up] = (uint16_t)idx[r];
        svals[up] = fmix64(key[r]);
        order[down] = (uint16_t)idx[d - 1 - r];
        svals[down] = fmix64(key[d - 1 - r]);
    }
}

// ------------------------------------------------------------ signatures
__device__ __forceinline__ uint64_t mix_key(uint64_t s) { return fmix64(s ^ GOLDEN64); }

// One warp per fingerprint row (grid-stride).  Shared memory per warp: the
// d-bit bitmap and the rank at which each of the 2F probe sequences hit.  The
// probe loop only touches the (L1-resident) prefixes of the order array; the
// hit values are gathered afterwards with independent loads.
template <bool SEARCH>
__global__ void __launch_bounds__(256) k_signatures(
    const uint32_t* __restrict__ bits, uint64_t n, uint32_t K,
    const uint16_t* __restrict__ order, const uint64_t* __restrict__ svals, uint32_t d,
    uint32_t F, uint32_t t, uint32_t kh, uint64_t* __restrict__ sigs,
    uint64_t* __restrict__ keys, uint64_t* __restrict__ rkeys, uint32_t* __restrict__ tags,
    uint32_t* __restrict__ bad, uint64_t row0, uint64_t row_end,
    const uint4* __restrict__ blk) {
    // rows [row0, row_end) of an n-row layout (n: the stride of keys / tags)
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t words = (d + 31) >> 5;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per_warp = ((words * 4 + 15) & ~15u) + ((2 * F * 2 + 15) & ~15u);
    uint32_t* bm = (uint32_t*)(smem + warp * per_warp);
    uint16_t* rk = (uint16_t*)((unsigned char*)bm + ((words * 4 + 15) & ~15u));
    const uint64_t gwarp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t W = (t + 31) >> 5;
    const bool vec = (K % 4 == 0) && ((((uintptr_t)bits) & 15) == 0);

    for (uint64_t row = row0 + gwarp; row < row_end; row += nwarps) {
        for (uint32_t w = lane; w < words; w += 32) bm[w] = 0u;
        __syncwarp();
        const uint32_t* rb = bits + row * K;
        uint32_t badrow = 0;
        if (vec) {
            const uint4* rb4 = (const uint4*)rb;
            for (uint32_t q = lane; q < K / 4; q += 32) {
                uint4 x = __ldg(rb4 + q);
                uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (xs[e] < d) atomicOr(&bm[xs[e] >> 5], 1u << (xs[e] & 31));
                    else badrow = 1;
                }
            }
        } else {
            for (uint32_t q = lane; q < K; q += 32) {
                uint32_t x = __ldg(rb + q);
                if (x < d) atomicOr(&bm[x >> 5], 1u << (x & 31));
                else badrow = 1;
            }
        }
        if (__any_sync(0xffffffffu, badrow) && lane == 0) atomicExch(bad, 1u);
        __syncwarp();
        // merged probe loop: lane walks its columns seq = lane, lane+32, ... < 2F
        // (seq < F: minimum side, else maximum), eight ranks per step when the
        // plan rows are 16-byte aligned (d % 8 == 0)
        uint32_t seq = lane, r = 0;
        const uint16_t* ord = order + (uint64_t)seq * d;
        if ((d & 7) == 0) {
            while (seq < 2 * F) {
                const uint4 v = (blk != nullptr && r < PLAN_BLK)
                                    ? __ldg(blk + (r >> 3) * 2 * F + seq)
                                    : __ldg((const uint4*)(ord + r));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t h = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t xa = w[e] & 0xFFFFu, xb = w[e] >> 16;
                    h |= ((bm[xa >> 5] >> (xa & 31)) & 1u) << (2 * e);
                    h |= ((bm[xb >> 5] >> (xb & 31)) & 1u) << (2 * e + 1);
                }
                r += 8;
                QS_DASSERT(seq < 2 * F);
                if (h || r >= d) {  // r >= d only when every bit was invalid
                    rk[seq] = h ? (uint16_t)(r - 8 + __ffs(h) - 1) : (uint16_t)0;
                    seq += 32;
                    r = 0;
                    ord += (uint64_t)32 * d;
                }
            }
        } else {
            while (seq < 2 * F) {
                const uint32_t x = __ldg(ord + r);
                if ((bm[x >> 5] >> (x & 31)) & 1u) {
                    rk[seq] = (uint16_t)r;
                    seq += 32;
                    r = 0;
                    ord += (uint64_t)32 * d;
                } else if (++r >= d) {
                    rk[seq] = 0;
                    seq += 32;
                    r = 0;
                    ord += (uint64_t)32 * d;
                }
            }
        }
        __syncwarp();
        for (uint32_t wr = 0; wr < W; ++wr) {
            const uint32_t i = wr * 32 + lane;
            uint64_t acc = 0;
            if (i < t) {
                for (uint32_t j = 0; j < kh; ++j) {
                    const uint32_t sq = i * kh + j;
                    acc = combine1_mixed(acc, __ldg(svals + (uint64_t)sq * d + rk[sq]));
                }
                for (uint32_t j = 0; j < kh; ++j) {
                    const uint32_t sq = F + i * kh + j;
                    acc = combine1_mixed(acc, __ldg(svals + (uint64_t)sq * d + rk[sq]));
                }
                if (sigs) sigs[row * t + i] = acc;
            }
            if (SEARCH) {
                const uint64_t key = mix_key(acc);
                if (i < t) {
                    if (keys) keys[(uint64_t)i * n + row] = key;
                    rkeys[row * t + i] = key;
                }
                const uint32_t tag = (uint32_t)key & 0xFFFFu;
                uint32_t plane = 0;
#pragma unroll
                for (int b = 0; b < 16; ++b) {
                    uint32_t word = __ballot_sync(0xffffffffu, (i < t) && ((tag >> b) & 1u));
                    if (lane == (uint32_t)b) plane = word;
                }
                if (lane < 16) tags[((uint64_t)(lane >> 3) * n + row) * W * 8 + wr * 8 + (lane & 7)] = plane;
            }
        }
        __syncwarp();
    }
}

static size_t sig_smem_per_warp(uint32_t d, uint32_t F) {
    uint32_t words = (d + 31) >> 5;
    return ((words * 4 + 15) & ~15u) + (((size_t)2 * F * 2 + 15) & ~(size_t)15);
}


// Plan-free Min-Max for d > PLAN_MAX_D (the probe plan's u16 element order and
// shared-memory sort stop there): the reference's own loop (_sigcore.pyx:60-75)
// — per row, elementwise min/max of the mapping rows of its K set bits, one
// warp per row, lanes over hash columns (coalesced 8-byte loads of a mapping
// row), then the same fold and search-layout epilogue as k_signatures.
template <bool SEARCH>
__global__ void __launch_bounds__(128) k_signatures_direct(
    const uint32_t* __restrict__ bits, uint64_t n, uint32_t K, const uint64_t* __restrict__ values,
    uint32_t d, uint32_t F, uint32_t t, uint32_t kh, uint64_t* __restrict__ sigs,
    uint64_t* __restrict__ keys, uint64_t* __restrict__ rkeys, uint32_t* __restrict__ tags,
    uint32_t* __restrict__ bad, uint64_t row_lo, uint64_t row_hi) {
    extern __shared__ __align__(16) uint64_t dsm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* mn = dsm + (uint64_t)warp * 2 * F;
    uint64_t* mx = mn + F;
    const uint32_t W = (t + 31) >> 5;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t row = row_lo + blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp; row < row_hi;
         row += nw) {
        const uint32_t* br = bits + row * K;
        bool badrow = false;
        for (uint32_t f0 = 0; f0 < F; f0 += 32) {
            const uint32_t f = f0 + lane;
            uint64_t lo = ~0ull, hi = 0;
            for (uint32_t k = 0; k < K; ++k) {
                uint32_t x = __ldg(br + k);
                if (x >= d) {
                    badrow = true;
                    x = 0;
                }
                if (f < F) {
                    const uint64_t v = __ldg(values + (uint64_t)x * F + f);
                    lo = v < lo ? v : lo;
                    hi = v > hi ? v : hi;
                }
            }
            if (f < F) {
                mn[f] = lo;
                mx[f] = hi;
            }
        }
        if (__any_sync(0xffffffffu, badrow) && lane == 0) atomicExch(bad, 1u);
        __syncwarp();
        for (uint32_t wr = 0; wr < W; ++wr) {
            const uint32_t i = wr * 32 + lane;
            uint64_t acc = 0;
            if (i < t) {
                for (uint32_t j = 0; j < kh; ++j) acc = combine1(acc, mn[i * kh + j]);
                for (uint32_t j = 0; j < kh; ++j) acc = combine1(acc, mx[i * kh + j]);
                if (sigs) sigs[row * t + i] = acc;
            }
            if (SEARCH) {
                const uint64_t key = mix_key(acc);
                if (i < t) {
                    if (keys) keys[(uint64_t)i * n + row] = key;
                    rkeys[row * t + i] = key;
                }
                const uint32_t tag = (uint32_t)key & 0xFFFFu;
                uint32_t plane = 0;
#pragma unroll
                for (int b = 0; b < 16; ++b) {
                    uint32_t word = __ballot_sync(0xffffffffu, (i < t) && ((tag >> b) & 1u));
                    if (lane == (uint32_t)b) plane = word;
                }
                if (lane < 16) tags[((uint64_t)(lane >> 3) * n + row) * W * 8 + wr * 8 + (lane & 7)] = plane;
            }
        }
        __syncwarp();
    }
}

static int launch_direct(bool search, const uint32_t* bits, uint64_t n, uint32_t K,
                         const uint64_t* values, uint32_t d, uint32_t t, uint32_t kh,
                         uint64_t* sigs, uint64_t* keys, uint64_t* rkeys, uint32_t* tags,
                         uint32_t* bad, cudaStream_t st, uint64_t row0, uint64_t nrows) {
    const uint32_t F = t * kh;
    const size_t smem = (size_t)4 * 2 * F * 8;
    QS_ARG(smem <= 200 * 1024, "t*k too large for the signature kernel (F=%u)", F);
    const unsigned grid = qs_blocks((nrows + 3) / 4, 1, 148 * 16);
    if (search) {
        QS_CUDA(cudaFuncSetAttribute(k_signatures_direct<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
        k_signatures_direct<true><<<grid, 128, smem, st>>>(bits, n, K, values, d, F, t, kh, sigs, keys,
                                                           rkeys, tags, bad, row0, row0 + nrows);
    } else {
        QS_CUDA(cudaFuncSetAttribute(k_signatures_direct<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
        k_signatures_direct<false><<<grid, 128, smem, st>>>(bits, n, K, values, d, F, t, kh, sigs,
                                                            nullptr, nullptr, nullptr, bad, row0,
                                                            row0 + nrows);
    }
    QS_CHECK_LAUNCH("k_signatures_direct");
    return QS_OK;
}

static int launch_signatures(bool search, const uint32_t* bits, uint64_t n, uint32_t K,
                             const void* plan, uint32_t d, uint32_t t, uint32_t kh,
                             uint64_t* sigs, uint64_t* keys, uint64_t* rkeys, uint32_t* tags,
                             uint32_t* bad, cudaStream_t st, uint64_t row0 = 0,
                             uint64_t nrows = ~0ull) {
    if (nrows == ~0ull) nrows = n - row0;
    QS_ARG(row0 <= n && nrows <= n - row0, "row range out of bounds");
    QS_ARG(K >= 1, "fingerprints must have at least one set bit");
    QS_ARG(d >= 1, "d must be >= 1");
    QS_ARG(t >= 1 && kh >= 1, "t and k/2 must be >= 1");
    if (nrows == 0) return QS_OK;
    if (d > PLAN_MAX_D)  // the "plan" is a copy of the mapping values (qs_minmax_plan)
        return launch_direct(search, bits, n, K, (const uint64_t*)plan, d, t, kh, sigs, keys,
                             rkeys, tags, bad, st, row0, nrows);
    const uint32_t F = t * kh;
    const uint16_t* order = (const uint16_t*)plan;
    const uint64_t* svals = (const uint64_t*)((const unsigned char*)plan + plan_order_bytes(d, F));
    const uint4* blk = d >= PLAN_BLK && (d & 7) == 0
                           ? (const uint4*)((const unsigned char*)plan + plan_blk_offset(d, F))
                           : nullptr;
    size_t per_warp = sig_smem_per_warp(d, F);
    int warps = 8;
    while (warps > 1 && per_warp * warps > 200 * 1024) warps >>= 1;
    QS_ARG(per_warp <= 220 * 1024, "t*k too large for the signature kernel (F=%u)", F);
    size_t smem = per_warp * warps;
    unsigned threads = warps * 32;
    uint64_t want = (nrows + warps - 1) / warps;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (search) {
        QS_CUDA(cudaFuncSetAttribute(k_signatures<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_signatures<true>, threads, smem);
    } else {
        QS_CUDA(cudaFuncSetAttribute(k_signatures<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_signatures<false>, threads, smem);
    }
    if (per_sm < 1) per_sm = 1;
    uint64_t cap = (uint64_t)sms * per_sm * 4;
    unsigned grid = (unsigned)(want < cap ? want : cap);
    if (search)
        k_signatures<true><<<grid, threads, smem, st>>>(bits, n, K, order, svals, d, F, t, kh,
                                                         sigs, keys, rkeys, tags, bad, row0,
                                                         row0 + nrows, blk);
    else
        k_signatures<false><<<grid, threads, smem, st>>>(bits, n, K, order, svals, d, F, t, kh,
                                                          sigs, nullptr, nullptr, nullptr, bad,
                                                          row0, row0 + nrows, blk);
    QS_CHECK_LAUNCH("k_signatures");
    return QS_OK;
}

}  // namespace qs

using namespace qs;


// persistent state of qs_gen_signatures_range (host plugin entry)
struct GsrCtx {
    int dev = -1;
    cudaStream_t st = nullptr;
    uint64_t *dv = nullptr, *dout = nullptr;
    uint32_t *dbits = nullptr, *dbad = nullptr;
    void* plan = nullptr;
    size_t dv_cap = 0, plan_cap = 0, dbits_cap = 0, dout_cap = 0, dbad_cap = 0;
    const uint64_t* key_values = nullptr;
    uint32_t key_d = 0, key_F = 0;
    uint64_t key_digest = 0;
    int ensure(void** p, size_t* cap, size_t bytes) {
        if (*cap >= bytes && *p) return QS_OK;
        if (*p) cudaFree(*p);
        *p = nullptr;
        *cap = 0;
        const cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) return qs::cuda_status(e, "cudaMalloc");
        *cap = bytes;
        if (p == (void**)&dv || p == &plan) key_values = nullptr;  // contents lost
        return QS_OK;
    }
    void release() {
        if (st) cudaStreamDestroy(st);
        for (void* q : {(void*)dv, (void*)dout, (void*)dbits, (void*)dbad, plan})
            if (q) cudaFree(q);
        *this = GsrCtx();
    }
};

// digest of a mapping: its shape plus every 97th value (the mapping is
// generated, never edited in place; a different array gets a new upload)
static uint64_t values_digest(const uint64_t* v, uint64_t count) {
    uint64_t h = count * 0x9E3779B97F4A7C15ULL;
    for (uint64_t i = 0; i < count; i += 97) h = qs::fmix64(h ^ v[i]);
    return qs::fmix64(h ^ v[count - 1]);
}

extern "C" {

int qs_gen_hash_mapping(uint64_t* values_dev, uint32_t d, uint32_t n_funcs, uint64_t seed,
                        void* stream) {
    QS_ARG(d >= 1 && n_funcs >= 1, "d and n_funcs must be >= 1");
    uint64_t total = (uint64_t)d * n_funcs;
    k_gen_mapping<<<qs_blocks(total, 256), 256, 0, (cudaStream_t)stream>>>(values_dev, d, n_funcs, seed);
    QS_CHECK_LAUNCH("k_gen_mapping");
    return QS_OK;
}

size_t qs_minmax_plan_bytes(uint32_t d, uint32_t n_funcs) {
    if (d > PLAN_MAX_D) return (size_t)d * n_funcs * 8;  // plan-free path: the values themselves
    return plan_blk_offset(d, n_funcs) + (size_t)2 * n_funcs * PLAN_BLK * sizeof(uint16_t);
}

int qs_minmax_plan(const uint64_t* values_dev, uint32_t d, uint32_t n_funcs, void* plan_dev,
                   void* stream) {
    QS_ARG(d >= 1, "d must be >= 1");
    QS_ARG(n_funcs >= 1, "n_funcs must be >= 1");
    if (d > PLAN_MAX_D) {  // plan-free (direct) signatures read the values
        QS_CUDA(cudaMemcpyAsync(plan_dev, values_dev, (size_t)d * n_funcs * 8,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "copy values");
        return QS_OK;
    }
    uint32_t dpad = 1;
    while (dpad < d) dpad <<= 1;
    if (dpad < 2) dpad = 2;
    size_t smem = (size_t)dpad * (sizeof(uint64_t) + sizeof(uint32_t));
    QS_CUDA(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "smem attr");
    uint16_t* order = (uint16_t*)plan_dev;
    uint64_t* svals = (uint64_t*)((unsigned char*)plan_dev + plan_order_bytes(d, n_funcs));
    unsigned threads = dpad >= 1024 ? 1024 : dpad;
    uint16_t* blk = d >= PLAN_BLK && (d & 7) == 0
                        ? (uint16_t*)((unsigned char*)plan_dev + plan_blk_offset(d, n_funcs))
                        : nullptr;
    k_plan<<<n_funcs, threads, smem, (cudaStream_t)stream>>>(values_dev, d, n_funcs, dpad, order, svals,
                                                             blk);
    QS_CHECK_LAUNCH("k_plan");
    return QS_OK;
}

int qs_minmax_signatures(const uint32_t* bits_dev, uint64_t n, uint32_t K, const void* plan_dev,
                         uint32_t d, uint32_t t, uint32_t k_half, uint64_t* out_dev,
                         uint32_t* bad_dev, void* stream) {
    return launch_signatures(false, bits_dev, n, K, plan_dev, d, t, k_half, out_dev, nullptr,
                             nullptr, nullptr, bad_dev, (cudaStream_t)stream);
}

int qs_minmax_signatures_search(const uint32_t* bits_dev, uint64_t n, uint32_t K,
                                const void* plan_dev, uint32_t d, uint32_t t, uint32_t k_half,
                                uint64_t* sigs_dev, uint64_t* keys_dev, uint64_t* rkeys_dev,
                                uint32_t* tags_dev, uint32_t* bad_dev, void* stream) {
    return launch_signatures(true, bits_dev, n, K, plan_dev, d, t, k_half, sigs_dev, keys_dev,
                             rkeys_dev, tags_dev, bad_dev, (cudaStream_t)stream);
}

int qs_minmax_signatures_search_rows(const uint32_t* bits_dev, uint64_t n, uint64_t row0,
                                     uint64_t nrows, uint32_t K, const void* plan_dev, uint32_t d,
                                     uint32_t t, uint32_t k_half, uint64_t* sigs_dev,
                                     uint64_t* keys_dev, uint64_t* rkeys_dev, uint32_t* tags_dev,
                                     uint32_t* bad_dev, void* stream) {
    return launch_signatures(true, bits_dev, n, K, plan_dev, d, t, k_half, sigs_dev, keys_dev,
                             rkeys_dev, tags_dev, bad_dev, (cudaStream_t)stream, row0, nrows);
}

int qs_gen_signatures_range(const uint32_t* bits, uint64_t n_rows, uint32_t K,
                            const uint64_t* values, uint32_t d, uint32_t F, int32_t t,
                            int32_t k_half, uint64_t* out, uint64_t start, uint64_t stop) {
    QS_ARG(t >= 1 && k_half >= 1 && (uint64_t)t * (uint64_t)k_half == F,
           "mapping width does not match t * k_half");
    QS_ARG(K >= 1, "fingerprints must have at least one set bit");
    QS_ARG(start <= stop && stop <= n_rows, "row range out of bounds");
    if (stop == start) return QS_OK;
    // The reference calls this once per worker chunk with the same mapping
    // (minmax_hash.py:113-128): the stream, the device buffers and the
    // uploaded mapping + probe plan persist across calls (keyed by the
    // mapping's address, shape and a strided digest of its values); calls
    // are serialised by a mutex (the device serialises them anyway).
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static GsrCtx ctx;
    int dev = 0;
    QS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    if (ctx.st == nullptr || ctx.dev != dev) {
        ctx.release();
        ctx.dev = dev;
        QS_CUDA(cudaStreamCreateWithFlags(&ctx.st, cudaStreamNonBlocking), "stream");
    }
    cudaStream_t st = ctx.st;
    const uint64_t rows = stop - start;
    const uint64_t chunk = rows < (1u << 20) ? rows : (1u << 20);
    const size_t vb = (size_t)d * F * 8, pb = qs_minmax_plan_bytes(d, F);
    int rc = QS_OK;
    if ((rc = ctx.ensure((void**)&ctx.dv, &ctx.dv_cap, vb)) ||
        (rc = ctx.ensure(&ctx.plan, &ctx.plan_cap, pb)) ||
        (rc = ctx.ensure((void**)&ctx.dbits, &ctx.dbits_cap, chunk * K * 4)) ||
        (rc = ctx.ensure((void**)&ctx.dout, &ctx.dout_cap, chunk * (uint64_t)t * 8)) ||
        (rc = ctx.ensure((void**)&ctx.dbad, &ctx.dbad_cap, 4)))
        return rc;
    const uint64_t digest = values_digest(values, (uint64_t)d * F);
    if (!(ctx.key_values == values && ctx.key_d == d && ctx.key_F == F && ctx.key_digest == digest)) {
        QS_CUDA(cudaMemcpyAsync(ctx.dv, values, vb, cudaMemcpyHostToDevice, st), "H2D mapping");
        rc = qs_minmax_plan(ctx.dv, d, F, ctx.plan, st);
        if (rc) {
            ctx.key_values = nullptr;
            return rc;
        }
        ctx.key_values = values;
        ctx.key_d = d;
        ctx.key_F = F;
        ctx.key_digest = digest;
    }
    QS_CUDA(cudaMemsetAsync(ctx.dbad, 0, 4, st), "memset");
    for (uint64_t a = start; rc == QS_OK && a < stop; a += chunk) {
        uint64_t m = (stop - a) < chunk ? (stop - a) : chunk;
        QS_CUDA(cudaMemcpyAsync(ctx.dbits, bits + a * K, m * K * 4, cudaMemcpyHostToDevice, st), "H2D");
        rc = qs_minmax_signatures(ctx.dbits, m, K, ctx.plan, d, (uint32_t)t, (uint32_t)k_half,
                                  ctx.dout, ctx.dbad, st);
        if (rc == QS_OK)
            QS_CUDA(cudaMemcpyAsync(out + a * t, ctx.dout, m * (uint64_t)t * 8,
                                    cudaMemcpyDeviceToHost, st), "D2H");
    }
    uint32_t hbad = 0;
    if (rc == QS_OK) QS_CUDA(cudaMemcpyAsync(&hbad, ctx.dbad, 4, cudaMemcpyDeviceToHost, st), "D2H");
    const cudaError_t e = cudaStreamSynchronize(st);
    if (rc == QS_OK && e != cudaSuccess) rc = cuda_status(e, "qs_gen_signatures_range");
    if (rc == QS_OK && hbad) {
        set_error("fingerprint bit index out of range for mapping");
        rc = QS_ERR_DATA;
    }
    return rc;
}

}  // extern "C"
