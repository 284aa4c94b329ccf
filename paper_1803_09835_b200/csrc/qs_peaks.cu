// CUDA-core throughput microbenchmarks (the FP64 / FP32 / 64-bit
// integer peaks are not in MEASURED_PEAKS.json, so the fingerprint and
// Min-Max rooflines are taken against these measured numbers).
//
// Each thread runs 8 independent dependency chains (enough ILP to keep the
// pipe busy) for `iters` iterations; the grid covers every SM several times.
// The result is folded into one store per thread so nothing is optimised away.
#include "qs_common.cuh"

namespace qs {

constexpr int PK_CHAINS = 8;
constexpr int PK_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(PK_THREADS) k_peak_fma(T* __restrict__ out, uint32_t iters, T b, T c) {
    T a[PK_CHAINS];
#pragma unroll
    for (int k = 0; k < PK_CHAINS; ++k) a[k] = (T)(threadIdx.x + k);
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < PK_CHAINS; ++k) a[k] = fma(a[k], b, c);
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < PK_CHAINS; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 64-bit min/max compare-selects (the Min-Max reference's inner operation)
__global__ void __launch_bounds__(PK_THREADS) k_peak_minmax64(uint64_t* __restrict__ out, uint32_t iters,
                                                             uint64_t x0, uint64_t step) {
    uint64_t mn[PK_CHAINS / 2], mx[PK_CHAINS / 2];
    uint64_t x = x0 + threadIdx.x;
#pragma unroll
    for (int k = 0; k < PK_CHAINS / 2; ++k) {
        mn[k] = ~0ull - k;
        mx[k] = k;
    }
    for (uint32_t i = 0; i < iters; ++i) {
        x += step;
#pragma unroll
        for (int k = 0; k < PK_CHAINS / 2; ++k) {
            const uint64_t v = x ^ (uint64_t)k;
            mn[k] = v < mn[k] ? v : mn[k];
            mx[k] = v > mx[k] ? v : mx[k];
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < PK_CHAINS / 2; ++k) s ^= mn[k] ^ mx[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// The north-star pair-count table (BASELINE.json north_star: "collision
// counting in an HBM open-addressed hash table"), measured rather than built:
// every candidate (pair, table) hit inserts its 64-bit pair key into an
// open-addressed table (linear probing, atomicCAS on the key, atomicAdd on a
// 32-bit count).  Hit i inserts key fmix64(seed ^ (i mod distinct)), so each
// of `distinct` pairs is hit n / distinct times in scattered order — the
// access pattern of counting the hits of a bucket enumeration.
__global__ void __launch_bounds__(256) k_pair_table(uint64_t n, uint64_t distinct,
                                                   unsigned long long* __restrict__ keys,
                                                   uint32_t* __restrict__ cnt, uint64_t mask,
                                                   unsigned long long* __restrict__ probes) {
    unsigned long long pr = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = fmix64(0x5851F42D4C957F2Dull ^ (i % distinct)) | 1ull;
        uint64_t slot = fmix64(k) & mask;
        while (true) {
            ++pr;
            const unsigned long long old = atomicCAS(keys + slot, 0ull, k);
            if (old == 0ull || old == k) {
                atomicAdd(cnt + slot, 1u);
                break;
            }
            slot = (slot + 1) & mask;
        }
    }
    atomicAdd(probes, pr);
}

}  // namespace qs

using namespace qs;

extern "C" {

// Launches microbenchmark `kind` on `stream` (0: FP64 FMA, 1: FP32 FMA,
// 2: 64-bit min/max) over `blocks` x 256 threads, `iters` iterations of 8
// operations per thread; *ops_out = operations performed (an FMA counts as
// one operation = two flops; a min or a max as one compare-select).  The
// caller times the launch (CUDA events on the same stream).
int qs_peak_launch(int kind, uint32_t blocks, uint32_t iters, void* scratch_dev,
                   double* ops_out, void* stream) {
    QS_ARG(kind >= 0 && kind <= 2, "kind must be 0 (fp64 fma), 1 (fp32 fma) or 2 (u64 min/max)");
    QS_ARG(blocks >= 1 && iters >= 1, "blocks and iters must be >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    if (kind == 0)
        k_peak_fma<double><<<blocks, PK_THREADS, 0, st>>>((double*)scratch_dev, iters, 0.999999,
                                                           1e-7);
    else if (kind == 1)
        k_peak_fma<float><<<blocks, PK_THREADS, 0, st>>>((float*)scratch_dev, iters, 0.9999f, 1e-5f);
    else
        k_peak_minmax64<<<blocks, PK_THREADS, 0, st>>>((uint64_t*)scratch_dev, iters,
                                                        0x9E3779B97F4A7C15ull, 0xD1B54A32D192ED03ull);
    QS_CHECK_LAUNCH("k_peak");
    *ops_out = (double)blocks * PK_THREADS * iters * PK_CHAINS;
    return QS_OK;
}

// One launch of the pair-count-table insert microbenchmark above: n inserts of
// `distinct` keys into a table of `slots` (power of two) 12-byte slots at
// table_dev (keys [slots] u64 then counts [slots] u32, zeroed by the caller);
// probes_dev (u64, zeroed) receives the probe count.  Time it with events.
int qs_bench_pair_table(uint64_t n, uint64_t distinct, void* table_dev, uint64_t slots,
                        uint64_t* probes_dev, void* stream) {
    QS_ARG(slots >= 2 && (slots & (slots - 1)) == 0, "slots must be a power of two");
    QS_ARG(distinct >= 1 && distinct < slots, "distinct keys must fit the table");
    unsigned long long* keys = (unsigned long long*)table_dev;
    uint32_t* cnt = (uint32_t*)(keys + slots);
    k_pair_table<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(n, distinct, keys, cnt, slots - 1,
                                                             (unsigned long long*)probes_dev);
    QS_CHECK_LAUNCH("k_pair_table");
    return QS_OK;
}

}  // extern "C"
