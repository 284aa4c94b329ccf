// Shared device/host helpers for the quakescan-b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/quakescan_b200.h"

namespace qs {

constexpr uint64_t GOLDEN64 = 0x9E3779B97F4A7C15ULL;

// Murmur3 64-bit finalizer (reference _sigcore.pyx:18-24).
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDULL;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ULL;
    x ^= x >> 33;
    return x;
}

// One boost-style fold step (reference _sigcore.pyx:27-29).
__host__ __device__ __forceinline__ uint64_t combine1(uint64_t acc, uint64_t w) {
    return acc ^ (fmix64(w) + GOLDEN64 + (acc << 6) + (acc >> 2));
}

// The same step with fmix64(w) precomputed (the Min-Max plan stores mixed values).
__host__ __device__ __forceinline__ uint64_t combine1_mixed(uint64_t acc, uint64_t fw) {
    return acc ^ (fw + GOLDEN64 + (acc << 6) + (acc >> 2));
}

// Per-thread last error text, retrievable through qs_last_error().
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

}  // namespace qs

// Debug builds (make EXTRA=-DQS_DEBUG_CHECKS, the sanitizer substitute of
// DESIGN.md §3): device-side bounds assertions on the shared-memory and global
// indices of the asynchronous kernels; a failure traps the kernel.
#ifdef QS_DEBUG_CHECKS
#define QS_DASSERT(c)                                                                   \
    do {                                                                                \
        if (!(c)) {                                                                     \
            printf("QS_DASSERT %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,      \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                              \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define QS_DASSERT(c) \
    do {              \
    } while (0)
#endif

#define QS_CHECK_LAUNCH(what)                                              \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return qs::cuda_status(_e, what);           \
    } while (0)

#define QS_CUDA(call, what)                                                \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return qs::cuda_status(_e, what);           \
    } while (0)

#define QS_ARG(cond, ...)                                                  \
    do {                                                                   \
        if (!(cond)) {                                                     \
            qs::set_error(__VA_ARGS__);                                    \
            return QS_ERR_ARG;                                             \
        }                                                                  \
    } while (0)

#define QS_DATA(cond, ...)                                                 \
    do {                                                                   \
        if (!(cond)) {                                                     \
            qs::set_error(__VA_ARGS__);                                    \
            return QS_ERR_DATA;                                            \
        }                                                                  \
    } while (0)

static inline unsigned qs_blocks(uint64_t n, unsigned threads, unsigned cap = 148u * 32u) {
    uint64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}
