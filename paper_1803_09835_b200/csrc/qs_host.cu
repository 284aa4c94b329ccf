// Host <-> device transfer helpers of the end-to-end entry points.
//
// The reference's search_fingerprints / fingerprint_series take host numpy
// arrays (lsh_search.py:314-333, fingerprint.py:581-623); here the copy of
// those inputs is part of the call.  Three pieces keep it at the PCIe rate:
//   * qs_host_ptr_pinned: a caller's array that already lives in page-locked
//     memory is copied by DMA straight from where it lies (no staging pass);
//   * qs_host_pack_u16 + qs_bits_widen_u16: pageable (n, K) uint32 bit indices
//     are narrowed to uint16 while they are staged into pinned buffers (d <=
//     65535; larger values saturate to 65535 >= d and are flagged by the
//     signature kernel's range check like any other out-of-range index), so
//     both the staging writes and the DMA move half the bytes, and widened
//     again on the device;
//   * qs_host_pack_u12 + qs_bits_widen_u12: the same for d <= 4096 (the
//     BASELINE fingerprints) with 12-bit fields, 1.5 bytes per index instead of
//     2; a value above 4095 cannot be represented, so the pack reports it and the
//     caller sends that chunk through the uint16 route (whose saturation the
//     kernel flags);
//   * qs_host_pack_f32: a pageable float64 trace whose samples are all exactly
//     representable in float32 (a float32 recording coerced to float64, as
//     reference ingest.py:36 does) is narrowed the same way; the chain widens
//     float32 samples exactly, so the result is unchanged.  The first inexact
//     chunk makes the caller fall back to the float64 copy;
//   * qs_memcpy_h2d_async / qs_memcpy_d2h_async: plain cudaMemcpyAsync on the
//     caller's stream.
#include <immintrin.h>

#include "qs_common.cuh"

namespace qs {

// saturating uint32 -> uint16 narrow, 16 values per step (vpackusdw + a lane fix-up)
__attribute__((target("avx2"))) static uint64_t pack_u16_avx2(const uint32_t* src, uint16_t* dst,
                                                              uint64_t count) {
    const __m256i lim = _mm256_set1_epi32(0xFFFF);
    uint64_t i = 0;
    for (; i + 16 <= count; i += 16) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 8));
        a = _mm256_min_epu32(a, lim);  // packus treats its input as signed
        b = _mm256_min_epu32(b, lim);
        const __m256i p = _mm256_permute4x64_epi64(_mm256_packus_epi32(a, b), 0xD8);
        _mm256_storeu_si256((__m256i*)(dst + i), p);
    }
    return i;
}

// uint32 (< 4096) -> 12-bit fields, 8 values -> 12 bytes per step: value i of the
// stream occupies bits [12 i, 12 i + 12) (little endian).  Each 64-bit lane
// holds two values -> one 24-bit group; the three low bytes of the four lanes
// are gathered per 128-bit half and written with two overlapping 8-byte stores
// (the caller keeps one more group after the last step, so the 2 spare bytes
// stay inside this call's range).  *over accumulates the OR of every input.
__attribute__((target("avx2"))) static uint64_t pack_u12_avx2(const uint32_t* src, uint8_t* dst,
                                                              uint64_t count, uint32_t* over) {
    const __m256i m12 = _mm256_set1_epi64x(0xFFF);
    const __m256i shuf = _mm256_setr_epi8(0, 1, 2, 8, 9, 10, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                          0, 1, 2, 8, 9, 10, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
    __m256i acc = _mm256_setzero_si256();
    uint64_t i = 0;
    for (; i + 16 <= count; i += 8) {
        const __m256i v = _mm256_loadu_si256((const __m256i*)(src + i));
        acc = _mm256_or_si256(acc, v);
        const __m256i lo = _mm256_and_si256(v, m12);
        const __m256i hi = _mm256_slli_epi64(_mm256_and_si256(_mm256_srli_epi64(v, 32), m12), 12);
        const __m256i g = _mm256_shuffle_epi8(_mm256_or_si256(lo, hi), shuf);
        uint8_t* o = dst + (i / 8) * 12;
        _mm_storel_epi64((__m128i*)o, _mm256_castsi256_si128(g));
        _mm_storel_epi64((__m128i*)(o + 6), _mm256_extracti128_si256(g, 1));
    }
    const __m128i a = _mm_or_si128(_mm256_castsi256_si128(acc), _mm256_extracti128_si256(acc, 1));
    uint32_t t[4];
    _mm_storeu_si128((__m128i*)t, a);
    *over |= t[0] | t[1] | t[2] | t[3];
    return i;
}

// float64 -> float32 narrow with an exactness check (every value must widen
// back to itself; NaN, overflow and inexact values report 0)
__attribute__((target("avx2"))) static uint64_t pack_f32_avx2(const double* src, float* dst,
                                                              uint64_t count, int* exact) {
    __m256d ok = _mm256_castsi256_pd(_mm256_set1_epi64x(-1));
    uint64_t i = 0;
    for (; i + 8 <= count; i += 8) {
        const __m256d a = _mm256_loadu_pd(src + i), b = _mm256_loadu_pd(src + i + 4);
        const __m128 fa = _mm256_cvtpd_ps(a), fb = _mm256_cvtpd_ps(b);
        ok = _mm256_and_pd(ok, _mm256_cmp_pd(_mm256_cvtps_pd(fa), a, _CMP_EQ_OQ));
        ok = _mm256_and_pd(ok, _mm256_cmp_pd(_mm256_cvtps_pd(fb), b, _CMP_EQ_OQ));
        _mm_storeu_ps(dst + i, fa);
        _mm_storeu_ps(dst + i + 4, fb);
    }
    if (_mm256_movemask_pd(ok) != 0xF) *exact = 0;
    return i;
}

__global__ void k_widen_u16(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst,
                            uint64_t count8) {
    // 8 values per thread: one 16-byte load, two 16-byte stores
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count8;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs((const uint4*)src + i);
        uint4 a, b;
        a.x = v.x & 0xFFFFu; a.y = v.x >> 16; a.z = v.y & 0xFFFFu; a.w = v.y >> 16;
        b.x = v.z & 0xFFFFu; b.y = v.z >> 16; b.z = v.w & 0xFFFFu; b.w = v.w >> 16;
        ((uint4*)dst)[2 * i] = a;
        ((uint4*)dst)[2 * i + 1] = b;
    }
}

__global__ void k_widen_u16_tail(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst,
                                 uint64_t lo, uint64_t count) {
    const uint64_t i = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < count) dst[i] = src[i];
}

// 12-bit fields -> uint32, 8 values (three 32-bit words) per thread
__global__ void k_widen_u12(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                            uint64_t count8) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count8;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w0 = __ldcs(src + 3 * i), w1 = __ldcs(src + 3 * i + 1), w2 = __ldcs(src + 3 * i + 2);
        uint4 a, b;
        a.x = w0 & 0xFFFu;
        a.y = (w0 >> 12) & 0xFFFu;
        a.z = (w0 >> 24) | ((w1 & 0xFu) << 8);
        a.w = (w1 >> 4) & 0xFFFu;
        b.x = (w1 >> 16) & 0xFFFu;
        b.y = (w1 >> 28) | ((w2 & 0xFFu) << 4);
        b.z = (w2 >> 8) & 0xFFFu;
        b.w = w2 >> 20;
        ((uint4*)dst)[2 * i] = a;
        ((uint4*)dst)[2 * i + 1] = b;
    }
}

__global__ void k_widen_u12_tail(const uint8_t* __restrict__ src, uint32_t* __restrict__ dst,
                                 uint64_t lo, uint64_t count) {
    const uint64_t i = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < count) {
        const uint64_t bit = 12 * i, by = bit >> 3;
        const uint32_t two = (uint32_t)src[by] | ((uint32_t)src[by + 1] << 8);
        dst[i] = (bit & 4) ? (two >> 4) : (two & 0xFFFu);
    }
}

}  // namespace qs

extern "C" {

int qs_host_ptr_pinned(const void* host_ptr) {
    if (host_ptr == nullptr) return 0;
    cudaPointerAttributes a;
    const cudaError_t e = cudaPointerGetAttributes(&a, host_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();  // unknown to the driver: pageable
        return 0;
    }
    return a.type == cudaMemoryTypeHost ? 1 : 0;
}

int qs_host_pack_u16(const uint32_t* src_host, uint16_t* dst_host, uint64_t count) {
    uint64_t i0 = 0;
    if (__builtin_cpu_supports("avx2")) i0 = qs::pack_u16_avx2(src_host, dst_host, count);
    for (uint64_t i = i0; i < count; ++i) {
        const uint32_t v = src_host[i];
        dst_host[i] = (uint16_t)(v > 0xFFFFu ? 0xFFFFu : v);
    }
    return QS_OK;
}

int qs_host_pack_u12(const uint32_t* src_host, uint8_t* dst_host, uint64_t count, int* fits_out) {
    uint32_t over = 0;
    uint64_t i = 0;
    if (__builtin_cpu_supports("avx2")) i = qs::pack_u12_avx2(src_host, dst_host, count, &over);
    uint8_t* o = dst_host + (i / 2) * 3;  // i is a multiple of 8
    for (; i + 2 <= count; i += 2, o += 3) {
        const uint32_t a = src_host[i], b = src_host[i + 1];
        over |= a | b;
        o[0] = (uint8_t)a;
        o[1] = (uint8_t)(((a >> 8) & 0xFu) | ((b & 0xFu) << 4));
        o[2] = (uint8_t)(b >> 4);
    }
    if (i < count) {  // an odd count ends with a 2-byte field
        const uint32_t a = src_host[i];
        over |= a;
        o[0] = (uint8_t)a;
        o[1] = (uint8_t)((a >> 8) & 0xFu);
    }
    *fits_out = over <= 0xFFFu ? 1 : 0;
    return QS_OK;
}

int qs_host_pack_f32(const double* src_host, float* dst_host, uint64_t count, int* exact_out) {
    int exact = 1;
    uint64_t i0 = 0;
    if (__builtin_cpu_supports("avx2")) i0 = qs::pack_f32_avx2(src_host, dst_host, count, &exact);
    for (uint64_t i = i0; i < count; ++i) {
        const float f = (float)src_host[i];
        dst_host[i] = f;
        if (!((double)f == src_host[i])) exact = 0;
    }
    *exact_out = exact;
    return QS_OK;
}

int qs_bits_widen_u16(const uint16_t* src_dev, uint32_t* dst_dev, uint64_t count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (count == 0) return QS_OK;
    QS_ARG((((uintptr_t)src_dev) & 15) == 0 && (((uintptr_t)dst_dev) & 15) == 0,
           "widen: buffers must be 16-byte aligned");
    const uint64_t c8 = count / 8;
    if (c8) qs::k_widen_u16<<<qs_blocks(c8, 256, 148u * 16u), 256, 0, st>>>(src_dev, dst_dev, c8);
    if (count % 8)
        qs::k_widen_u16_tail<<<1, 32, 0, st>>>(src_dev, dst_dev, c8 * 8, count);
    QS_CHECK_LAUNCH("widen u16");
    return QS_OK;
}

int qs_bits_widen_u12(const uint8_t* src_dev, uint32_t* dst_dev, uint64_t count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (count == 0) return QS_OK;
    QS_ARG((((uintptr_t)src_dev) & 3) == 0 && (((uintptr_t)dst_dev) & 15) == 0,
           "widen u12: source must be 4-byte, destination 16-byte aligned");
    const uint64_t c8 = count / 8;
    if (c8)
        qs::k_widen_u12<<<qs_blocks(c8, 256, 148u * 16u), 256, 0, st>>>((const uint32_t*)src_dev, dst_dev, c8);
    if (count % 8) qs::k_widen_u12_tail<<<1, 32, 0, st>>>(src_dev, dst_dev, c8 * 8, count);
    QS_CHECK_LAUNCH("widen u12");
    return QS_OK;
}

int qs_memcpy_h2d_async(void* dst_dev, const void* src_host, size_t bytes, void* stream) {
    QS_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream),
            "cudaMemcpyAsync H2D");
    return QS_OK;
}

int qs_memcpy_d2h_async(void* dst_host, const void* src_dev, size_t bytes, void* stream) {
    QS_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
            "cudaMemcpyAsync D2H");
    return QS_OK;
}

}  // extern "C"
