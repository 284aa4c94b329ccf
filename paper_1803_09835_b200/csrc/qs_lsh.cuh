// Device helpers shared by the LSH search translation units.
#pragma once

#include "qs_common.cuh"

namespace qs {

int radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t seg_len, uint32_t segments,
                     uint32_t key_bits, uint64_t* keys_alt, uint32_t* vals_alt, void* ws,
                     size_t ws_bytes, int* in_alt, cudaStream_t st, uint32_t bit_lo = 0,
                     uint32_t lo_bits = 32);
size_t radix_ws_bytes(uint64_t seg_len, uint32_t segments);
int radix_sort_pairs_to(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t seg_len,
                        uint32_t segments, uint32_t bit_lo, uint32_t key_bits, uint64_t* keys_out,
                        uint32_t* vals_out, uint64_t* keys_alt, uint32_t* vals_alt, void* ws,
                        size_t ws_bytes, cudaStream_t st);
int scan_u64(const uint64_t* in, uint64_t* out, uint64_t len, uint64_t* total, void* ws,
             cudaStream_t st);
size_t scan_ws_bytes(uint64_t len);
int num_sms();
int make_bucket_sizes(const uint64_t* bstart, const uint64_t* counts, uint64_t n, uint32_t* bsize,
                      uint32_t* btab, const uint32_t* table_ids, cudaStream_t st);

// bucket build by key-range bins + shared-memory bin sorts (qs_bucket_bins.cu)
size_t bucket_bins_ws_bytes(uint64_t n, uint32_t t);
int bucket_bins_build(const uint64_t* keys, uint64_t n, uint32_t t, uint32_t* sids, uint8_t* flags,
                      void* ws, size_t ws_bytes, cudaStream_t st);

__device__ __forceinline__ uint64_t mix_key(uint64_t s) { return fmix64(s ^ GOLDEN64); }

// partition index of fingerprint i: edges[k] <= i < edges[k+1]
__device__ __forceinline__ uint32_t part_of(const uint64_t* __restrict__ edges, uint32_t p,
                                            uint64_t i) {
    uint32_t lo = 0, hi = p;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(edges + mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

}  // namespace qs
