// Channel combine and triplet sort on the device (the steps after the search,
// reference align.py:87-140).
//
// combine_channel_triplets merges per-channel triplet streams sorted by
// (dt, idx1), sums the table-match counts of equal window pairs and keeps the
// sums >= threshold.  Here: unpack all records to (dt << 32 | idx1, sim),
// one LSD radix sort over the concatenation, reduce-by-key over the sorted
// runs (heads sum their run), an exclusive scan of the kept flags and a
// scatter of the packed 20-byte records — the same output as the k-way heap
// merge, in the same (dt, idx1) order.
#include "qs_lsh.cuh"

namespace qs {

__global__ void k_tri_unpack(const uint32_t* __restrict__ rec, uint64_t n,
                             uint64_t* __restrict__ key, uint32_t* __restrict__ sim,
                             unsigned long long* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t* r = rec + i * 5;  // <u8 dt, <u8 idx1, <u4 sim
        const uint64_t dt = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
        const uint64_t i1 = (uint64_t)r[2] | ((uint64_t)r[3] << 32);
        if (dt >= (1ull << 32) || i1 >= (1ull << 32)) atomicAdd(bad, 1ULL);
        key[i] = (dt << 32) | (i1 & 0xFFFFFFFFull);
        sim[i] = r[4];
    }
}

// heads of equal-key runs: run sum, keep flag (threshold > 0) or 1 (sort only)
__global__ void k_tri_heads(const uint64_t* __restrict__ key, const uint32_t* __restrict__ sim,
                            uint64_t n, uint32_t threshold, uint64_t* __restrict__ flag,
                            uint64_t* __restrict__ sum) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[i];
        if (threshold == 0) {  // plain sort: every record kept as is
            flag[i] = 1;
            sum[i] = sim[i];
            continue;
        }
        if (i > 0 && key[i - 1] == k) {
            flag[i] = 0;
            continue;
        }
        uint64_t s = 0;
        for (uint64_t j = i; j < n && key[j] == k; ++j) s += sim[j];
        flag[i] = s >= threshold ? 1 : 0;
        sum[i] = s;
    }
}

__global__ void k_tri_emit(const uint64_t* __restrict__ key, const uint64_t* __restrict__ raw,
                           const uint64_t* __restrict__ off, const uint64_t* __restrict__ sum,
                           uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!raw[i]) continue;
        const uint64_t k = key[i];
        uint32_t* r = out + off[i] * 5;
        r[0] = (uint32_t)(k >> 32);
        r[1] = 0;
        r[2] = (uint32_t)k;
        r[3] = 0;
        r[4] = (uint32_t)sum[i];
    }
}

}  // namespace qs

using namespace qs;

extern "C" {

size_t qs_triplets_combine_ws_bytes(uint64_t n) {
    return (size_t)n * (8 + 4 + 8 + 4 + 8 + 8 + 8) + radix_ws_bytes(n, 1) + scan_ws_bytes(n) + 2048;
}

int qs_triplets_combine(const uint8_t* triplets_dev, uint64_t n, uint32_t threshold,
                        uint32_t key_bits, uint8_t* out_dev, uint64_t* count_dev, void* ws_dev,
                        size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(key_bits >= 1 && key_bits <= 64, "key_bits must be in [1, 64]");
    QS_ARG(ws_bytes >= qs_triplets_combine_ws_bytes(n), "combine workspace too small");
    if (n == 0) {
        QS_CUDA(cudaMemsetAsync(count_dev, 0, 8, st), "memset");
        return QS_OK;
    }
    unsigned char* w = (unsigned char*)ws_dev;
    auto take = [&](size_t bytes) {
        unsigned char* p = w;
        w = (unsigned char*)(((uintptr_t)(w + bytes) + 255) & ~(uintptr_t)255);
        return (void*)p;
    };
    uint64_t* key = (uint64_t*)take(n * 8);
    uint32_t* sim = (uint32_t*)take(n * 4);
    uint64_t* akey = (uint64_t*)take(n * 8);
    uint32_t* asim = (uint32_t*)take(n * 4);
    uint64_t* flag = (uint64_t*)take(n * 8);
    uint64_t* off = (uint64_t*)take(n * 8);
    uint64_t* sum = (uint64_t*)take(n * 8);
    unsigned long long* bad = (unsigned long long*)take(64);
    void* rws = take(radix_ws_bytes(n, 1));
    void* sws = take(scan_ws_bytes(n));
    QS_CUDA(cudaMemsetAsync(bad, 0, 8, st), "memset");
    const unsigned g = qs_blocks(n, 256);
    k_tri_unpack<<<g, 256, 0, st>>>((const uint32_t*)triplets_dev, n, key, sim, bad);
    int in_alt = 0;
    const uint32_t bits = (key_bits + 7) / 8 * 8;
    int rc = radix_sort_pairs(key, sim, n, 1, bits, akey, asim, rws, radix_ws_bytes(n, 1), &in_alt, st);
    if (rc) return rc;
    const uint64_t* k = in_alt ? akey : key;
    const uint32_t* v = in_alt ? asim : sim;
    k_tri_heads<<<g, 256, 0, st>>>(k, v, n, threshold, flag, sum);
    rc = scan_u64(flag, off, n, count_dev, sws, st);
    if (rc) return rc;
    k_tri_emit<<<g, 256, 0, st>>>(k, flag, off, sum, n, (uint32_t*)out_dev);
    QS_CHECK_LAUNCH("triplet combine");
    unsigned long long hbad = 0;
    QS_CUDA(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st), "copy");
    QS_CUDA(cudaStreamSynchronize(st), "sync");
    QS_DATA(hbad == 0, "triplet with dt or idx1 >= 2**32");
    return QS_OK;
}

}  // extern "C"
