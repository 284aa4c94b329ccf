// LSH search stages on sm_100a (integer / byte work, HBM- and ALU-bound).
//
// Reference: lsh_search.py:157-303.  The reference builds per-table sorted
// columns, then for every query gathers all equal-signature members of every
// table, materialises one 8-byte (q, c) key per (pair, table) hit, sorts all
// keys and run-length counts them (lsh_search.py:175-219).
//
// B200 design:
//   * keys (t, n) = mix64(signature word) (a bijection, so bucket equality is
//     exactly the reference's), the same keys row-major (n, t) for exact
//     verification, and bit-sliced 16-bit tags (n, W, 16) per row
//     (W = ceil(t/32): plane p of word w holds bit p of the tags of tables
//     32w..32w+31);
//   * buckets = per-table stable (key, id) sort, ids ascending in a bucket;
//   * pair enumeration inside buckets, each unordered pair handled ONLY in
//     the bucket of its first colliding table: earlier tables are screened
//     with 16 LOP3s per 32-table word on the tag planes (only the words up to
//     the bucket's table: warp-uniform) and confirmed on the 64-bit keys; the
//     collision count is screened on 8 planes and made exact (16 planes + key
//     confirmation) only when it could reach m.  No (pair, table) key is ever
//     materialised and no global hash table is needed.
//   * occurrence filter: pass 1 ("matched" mode) collects pairs with >= m
//     collisions, the filter marks excluded fingerprints, pass 2 ("distinct"
//     mode) counts distinct pairs over buckets with the excluded members
//     removed (partitions == 1) or masked (partitions > 1).
#include "qs_lsh.cuh"

namespace qs {

// ------------------------------------------------------------------ scan
// Multi-block exclusive scan of uint64 (in place allowed).
constexpr int SCAN_T = 512;
constexpr int SCAN_I = 8;
constexpr uint64_t SCAN_TILE = SCAN_T * SCAN_I;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* wsum, uint64_t* total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < (blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const uint64_t r = (warp ? wsum[warp - 1] : 0) + x - v;
    if (total) *total = wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(const uint64_t* __restrict__ in, uint64_t len,
                                                        uint64_t* __restrict__ part) {
    __shared__ uint64_t red[SCAN_T / 32];
    const uint64_t base = blockIdx.x * SCAN_TILE;
    uint64_t s = 0;
    for (int e = 0; e < SCAN_I; ++e) {
        uint64_t i = base + (uint64_t)e * SCAN_T + threadIdx.x;
        if (i < len) s += in[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < SCAN_T / 32; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_scan_top(uint64_t* __restrict__ a, uint64_t len,
                                                   uint64_t* __restrict__ total) {
    __shared__ uint64_t ws[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < len; b0 += 1024) {
        const uint64_t i = b0 + threadIdx.x;
        const uint64_t v = i < len ? a[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, ws, &tot);
        if (i < len) a[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_down(const uint64_t* __restrict__ in, uint64_t len,
                                                      const uint64_t* __restrict__ part,
                                                      uint64_t* __restrict__ out) {
    __shared__ uint64_t ws[32];
    const uint64_t base = blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_I;
    uint64_t v[SCAN_I], s = 0;
#pragma unroll
    for (int e = 0; e < SCAN_I; ++e) {
        v[e] = (base + e < len) ? in[base + e] : 0;
        s += v[e];
    }
    uint64_t ex = block_excl_scan(s, ws, nullptr) + part[blockIdx.x];
#pragma unroll
    for (int e = 0; e < SCAN_I; ++e) {
        if (base + e < len) out[base + e] = ex;
        ex += v[e];
    }
}

size_t scan_ws_bytes(uint64_t len) { return ((len + SCAN_TILE - 1) / SCAN_TILE + 1) * 8 + 64; }

// out[i] = sum(in[0..i)); *total (device) = sum(in) if total != nullptr.
int scan_u64(const uint64_t* in, uint64_t* out, uint64_t len, uint64_t* total, void* ws,
             cudaStream_t st) {
    if (len == 0) {
        if (total) QS_CUDA(cudaMemsetAsync(total, 0, 8, st), "memset");
        return QS_OK;
    }
    const uint64_t nb = (len + SCAN_TILE - 1) / SCAN_TILE;
    uint64_t* part = (uint64_t*)ws;
    k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, st>>>(in, len, part);
    k_scan_top<<<1, 1024, 0, st>>>(part, nb, total);
    k_scan_down<<<(unsigned)nb, SCAN_T, 0, st>>>(in, len, part, out);
    QS_CHECK_LAUNCH("scan");
    return QS_OK;
}

// ------------------------------------------------------------------- prep
// Row-major signatures -> table-major keys, row-major keys, bit-sliced tags.
__global__ void __launch_bounds__(256) k_prep(const uint64_t* __restrict__ sigs, uint64_t n,
                                              uint32_t t, uint64_t* __restrict__ keys,
                                              uint64_t* __restrict__ rkeys,
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
}

// After a sort on the top 32 key bits: each run of equal prefix is scanned by
// the thread at its start; if its full keys are not already grouped, the run
// is insertion-sorted by full key (stable, so ids stay ascending per key).
// Runs are short (mixed runs are rare prefix collisions), so cost ~ one pass.
// Keys are sorted on their top (64 - SORT_LO) bits only; runs of equal prefix
// holding several distinct keys (prefix collisions) are then restored to
// full-key order.  Detection reads the sorted keys once, coalesced; only the
// first out-of-order position of a run reports the run start.
constexpr uint32_t SORT_LO = 32;

constexpr uint32_t FIX_LMAX = 8192;   // elements sorted in shared memory per long run
constexpr uint32_t FIX_LCAP = 65536;  // long runs listed per build

__device__ void insertion_run(uint64_t* __restrict__ keys, uint32_t* __restrict__ ids, uint64_t g,
                              uint64_t e) {
    for (uint64_t i = g + 1; i < e; ++i) {
        const uint64_t key = keys[i];
        const uint32_t id = ids[i];
        uint64_t j = i;
        while (j > g && keys[j - 1] > key) {
            keys[j] = keys[j - 1];
            ids[j] = ids[j - 1];
            --j;
        }
        keys[j] = key;
        ids[j] = id;
    }
}

// grid (blocks, t): table blockIdx.y, in-table positions grid-strided (no
// 64-bit modulo per element)
__global__ void k_fix_detect(const uint64_t* __restrict__ keys, uint64_t n, uint64_t total,
                             uint64_t* __restrict__ runs, uint64_t cap,
                             unsigned long long* __restrict__ nruns) {
    (void)total;
    const uint64_t* k = keys + (uint64_t)blockIdx.y * n;
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; pos < n;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k0 = k[pos], k1 = k[pos - 1];
        if ((k0 >> SORT_LO) != (k1 >> SORT_LO) || k0 >= k1) continue;
        // out of order at pos: walk back to the run start; report only if no
        // earlier out-of-order position in the run
        uint64_t j = pos - 1;
        bool firstbad = true;
        while (j > 0 && (k[j - 1] >> SORT_LO) == (k0 >> SORT_LO)) {
            if (k[j] < k[j - 1]) firstbad = false;
            --j;
        }
        if (!firstbad) continue;
        const unsigned long long o = atomicAdd(nruns, 1ULL);
        if (o < cap) runs[o] = (uint64_t)blockIdx.y * n + j;
    }
}

// each reported run restored to full-key order: one warp per run; runs of up
// to 32 members are ranked in registers (key, then position: stable), longer
// runs by one lane's insertion sort
__global__ void k_fix_runs(uint64_t* __restrict__ keys, uint32_t* __restrict__ ids, uint64_t n,
                           const uint64_t* __restrict__ runs, uint64_t cap,
                           unsigned long long* __restrict__ nruns,
                           ulonglong2* __restrict__ longruns) {
    const uint64_t cnt = min((uint64_t)*nruns, cap);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < cnt; r += nw) {
        const uint64_t g = runs[r];
        const uint64_t seg_end = g - g % n + n;
        const uint64_t pre = keys[g] >> SORT_LO;
        // run length: 32-wide probes
        uint64_t e = g;
        while (true) {
            const uint64_t i = e + lane;
            const bool in = i < seg_end && (keys[i] >> SORT_LO) == pre;
            const uint32_t bal = __ballot_sync(0xffffffffu, in);
            if (bal != 0xffffffffu) {
                e += __ffs(~bal) - 1;
                break;
            }
            e += 32;
        }
        const uint64_t len = e - g;
        if (len <= 32) {
            const bool ok = lane < len;
            const uint64_t k = ok ? keys[g + lane] : ~0ull;
            const uint32_t id = ok ? ids[g + lane] : 0u;
            uint32_t rank = 0;
            for (uint32_t j = 0; j < len; ++j) {
                const uint64_t kj = __shfl_sync(0xffffffffu, k, j);
                rank += (kj < k) || (kj == k && j < lane);
            }
            __syncwarp();
            if (ok) {
                keys[g + rank] = k;
                ids[g + rank] = id;
            }
        } else if (lane == 0) {
            const unsigned long long o = atomicAdd(nruns + 1, 1ULL);
            if (o < FIX_LCAP) longruns[o] = make_ulonglong2(g, len);
            else insertion_run(keys, ids, g, e);  // overflow: serial (never seen at cfg1)
        }
        __syncwarp();
    }
}

// runs longer than 32: one CTA per run, stable bitonic sort of (key, position)
// in shared memory (FIX_LMAX elements); longer runs by serial insertion
__global__ void __launch_bounds__(1024) k_fix_long_runs(uint64_t* __restrict__ keys,
                                                        uint32_t* __restrict__ ids,
                                                        const ulonglong2* __restrict__ longruns,
                                                        const unsigned long long* __restrict__ nruns) {
    extern __shared__ __align__(16) unsigned char fx_smem[];
    uint64_t* sk = (uint64_t*)fx_smem;                 // [FIX_LMAX]
    uint32_t* sp = (uint32_t*)(sk + FIX_LMAX);         // [FIX_LMAX] original position
    uint32_t* si = sp + FIX_LMAX;                      // [FIX_LMAX] ids in original order
    const uint64_t cnt = min((uint64_t)nruns[1], (uint64_t)FIX_LCAP);
    for (uint64_t r = blockIdx.x; r < cnt; r += gridDim.x) {
        const uint64_t g = longruns[r].x, len = longruns[r].y;
        if (len > FIX_LMAX) {
            if (threadIdx.x == 0) insertion_run(keys, ids, g, g + len);
            __syncthreads();
            continue;
        }
        uint32_t P = 1;
        while (P < len) P <<= 1;
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
            sk[i] = i < len ? keys[g + i] : ~0ull;
            sp[i] = i;
            if (i < len) si[i] = ids[g + i];
        }
        __syncthreads();
        for (uint32_t k = 2; k <= P; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                    const uint32_t l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        const uint64_t a = sk[i], b = sk[l];
                        const uint32_t pa = sp[i], pb = sp[l];
                        const bool gt = a > b || (a == b && pa > pb);
                        if (gt == up) {
                            sk[i] = b; sk[l] = a;
                            sp[i] = pb; sp[l] = pa;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
            keys[g + i] = sk[i];
            ids[g + i] = si[sp[i]];
        }
        __syncthreads();
    }
}

// fallback when the run list overflowed: every run start fixes its own run
__global__ void k_fix_prefix_runs(uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                                  uint64_t n, uint64_t total, uint64_t cap,
                                  const unsigned long long* __restrict__ nruns) {
    if (*nruns <= cap) return;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pos = g % n;
        const uint64_t k0 = keys[g];
        if (pos != 0 && (keys[g - 1] >> SORT_LO) == (k0 >> SORT_LO)) continue;  // not a run start
        const uint64_t seg_end = g - pos + n;
        uint64_t e = g + 1;
        bool sorted = true;
        uint64_t prev = k0;
        while (e < seg_end) {
            const uint64_t k = keys[e];
            if ((k >> SORT_LO) != (k0 >> SORT_LO)) break;
            if (k < prev) sorted = false;
            prev = k;
            ++e;
        }
        if (sorted) continue;
        for (uint64_t i = g + 1; i < e; ++i) {
            const uint64_t key = keys[i];
            const uint32_t id = ids[i];
            uint64_t j = i;
            while (j > g && keys[j - 1] > key) {
                keys[j] = keys[j - 1];
                ids[j] = ids[j - 1];
                --j;
            }
            keys[j] = key;
            ids[j] = id;
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
// kind 0: heads of non-singleton buckets, 1: tails of non-singleton buckets,
// 2: all heads (count only).
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

// per block: [0] heads of non-singleton buckets, [1] all heads
__global__ void __launch_bounds__(LIST_THREADS) k_list_count(const uint64_t* __restrict__ k,
                                                             uint64_t n, uint64_t total,
                                                             uint64_t chunk, uint64_t nblk,
                                                             uint64_t* __restrict__ counts) {
    __shared__ uint32_t red[2][LIST_THREADS / 32];
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    uint32_t c0 = 0, c1 = 0;
    for (uint64_t g = lo + threadIdx.x; g < hi; g += LIST_THREADS) {
        c0 += list_flag(k, n, g, 0);
        c1 += list_flag(k, n, g, 2);
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
        for (int w = 0; w < LIST_THREADS / 32; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        counts[blockIdx.x] = s0;
        counts[nblk + blockIdx.x] = s1;
    }
}

// One sweep writes both ends of every non-singleton bucket: heads store their
// global position into bstart[i], tails their in-table position into bsize[i],
// i = number of non-singleton heads at or before the element, minus one (the
// head may sit in an earlier block: offs carries the count of earlier blocks).
__global__ void __launch_bounds__(LIST_THREADS) k_list_write(const uint64_t* __restrict__ k,
                                                             uint64_t n, uint64_t total,
                                                             uint64_t chunk,
                                                             const uint64_t* __restrict__ offs,
                                                             uint64_t* __restrict__ out64,
                                                             uint32_t* __restrict__ out32) {
    constexpr int PER = 4;  // consecutive elements per thread
    __shared__ uint32_t wsum[LIST_THREADS / 32];
    __shared__ uint64_t base;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(total, lo + chunk);
    if (threadIdx.x == 0) base = offs[blockIdx.x];
    __syncthreads();
    for (uint64_t g0 = lo; g0 < hi; g0 += LIST_THREADS * PER) {
        const uint64_t gt = g0 + (uint64_t)threadIdx.x * PER;
        bool hd[PER], tl[PER];
        uint32_t c = 0;
        if (gt < hi) {
            uint64_t kk[PER + 2];
#pragma unroll
            for (int e = 0; e < PER + 2; ++e) {
                const uint64_t i = gt + e - 1;
                kk[e] = (i < total && (e > 0 || gt > 0)) ? k[i] : 0;
            }
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const uint64_t g = gt + e;
                const uint64_t pos = g % n;
                const bool in = g < hi;
                const bool head = pos == 0 || kk[e] != kk[e + 1];
                const bool tail = pos == n - 1 || kk[e + 2] != kk[e + 1];
                hd[e] = in && head && !tail;
                tl[e] = in && tail && !head;
                c += hd[e];
            }
        } else {
#pragma unroll
            for (int e = 0; e < PER; ++e) hd[e] = tl[e] = false;
        }
        // block exclusive scan of per-thread head counts
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
        for (int w = 0; w < LIST_THREADS / 32; ++w) {
            if (w < (int)warp) wb += wsum[w];
            tot += wsum[w];
        }
        uint64_t incl = wb + x - c;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            incl += hd[e];
            if (hd[e]) out64[incl - 1] = gt + e;
            if (tl[e]) out32[incl - 1] = (uint32_t)((gt + e) % n);
        }
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
}

// bsize holds in-table tail positions on entry, bucket sizes on exit
__global__ void k_make_sizes(const uint64_t* __restrict__ heads, const uint64_t* __restrict__ nbp,
                             uint64_t n, uint32_t* __restrict__ bsize, uint32_t* __restrict__ btab,
                             const uint32_t* __restrict__ table_ids) {
    const uint64_t nb = *nbp;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x) {
        bsize[i] = (uint32_t)(bsize[i] - heads[i] % n + 1);
        const uint32_t local = (uint32_t)(heads[i] / n);
        btab[i] = table_ids ? table_ids[local] : local;
    }
}

int make_bucket_sizes(const uint64_t* bstart, const uint64_t* counts, uint64_t n, uint32_t* bsize,
                      uint32_t* btab, const uint32_t* table_ids, cudaStream_t st) {
    k_make_sizes<<<148 * 8, 256, 0, st>>>(bstart, counts, n, bsize, btab, table_ids);
    QS_CHECK_LAUNCH("bucket sizes");
    return QS_OK;
}

// ----------------------------------------------------------------- stats
constexpr int ST_HIST = 256;
constexpr uint32_t KEEP_LANE = 16;  // compaction: buckets above this are handled by a warp

__device__ __forceinline__ void stats_piece(uint64_t nP, unsigned long long* sh,
                                            unsigned long long* __restrict__ hist,
                                            uint32_t hist_len, uint32_t* __restrict__ big,
                                            uint64_t big_cap, unsigned long long* __restrict__ out,
                                            unsigned long long& mx) {
    if (nP > mx) mx = nP;
    if (nP < ST_HIST) atomicAdd(sh + nP, 1ULL);
    else if (nP < hist_len) atomicAdd(hist + nP, 1ULL);
    else {
        unsigned long long k = atomicAdd(out + 2, 1ULL);
        if (k < big_cap) big[k] = (uint32_t)nP;
    }
}

// One thread per non-singleton bucket: partition split, lookups, size histogram.
__global__ void __launch_bounds__(256) k_bucket_stats(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, uint64_t nb, const uint8_t* __restrict__ excl_mask,
    const uint64_t* __restrict__ edges, uint32_t p, unsigned long long* __restrict__ hist,
    uint32_t hist_len, uint32_t* __restrict__ big, uint64_t big_cap,
    unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sh[ST_HIST];
    for (int i = threadIdx.x; i < ST_HIST; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    unsigned long long looks = 0, pieces = 0, mx = 0;
    const bool simple = (p <= 1) && (excl_mask == nullptr);
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = bsize[b];
        if (simple) {
            looks += s * (s - 1);
            ++pieces;
            stats_piece(s, sh, hist, hist_len, big, big_cap, out, mx);
            continue;
        }
        const uint64_t st = bstart[b];
        uint64_t cum_e = 0, e_tot = 0, j = 0;
        unsigned long long lb = 0;
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
            lb += nP * (s - cum_e);
            ++pieces;
            stats_piece(nP, sh, hist, hist_len, big, big_cap, out, mx);
        }
        looks += lb - (s - e_tot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        looks += __shfl_down_sync(0xffffffffu, looks, o);
        pieces += __shfl_down_sync(0xffffffffu, pieces, o);
        unsigned long long y = __shfl_down_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (looks) atomicAdd(out + 0, looks);
        if (pieces) atomicAdd(out + 1, pieces);
        if (mx) atomicMax(out + 3, mx);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ST_HIST; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// -------------------------------------------------- exclusion compaction
// partitions == 1 only: an excluded member can never be part of a counted
// pair, so it is removed from the bucket before enumeration.
// keep counts per bucket; with `hist` (single partition) also the bucket
// statistics of k_bucket_stats: one piece of size s per bucket, lookups
// (s - 1)(s - e) with e excluded members (lsh_search.py:192-194)
__global__ void __launch_bounds__(256) k_keep_count(
    const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
    const uint32_t* __restrict__ bsize, uint64_t nb, const uint8_t* __restrict__ ex,
    uint64_t* __restrict__ cnt, uint64_t* __restrict__ flag, unsigned long long* __restrict__ hist,
    uint32_t hist_len, uint32_t* __restrict__ big, uint64_t big_cap,
    unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sh[ST_HIST];
    if (hist) {
        for (int i = threadIdx.x; i < ST_HIST; i += blockDim.x) sh[i] = 0;
        __syncthreads();
    }
    unsigned long long looks = 0, pieces = 0, mx = 0;
    const uint32_t lane = threadIdx.x & 31;
    // a warp takes 32 consecutive buckets: a lane counts its own bucket when it
    // is small; buckets above KEEP_LANE members are counted by the whole warp
    // afterwards (coalesced member reads, no single-lane tail)
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t b0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; b0 < nb;
         b0 += nwarps * 32) {
        const uint64_t b = b0 + lane;
        uint64_t st = 0;
        uint32_t s = 0;
        if (b < nb) {
            st = bstart[b];
            s = bsize[b];
        }
        uint32_t k = 0;
        const bool lone = s <= KEEP_LANE;
        if (lone)
            for (uint32_t j = 0; j < s; ++j) k += ex[sids[st + j]] == 0;
        uint32_t bigl = __ballot_sync(0xffffffffu, !lone);
        while (bigl) {
            const int src = __ffs(bigl) - 1;
            bigl &= bigl - 1;
            const uint64_t bst = __shfl_sync(0xffffffffu, st, src);
            const uint32_t bs = __shfl_sync(0xffffffffu, s, src);
            uint32_t kk = 0;
            for (uint32_t j = lane; j < bs; j += 32) kk += ex[sids[bst + j]] == 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
            if (lane == (uint32_t)src) k = kk;
        }
        if (b >= nb) continue;
        cnt[b] = k >= 2 ? k : 0;
        flag[b] = k >= 2 ? 1 : 0;
        if (hist) {
            looks += (unsigned long long)(s - 1) * k;
            ++pieces;
            stats_piece(s, sh, hist, hist_len, big, big_cap, out, mx);
        }
    }
    if (!hist) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        looks += __shfl_down_sync(0xffffffffu, looks, o);
        pieces += __shfl_down_sync(0xffffffffu, pieces, o);
        unsigned long long y = __shfl_down_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (looks) atomicAdd(out + 0, looks);
        if (pieces) atomicAdd(out + 1, pieces);
        if (mx) atomicMax(out + 3, mx);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ST_HIST; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

__global__ void k_keep_write(const uint32_t* __restrict__ sids, const uint64_t* __restrict__ bstart,
                             const uint32_t* __restrict__ bsize, const uint32_t* __restrict__ btab,
                             uint64_t nb, const uint8_t* __restrict__ ex,
                             const uint64_t* __restrict__ cnt_raw, const uint64_t* __restrict__ mem_off,
                             const uint64_t* __restrict__ slot, uint32_t* __restrict__ sids2,
                             uint64_t* __restrict__ bstart2, uint32_t* __restrict__ bsize2,
                             uint32_t* __restrict__ btab2) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t b0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; b0 < nb;
         b0 += nwarps * 32) {
        const uint64_t b = b0 + lane;
        const uint64_t k = b < nb ? cnt_raw[b] : 0;
        uint64_t st = 0, o = 0;
        uint32_t s = 0;
        if (k) {
            st = bstart[b];
            o = mem_off[b];
            s = bsize[b];
            const uint64_t sl = slot[b];
            bstart2[sl] = o;
            bsize2[sl] = (uint32_t)k;
            btab2[sl] = btab[b];
        }
        const bool lone = s <= KEEP_LANE;
        if (k && lone) {
            uint64_t w = o;
            for (uint32_t j = 0; j < s; ++j) {
                const uint32_t x = sids[st + j];
                if (!ex[x]) sids2[w++] = x;
            }
        }
        uint32_t bigl = __ballot_sync(0xffffffffu, k && !lone);
        while (bigl) {
            const int src = __ffs(bigl) - 1;
            bigl &= bigl - 1;
            const uint64_t bst = __shfl_sync(0xffffffffu, st, src);
            const uint32_t bs = __shfl_sync(0xffffffffu, s, src);
            uint64_t w = __shfl_sync(0xffffffffu, o, src);
            for (uint32_t j0 = 0; j0 < bs; j0 += 32) {
                const uint32_t j = j0 + lane;
                uint32_t x = 0;
                bool keep = false;
                if (j < bs) {
                    x = sids[bst + j];
                    keep = !ex[x];
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (keep) sids2[w + __popc(bal & lt)] = x;
                w += __popc(bal);
            }
        }
    }
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

// matched pairs of the filter-free pass that survive the exclusion rule
__global__ void k_filter_pairs(const uint64_t* __restrict__ pk, const uint32_t* __restrict__ ps,
                               const uint32_t* __restrict__ rest, uint32_t W,
                               uint64_t np, const uint8_t* __restrict__ ex,
                               const uint64_t* __restrict__ edges, uint32_t p,
                               uint64_t* __restrict__ opk, uint32_t* __restrict__ ops,
                               uint32_t* __restrict__ orest,
                               unsigned long long* __restrict__ counter) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = pk[i];
        const uint64_t c = k & 0xFFFFFFFFull, q = c + (k >> 32);
        if (ex[c]) continue;
        if (ex[q] && (p <= 1 || part_of(edges, p, c) == part_of(edges, p, q))) continue;
        const unsigned long long o = atomicAdd(counter, 1ULL);
        opk[o] = k;
        ops[o] = ps[i];
        if (rest)
            for (uint32_t w = 0; w < W; ++w) orest[o * W + w] = rest[i * W + w];
    }
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

int num_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace qs

using namespace qs;

extern "C" {

int qs_lsh_prep(const uint64_t* sigs_dev, uint64_t n, uint32_t t, uint64_t* keys_dev,
                uint64_t* rkeys_dev, uint32_t* tags_dev, void* stream) {
    QS_ARG(t >= 1, "tables must be >= 1");
    if (n == 0) return QS_OK;
    k_prep<<<qs_blocks(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(sigs_dev, n, t, keys_dev,
                                                                      rkeys_dev, tags_dev);
    QS_CHECK_LAUNCH("k_prep");
    return QS_OK;
}

// reported-run capacity of the prefix fix-up (overflow falls back to a full scan)
static uint64_t fix_cap(uint64_t total) { return total / 16 + 1024; }

size_t qs_lsh_bucket_ws_bytes(uint64_t n, uint32_t t) {
    const uint64_t total = n * t;
    return (size_t)total * (sizeof(uint64_t) + sizeof(uint32_t)) + radix_ws_bytes(n, t) +
           fix_cap(total) * 8 + (size_t)FIX_LCAP * 16 + 1024;
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
    unsigned char* rest = (unsigned char*)(((uintptr_t)(w + total * 12) + 255) & ~(uintptr_t)255);
    void* rws = rest;
    const size_t rws_bytes = radix_ws_bytes(n, t);
    unsigned long long* nruns =
        (unsigned long long*)(((uintptr_t)(rest + rws_bytes) + 255) & ~(uintptr_t)255);
    ulonglong2* longruns = (ulonglong2*)(nruns + 32);
    uint64_t* runs = (uint64_t*)(longruns + FIX_LCAP);
    const uint64_t cap = fix_cap(total);
    // keys are fmix64-mixed, so their top 24 bits separate almost all distinct
    // keys: sort (stably, ids = in-table position) on bits [40, 64) in three
    // 8-bit passes straight from the caller's keys, then restore full-key order
    // in the runs whose prefixes collide
    int rc = radix_sort_pairs_to(keys_dev, nullptr, n, t, SORT_LO, 64, keys_out_dev, ids_out_dev,
                                 alt_k, alt_v, rws, rws_bytes, st);
    if (rc) return rc;
    QS_CUDA(cudaMemsetAsync(nruns, 0, 16, st), "memset");
    const unsigned g = qs_blocks(total, 256);
    k_fix_detect<<<dim3(qs_blocks(n, 256, 1184), t), 256, 0, st>>>(keys_out_dev, n, total, runs,
                                                                    cap, nruns);
    k_fix_runs<<<148 * 16, 256, 0, st>>>(keys_out_dev, ids_out_dev, n, runs, cap, nruns, longruns);
    const int long_smem = (int)(FIX_LMAX * 16);
    QS_CUDA(cudaFuncSetAttribute(k_fix_long_runs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 long_smem), "smem attr");
    k_fix_long_runs<<<148, 1024, long_smem, st>>>(keys_out_dev, ids_out_dev, longruns, nruns);
    k_fix_prefix_runs<<<g, 256, 0, st>>>(keys_out_dev, ids_out_dev, n, total, cap, nruns);
    QS_CHECK_LAUNCH("fix prefix runs");
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
    return (size_t)(2 * b + 1) * 8 + scan_ws_bytes(b) + 256;
}

int qs_lsh_list_buckets(const uint64_t* skeys_dev, uint64_t n, uint32_t t, uint64_t* bstart_dev,
                        uint32_t* bsize_dev, uint32_t* btab_dev, const uint32_t* table_ids_dev,
                        uint64_t* counts_dev, void* ws_dev, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_list_ws_bytes(n, t), "list workspace too small");
    const uint64_t total = n * t;
    if (total == 0) {
        QS_CUDA(cudaMemsetAsync(counts_dev, 0, 16, st), "memset");
        return QS_OK;
    }
    const uint64_t B = list_blocks(total);
    const uint64_t chunk = (total + B - 1) / B;
    uint64_t* cnt = (uint64_t*)ws_dev;  // [0, B): non-singleton heads, [B, 2B): all heads
    void* sws = (void*)(((uintptr_t)(cnt + 2 * B + 1) + 63) & ~(uintptr_t)63);
    k_list_count<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, B, cnt);
    int rc = scan_u64(cnt, cnt, B, counts_dev + 0, sws, st);
    if (rc) return rc;
    rc = scan_u64(cnt + B, cnt + B, B, counts_dev + 1, sws, st);
    if (rc) return rc;
    if (bstart_dev != nullptr) {
        k_list_write<<<B, LIST_THREADS, 0, st>>>(skeys_dev, n, total, chunk, cnt, bstart_dev,
                                                 bsize_dev);
        k_make_sizes<<<148 * 8, 256, 0, st>>>(bstart_dev, counts_dev, n, bsize_dev, btab_dev,
                                              table_ids_dev);
    }
    QS_CHECK_LAUNCH("list buckets");
    return QS_OK;
}

int qs_lsh_bucket_stats(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                        const uint32_t* bsize_dev, uint64_t n_nonsingle,
                        const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p,
                        uint64_t* hist_dev, uint32_t hist_len, uint32_t* big_dev, uint64_t big_cap,
                        uint64_t* out_dev, void* stream) {
    if (n_nonsingle == 0) return QS_OK;
    QS_ARG(hist_len >= ST_HIST, "hist_len must be >= %d", ST_HIST);
    k_bucket_stats<<<qs_blocks(n_nonsingle, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        sids_dev, bstart_dev, bsize_dev, n_nonsingle, excluded_dev, edges_dev, p,
        (unsigned long long*)hist_dev, hist_len, big_dev, big_cap, (unsigned long long*)out_dev);
    QS_CHECK_LAUNCH("k_bucket_stats");
    return QS_OK;
}

size_t qs_lsh_compact_ws_bytes(uint64_t n_nonsingle) {
    return (size_t)(n_nonsingle + 1) * 8 * 3 + scan_ws_bytes(n_nonsingle + 1) + 512;
}

int qs_lsh_compact_buckets(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                           const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t nb,
                           const uint8_t* excluded_dev, uint32_t* sids2_dev, uint64_t* bstart2_dev,
                           uint32_t* bsize2_dev, uint32_t* btab2_dev, uint64_t* counts_dev,
                           uint64_t* hist_dev, uint32_t hist_len, uint32_t* big_dev,
                           uint64_t big_cap, uint64_t* stats_out_dev,
                           void* ws_dev, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    QS_ARG(ws_bytes >= qs_lsh_compact_ws_bytes(nb), "compact workspace too small");
    if (nb == 0) {
        QS_CUDA(cudaMemsetAsync(counts_dev, 0, 16, st), "memset");
        return QS_OK;
    }
    uint64_t* cnt = (uint64_t*)ws_dev;
    uint64_t* off = cnt + (nb + 1);
    uint64_t* slot = off + (nb + 1);
    void* sws = (void*)(((uintptr_t)(slot + nb + 1) + 63) & ~(uintptr_t)63);
    const unsigned g = qs_blocks(nb, 256);
    if (hist_dev) QS_ARG(hist_len >= ST_HIST && stats_out_dev, "stats outputs: hist_len >= %d and out", ST_HIST);
    k_keep_count<<<g, 256, 0, st>>>(sids_dev, bstart_dev, bsize_dev, nb, excluded_dev, cnt, slot,
                                    (unsigned long long*)hist_dev, hist_len, big_dev, big_cap,
                                    (unsigned long long*)stats_out_dev);
    int rc = scan_u64(cnt, off, nb, counts_dev + 1, sws, st);
    if (rc) return rc;
    rc = scan_u64(slot, slot, nb, counts_dev + 0, sws, st);
    if (rc) return rc;
    k_keep_write<<<g, 256, 0, st>>>(sids_dev, bstart_dev, bsize_dev, btab_dev, nb, excluded_dev, cnt,
                                     off, slot, sids2_dev, bstart2_dev, bsize2_dev, btab2_dev);
    QS_CHECK_LAUNCH("compact buckets");
    return QS_OK;
}

int qs_lsh_occ_degree(const uint64_t* pair_key_dev, uint64_t n_pairs, const uint64_t* edges_dev,
                      uint32_t p, uint32_t* degree_dev, void* stream) {
    if (n_pairs == 0) return QS_OK;
    k_occ_degree<<<qs_blocks(n_pairs, 256), 256, 0, (cudaStream_t)stream>>>(pair_key_dev, n_pairs,
                                                                           edges_dev, p, degree_dev);
    QS_CHECK_LAUNCH("k_occ_degree");
    return QS_OK;
}

int qs_lsh_occ_mark(const uint64_t* pair_key_dev, uint64_t n_pairs, const uint32_t* degree_dev,
                    uint64_t n, double threshold, const uint64_t* edges_dev, uint32_t p,
                    uint8_t* excluded_dev, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return QS_OK;
    k_occ_core<<<qs_blocks(n, 256), 256, 0, st>>>(degree_dev, n, threshold, edges_dev, p, excluded_dev);
    if (n_pairs)
        k_occ_touch<<<qs_blocks(n_pairs, 256), 256, 0, st>>>(pair_key_dev, n_pairs, edges_dev, p,
                                                             excluded_dev);
    QS_CHECK_LAUNCH("occurrence mark");
    return QS_OK;
}

int qs_lsh_occ_finish(uint8_t* excluded_dev, uint64_t n, unsigned long long* counters_dev,
                      void* stream) {
    if (n == 0) return QS_OK;
    k_occ_finish<<<qs_blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(excluded_dev, n, counters_dev);
    QS_CHECK_LAUNCH("k_occ_finish");
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
    int rc = qs_lsh_occ_degree(pair_key_dev, n_pairs, edges_dev, p, deg, stream);
    if (rc) return rc;
    rc = qs_lsh_occ_mark(pair_key_dev, n_pairs, deg, n, threshold, edges_dev, p, excluded_dev, stream);
    if (rc) return rc;
    return qs_lsh_occ_finish(excluded_dev, n, counters_dev, stream);
}

int qs_lsh_filter_pairs(const uint64_t* pair_key_dev, const uint32_t* pair_sim_dev,
                        const uint32_t* rest_dev, uint32_t rest_words, uint64_t n_pairs,
                        const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p,
                        uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev,
                        unsigned long long* counter_dev, void* stream) {
    if (n_pairs == 0) return QS_OK;
    QS_ARG(!rest_dev || out_rest_dev, "out_rest_dev required with rest_dev");
    k_filter_pairs<<<qs_blocks(n_pairs, 256), 256, 0, (cudaStream_t)stream>>>(
        pair_key_dev, pair_sim_dev, rest_dev, rest_words, n_pairs, excluded_dev, edges_dev, p,
        out_key_dev, out_sim_dev, out_rest_dev, counter_dev);
    QS_CHECK_LAUNCH("k_filter_pairs");
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
                              radix_ws_bytes(n_pairs, 1), &in_alt, st, 0,
                              key_bits > 32 ? key_bits - 32 : 32);
    if (rc) return rc;
    const uint64_t* k = in_alt ? ak : pair_key_dev;
    const uint32_t* v = in_alt ? av : pair_sim_dev;
    k_pack_triplets<<<qs_blocks(n_pairs, 256), 256, 0, st>>>(k, v, n_pairs, (uint32_t*)triplets_dev);
    QS_CHECK_LAUNCH("k_pack_triplets");
    return QS_OK;
}

}  // extern "C"
