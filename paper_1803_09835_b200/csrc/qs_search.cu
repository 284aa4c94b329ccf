// One-call search entries of the C ABI (no Python host layer needed):
//   qs_lsh_search           signatures (n, t) -> sorted triplets + SearchStats
//                           (lsh_search.search_signatures, lsh_search.py:222-303)
//   qs_lsh_search_bits      set bits (n, K) -> mapping -> signatures -> search
//                           (lsh_search.search_fingerprints, lsh_search.py:314-333)
// Both run the same stage sequence as the Python orchestration
// (paper_1803_09835_b200/lsh_search.py run_search) over the stage entries of
// this library, with every buffer carved from ONE caller workspace (no
// cudaMalloc).  They synchronise the stream at the few points where a count
// decides the next allocation (bucket count, matched pairs).
#include <math.h>

#include <algorithm>
#include <vector>

#include "qs_common.cuh"

namespace {

constexpr uint32_t HIST_LEN = 1u << 16;

// bump allocator over the caller workspace (256-byte aligned pieces)
struct Bump {
    uint8_t* base;
    size_t cap, off;
    bool ok = true;
    template <class T>
    T* take(uint64_t count) {
        off = (off + 255) & ~(size_t)255;
        const size_t bytes = (size_t)count * sizeof(T);
        if (base == nullptr) {  // size query
            off += bytes;
            return nullptr;
        }
        if (off + bytes > cap) {
            ok = false;
            return nullptr;
        }
        T* p = (T*)(base + off);
        off += bytes;
        return p;
    }
    uint8_t* raw(size_t bytes) { return take<uint8_t>(bytes); }
};

// edges of partition_bounds (lsh_search.py:139-144): np.linspace(0, n, P + 1,
// dtype=int) with P = min(p, max(1, n)) — float64 i * (n / P) truncated, the
// last edge exactly n — keeping non-empty ranges only
std::vector<uint64_t> partition_edges(uint64_t n, uint32_t partitions) {
    const uint64_t P = std::min<uint64_t>(partitions, std::max<uint64_t>(1, n));
    std::vector<uint64_t> raw(P + 1);
    const double step = (double)n / (double)P;
    for (uint64_t i = 0; i <= P; ++i) raw[i] = (uint64_t)((double)i * step);
    raw[P] = n;
    std::vector<uint64_t> e{raw[0]};
    for (uint64_t i = 1; i <= P; ++i)
        if (raw[i] > e.back()) e.push_back(raw[i]);
    return e;
}

struct Sizes {  // worst-case element counts of one search
    uint64_t n, t, W, nbmax, cap;
};

Sizes sizes_of(uint64_t n, uint32_t t, uint64_t pair_cap) {
    Sizes s;
    s.n = n;
    s.t = t;
    s.W = (t + 31) / 32;
    s.nbmax = std::max<uint64_t>(1, n * t / 2);  // a non-singleton bucket has >= 2 members
    s.cap = std::max<uint64_t>(1, pair_cap);
    return s;
}

// layout shared by the size query and the run (same take() order)
struct Layout {
    uint64_t *keys, *rkeys, *edges, *counts, *bstart, *pk, *opk, *bstart2, *hist, *stats_out,
        *cnt2;
    unsigned long long* counters;
    uint32_t *tags, *sids, *bsize, *btab, *ps, *rest, *ops, *orest, *sids2, *bsize2, *btab2, *big;
    int32_t* occ_ws;
    uint8_t *flags, *emask, *trans;
    uint64_t big_cap;
    size_t trans_bytes;
};

size_t transient_bytes(const Sizes& s) {
    size_t b = qs_lsh_bucket_flags_ws_bytes(s.n, (uint32_t)s.t);
    b = std::max(b, qs_lsh_list_flags_ws_bytes(s.n, (uint32_t)s.t));
    b = std::max(b, qs_lsh_pairs_ws_bytes(s.nbmax));
    b = std::max(b, qs_lsh_compact_ws_bytes(s.nbmax));
    b = std::max(b, qs_sort_pairs_ws_bytes(s.cap));
    return b;
}

void carve(Bump& a, const Sizes& s, Layout& L, uint32_t p) {
    L.keys = a.take<uint64_t>(s.t * s.n);
    L.rkeys = a.take<uint64_t>(s.n * s.t);
    L.tags = a.take<uint32_t>(2 * s.n * s.W * 8);
    L.edges = a.take<uint64_t>(p + 1);
    L.counts = a.take<uint64_t>(4);
    L.counters = a.take<unsigned long long>(4);
    L.sids = a.take<uint32_t>(s.t * s.n);
    L.flags = a.take<uint8_t>(s.t * s.n);
    L.bstart = a.take<uint64_t>(s.nbmax);
    L.bsize = a.take<uint32_t>(s.nbmax);
    L.btab = a.take<uint32_t>(s.nbmax);
    L.pk = a.take<uint64_t>(s.cap);
    L.ps = a.take<uint32_t>(s.cap);
    L.rest = a.take<uint32_t>(s.cap * s.W);
    L.emask = a.take<uint8_t>(s.n);
    L.occ_ws = a.take<int32_t>(s.n);
    L.opk = a.take<uint64_t>(s.cap);
    L.ops = a.take<uint32_t>(s.cap);
    L.orest = a.take<uint32_t>(s.cap * s.W);
    L.sids2 = a.take<uint32_t>(s.t * s.n);
    L.bstart2 = a.take<uint64_t>(s.nbmax);
    L.bsize2 = a.take<uint32_t>(s.nbmax);
    L.btab2 = a.take<uint32_t>(s.nbmax);
    L.cnt2 = a.take<uint64_t>(2);
    L.hist = a.take<uint64_t>(HIST_LEN);
    L.big_cap = std::max<uint64_t>(1024, s.nbmax / 64);
    L.big = a.take<uint32_t>(L.big_cap);
    L.stats_out = a.take<uint64_t>(4);
    L.trans_bytes = transient_bytes(s);
    L.trans = a.raw(L.trans_bytes);
}

int d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    QS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    QS_CUDA(cudaStreamSynchronize(st), "stream sync");
    return QS_OK;
}

#define QS_TRY(x)              \
    do {                       \
        int _rc = (x);         \
        if (_rc) return _rc;   \
    } while (0)

// share of entries in the largest ceil(0.001 * n_buckets) buckets (lsh_search.py:295-302)
double top_mass(std::vector<uint64_t>& hist, std::vector<uint32_t>& big, uint64_t n_buckets,
                uint64_t total) {
    uint64_t need = std::max<uint64_t>(1, (uint64_t)ceil(0.001 * (double)n_buckets));
    uint64_t acc = 0;
    std::sort(big.begin(), big.end(), [](uint32_t a, uint32_t b) { return a > b; });
    for (uint32_t v : big) {
        if (need == 0) break;
        acc += v;
        --need;
    }
    for (int64_t sz = (int64_t)hist.size() - 1; sz >= 0 && need; --sz) {
        if (!hist[sz]) continue;
        const uint64_t take = std::min<uint64_t>(need, hist[sz]);
        acc += take * (uint64_t)sz;
        need -= take;
    }
    return total ? (double)acc / (double)total : 0.0;
}

// the stage sequence over a prepared search layout (keys/rkeys/tags in L)
int run(Layout& L, const Sizes& s, uint32_t m, uint64_t excl, double occ, uint32_t p,
        const std::vector<uint64_t>& edges, uint8_t* triplets, uint64_t* needed,
        qs_search_stats* stats, cudaStream_t st) {
    const uint64_t n = s.n;
    const uint32_t t = (uint32_t)s.t, W = (uint32_t)s.W;
    void* stv = (void*)st;
    QS_CUDA(cudaMemcpyAsync(L.edges, edges.data(), edges.size() * 8, cudaMemcpyHostToDevice, st),
            "H2D edges");
    // buckets: member ids grouped by key (stable), head/tail flags, listing
    QS_TRY(qs_lsh_build_bucket_flags(L.keys, n, t, L.sids, L.flags, L.trans, L.trans_bytes, stv));
    QS_CUDA(cudaMemsetAsync(L.counts, 0, 16, st), "memset");
    QS_TRY(qs_lsh_list_buckets_flags(L.flags, n, t, nullptr, nullptr, nullptr, nullptr, L.counts,
                                     L.trans, L.trans_bytes, stv));
    uint64_t hc[2];
    QS_TRY(d2h(hc, L.counts, 16, st));
    const uint64_t nb = hc[0], heads = hc[1];
    if (nb)
        QS_TRY(qs_lsh_list_buckets_flags(L.flags, n, t, L.bstart, L.bsize, L.btab, nullptr,
                                         L.counts, L.trans, L.trans_bytes, stv));
    auto pairs = [&](int mode, const uint8_t* emask, const uint32_t* sids, const uint64_t* bstart,
                     const uint32_t* bsize, const uint32_t* btab, uint64_t nbx, uint32_t* rest,
                     uint64_t& distinct, uint64_t& matched) -> int {
        QS_CUDA(cudaMemsetAsync(L.counters, 0, 16, st), "memset");
        QS_TRY(qs_lsh_pairs(sids, bstart, bsize, btab, nbx, L.rkeys, L.tags, n, t, m, excl, emask,
                            L.edges, p, mode, L.pk, L.ps, rest, mode == 2 ? 0 : s.cap, L.counters,
                            L.trans, L.trans_bytes, stv));
        unsigned long long c[2];
        QS_TRY(d2h(c, L.counters, 16, st));
        distinct = c[0];
        matched = c[1];
        if (mode != 2 && matched > s.cap) {
            if (needed) *needed = matched;
            qs::set_error("pair capacity %llu < %llu matched pairs", (unsigned long long)s.cap,
                          (unsigned long long)matched);
            return QS_ERR_CAPACITY;
        }
        return QS_OK;
    };
    uint64_t distinct = 0, matched = 0, n_ex = 0, dummy = 0;
    const uint8_t* emask = nullptr;
    uint64_t* pk = L.pk;
    uint32_t *ps = L.ps, *rest = nullptr;
    bool compacted = false;
    if (occ <= 0) {
        QS_TRY(pairs(0, nullptr, L.sids, L.bstart, L.bsize, L.btab, nb, nullptr, distinct, matched));
    } else {
        QS_TRY(pairs(1, nullptr, L.sids, L.bstart, L.bsize, L.btab, nb, L.rest, dummy, matched));
        rest = L.rest;
        QS_CUDA(cudaMemsetAsync(L.counters + 2, 0, 8, st), "memset");
        QS_TRY(qs_lsh_occurrence_filter(L.pk, L.ps, matched, n, occ, L.edges, p, L.emask,
                                        L.counters + 2, L.occ_ws, stv));
        unsigned long long ex;
        QS_TRY(d2h(&ex, L.counters + 2, 8, st));
        n_ex = ex;
        if (n_ex == 0) {
            QS_TRY(pairs(2, nullptr, L.sids, L.bstart, L.bsize, L.btab, nb, nullptr, distinct,
                         dummy));
        } else {
            emask = L.emask;
            QS_CUDA(cudaMemsetAsync(L.counters + 3, 0, 8, st), "memset");
            QS_TRY(qs_lsh_filter_pairs(L.pk, L.ps, L.rest, W, matched, L.emask, L.edges, p, L.opk,
                                       L.ops, L.orest, L.counters + 3, stv));
            unsigned long long k;
            QS_TRY(d2h(&k, L.counters + 3, 8, st));
            matched = k;
            pk = L.opk;
            ps = L.ops;
            rest = L.orest;
            if (p == 1) {
                QS_CUDA(cudaMemsetAsync(L.cnt2, 0, 16, st), "memset");
                QS_CUDA(cudaMemsetAsync(L.hist, 0, HIST_LEN * 8, st), "memset");
                QS_CUDA(cudaMemsetAsync(L.stats_out, 0, 32, st), "memset");
                QS_TRY(qs_lsh_compact_buckets(L.sids, L.bstart, L.bsize, L.btab, nb, L.emask,
                                              L.sids2, L.bstart2, L.bsize2, L.btab2, L.cnt2, L.hist,
                                              HIST_LEN, L.big, L.big_cap, L.stats_out, L.trans,
                                              L.trans_bytes, stv));
                uint64_t c2[2];
                QS_TRY(d2h(c2, L.cnt2, 16, st));
                compacted = true;
                QS_TRY(pairs(2, nullptr, L.sids2, L.bstart2, L.bsize2, L.btab2, c2[0], nullptr,
                             distinct, dummy));
            } else {
                QS_TRY(pairs(2, L.emask, L.sids, L.bstart, L.bsize, L.btab, nb, nullptr, distinct,
                             dummy));
            }
        }
        // exact sims of the lazily counted pairs that survived
        if (matched) QS_TRY(qs_lsh_complete_sims(pk, ps, rest, matched, L.rkeys, t, stv));
    }
    // bucket statistics (the compaction pass already produced them for p == 1)
    if (!compacted) {
        QS_CUDA(cudaMemsetAsync(L.hist, 0, HIST_LEN * 8, st), "memset");
        QS_CUDA(cudaMemsetAsync(L.stats_out, 0, 32, st), "memset");
        QS_TRY(qs_lsh_bucket_stats(L.sids, L.bstart, L.bsize, nb, emask, L.edges, p, L.hist,
                                   HIST_LEN, L.big, L.big_cap, L.stats_out, stv));
    }
    uint64_t so[4];
    QS_TRY(d2h(so, L.stats_out, 32, st));
    const uint64_t looks = so[0], pieces = so[1], n_big = so[2], mx = so[3];
    if (n_big > L.big_cap) {
        qs::set_error("bucket size overflow list too small");
        return QS_ERR_CUDA;
    }
    std::vector<uint64_t> hist(HIST_LEN);
    std::vector<uint32_t> big(n_big);
    QS_TRY(d2h(hist.data(), L.hist, HIST_LEN * 8, st));
    if (n_big) QS_TRY(d2h(big.data(), L.big, n_big * 4, st));
    // sorted triplets
    if (matched) {
        uint32_t bits = 0;
        while ((n >> bits) && bits < 32) ++bits;
        QS_TRY(qs_lsh_finalize(pk, ps, matched, 32 + std::max<uint32_t>(1, bits), triplets,
                               L.trans, L.trans_bytes, stv));
    }
    QS_CUDA(cudaStreamSynchronize(st), "stream sync");
    // SearchStats (lsh_search.py:295-302)
    const uint64_t singles = heads - nb;
    stats->lookups_total = looks;
    stats->distinct_pairs = distinct;
    stats->emitted_triplets = matched;
    stats->filtered_fingerprints = n_ex;
    stats->n_queries = n - n_ex;
    stats->n_buckets = pieces + singles;
    stats->max_bucket = std::max<uint64_t>(mx, singles ? 1 : 0);
    hist[1] += singles;
    stats->top_bucket_mass = top_mass(hist, big, stats->n_buckets, n * t);
    if (needed) *needed = matched;
    return QS_OK;
}

int begin(uint64_t n, uint32_t t, uint32_t m, uint32_t partitions, double occ, uint64_t pair_cap,
          void* ws, size_t ws_bytes, qs_search_stats* stats, Layout& L, Sizes& s,
          std::vector<uint64_t>& edges) {
    QS_ARG(t >= 1, "tables must be >= 1");
    QS_ARG(m >= 1 && m <= t, "min_matches must be in [1, tables]");
    QS_ARG(partitions >= 1, "partitions must be >= 1");
    QS_ARG(occ <= 1.0, "occurrence_threshold must be in (0, 1]");
    QS_ARG(n < (1ull << 32), "more than 2**32 fingerprints are not supported");
    QS_ARG(stats != nullptr, "stats must not be NULL");
    memset(stats, 0, sizeof(*stats));
    stats->n_fingerprints = n;
    if (n == 0) return QS_OK;
    edges = partition_edges(n, partitions);
    uint64_t peak = 0;
    for (size_t i = 1; i < edges.size(); ++i) peak = std::max(peak, edges[i] - edges[i - 1]);
    stats->peak_table_entries = peak * t;
    stats->n_partitions = (uint32_t)(edges.size() - 1);
    s = sizes_of(n, t, pair_cap);
    Bump a{(uint8_t*)ws, ws_bytes, 0};
    carve(a, s, L, stats->n_partitions);
    QS_ARG(ws != nullptr && a.ok, "search workspace too small (%zu bytes, need %zu)", ws_bytes,
           qs_lsh_search_ws_bytes(n, t, pair_cap, partitions));
    return QS_OK;
}

}  // namespace

extern "C" {

size_t qs_lsh_search_ws_bytes(uint64_t n, uint32_t t, uint64_t pair_cap, uint32_t partitions) {
    const Sizes s = sizes_of(n, t, pair_cap);
    Bump a{nullptr, 0, 0};
    Layout L;
    carve(a, s, L, (uint32_t)std::min<uint64_t>(std::max(partitions, 1u), std::max<uint64_t>(1, n)));
    return a.off + 256;
}

int qs_lsh_search(const uint64_t* sigs_dev, uint64_t n, uint32_t t, uint32_t m,
                  uint64_t exclusion_windows, double occurrence_threshold, uint32_t partitions,
                  uint8_t* triplets_dev, uint64_t pair_cap, uint64_t* needed_out,
                  qs_search_stats* stats, void* ws_dev, size_t ws_bytes, void* stream) {
    Layout L;
    Sizes s;
    std::vector<uint64_t> edges;
    if (needed_out) *needed_out = 0;
    QS_TRY(begin(n, t, m, partitions, occurrence_threshold, pair_cap, ws_dev, ws_bytes, stats, L,
                 s, edges));
    if (n == 0) return QS_OK;
    QS_TRY(qs_lsh_prep(sigs_dev, n, t, L.keys, L.rkeys, L.tags, stream));
    return run(L, s, m, exclusion_windows, occurrence_threshold, (uint32_t)(edges.size() - 1),
               edges, triplets_dev, needed_out, stats, (cudaStream_t)stream);
}

size_t qs_lsh_search_bits_ws_bytes(uint64_t n, uint32_t d, uint32_t t, uint32_t k_half,
                                   uint64_t pair_cap, uint32_t partitions) {
    const uint64_t F = (uint64_t)t * k_half;
    return qs_lsh_search_ws_bytes(n, t, pair_cap, partitions) +
           (((size_t)d * F * 8 + 255) & ~(size_t)255) +
           ((qs_minmax_plan_bytes(d, (uint32_t)F) + 255) & ~(size_t)255);
}

int qs_lsh_search_bits(const uint32_t* bits_dev, uint64_t n, uint32_t K, uint32_t d,
                       uint64_t seed, uint32_t t, uint32_t k_half, uint32_t m,
                       uint64_t exclusion_windows, double occurrence_threshold,
                       uint32_t partitions, uint8_t* triplets_dev, uint64_t pair_cap,
                       uint64_t* needed_out, qs_search_stats* stats, void* ws_dev,
                       size_t ws_bytes, void* stream) {
    QS_ARG(K >= 1, "fingerprints must have at least one set bit");
    QS_ARG(k_half >= 1 && d >= 1, "bad mapping geometry");
    const uint64_t F = (uint64_t)t * k_half;
    const size_t head = (((size_t)d * F * 8 + 255) & ~(size_t)255) +
                        ((qs_minmax_plan_bytes(d, (uint32_t)F) + 255) & ~(size_t)255);
    QS_ARG(ws_bytes >= head, "search workspace too small");
    uint64_t* values = (uint64_t*)ws_dev;
    void* plan = (uint8_t*)ws_dev + (((size_t)d * F * 8 + 255) & ~(size_t)255);
    void* rest = (uint8_t*)ws_dev + head;
    Layout L;
    Sizes s;
    std::vector<uint64_t> edges;
    if (needed_out) *needed_out = 0;
    QS_TRY(begin(n, t, m, partitions, occurrence_threshold, pair_cap, rest, ws_bytes - head, stats,
                 L, s, edges));
    if (n == 0) return QS_OK;
    // the hash mapping and its probe plan (minmax_hash.gen_hash_mapping,
    // minmax_hash.py:73-90), then Min-Max signatures straight into the layout
    QS_TRY(qs_gen_hash_mapping(values, d, (uint32_t)F, seed, stream));
    QS_TRY(qs_minmax_plan(values, d, (uint32_t)F, plan, stream));
    QS_CUDA(cudaMemsetAsync(L.counts, 0, 8, (cudaStream_t)stream), "memset");
    QS_TRY(qs_minmax_signatures_search(bits_dev, n, K, plan, d, t, k_half, nullptr, L.keys,
                                       L.rkeys, L.tags, (uint32_t*)L.counts, stream));
    uint32_t bad = 0;
    QS_TRY(d2h(&bad, L.counts, 4, (cudaStream_t)stream));
    if (bad) {
        qs::set_error("fingerprint bit index out of range for mapping");
        return QS_ERR_ARG;
    }
    return run(L, s, m, exclusion_windows, occurrence_threshold, (uint32_t)(edges.size() - 1),
               edges, triplets_dev, needed_out, stats, (cudaStream_t)stream);
}

}  // extern "C"
