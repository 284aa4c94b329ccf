/*
 * quakescan-b200 — C ABI of the B200 (sm_100a) hot path of the FAST-style
 * waveform similarity search (reference: quakescan 0.1.0, arXiv 1803.09835).
 *
 * Every entry point takes plain pointers and sizes (no torch or CUDA types in
 * the signatures; `stream` is a cudaStream_t passed as void*, NULL = legacy
 * default stream).  Pointers named *_dev are device memory; the caller owns
 * every buffer (outputs are preallocated by the caller, scratch comes from a
 * caller workspace sized by the matching *_bytes query).  Calls are
 * stream-ordered and never synchronize the device unless documented.
 *
 * Return value: QS_OK (0) or an error code; qs_last_error() returns the text
 * of the last error on the calling thread.  The Python host layer maps
 * QS_ERR_ARG -> ParameterError, QS_ERR_DATA -> DataError, QS_ERR_OOM ->
 * MemoryError, QS_ERR_CUDA -> RuntimeError (reference error taxonomy,
 * pkg/src/quakescan/errors.py:1-29).  Nothing aborts the process.
 *
 * Reference interfaces replaced are cited per function as file:line under
 * /root/reference/pkg/src/quakescan/.
 */
#ifndef QUAKESCAN_B200_H
#define QUAKESCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QS_OK 0
#define QS_ERR_ARG 1   /* bad shape / range / parameter      -> ParameterError */
#define QS_ERR_OOM 2   /* device allocation failed             -> MemoryError    */
#define QS_ERR_CUDA 3  /* CUDA runtime / launch failure        -> RuntimeError   */
#define QS_ERR_DATA 4  /* input data unusable (e.g. bit >= d)  -> DataError      */
#define QS_ERR_CAPACITY 5 /* caller's output capacity too small; *needed_out holds
                             the count to size it for (re-call with that)  */

/* ---------------------------------------------------------------- library */
const char* qs_version(void);
const char* qs_last_error(void);
/* Writes "name|sm_major.minor|n_sms|hbm_bytes" of the current device. */
int qs_device_info(char* buf, size_t len);

/* ------------------------------------------------- host <-> device transfer
 * Helpers of the host-buffer entry points: the reference's
 * search_fingerprints (lsh_search.py:314-333) and fingerprint_series
 * (fingerprint.py:581-623) take host arrays, so their copy is part of the
 * call here (csrc/qs_host.cu). */
/* 1 when host_ptr lies in page-locked memory (cudaHostAlloc / cudaHostRegister:
 * DMA straight from the caller's array), 0 for pageable memory. */
int qs_host_ptr_pinned(const void* host_ptr);
/* dst_host[i] = min(src_host[i], 65535): bit indices narrowed while they are
 * staged (valid for d <= 65535: a saturated value is >= d and is flagged by
 * the signature kernel's range check).  Host function, thread-safe. */
int qs_host_pack_u16(const uint32_t* src_host, uint16_t* dst_host, uint64_t count);
/* The same with 12-bit fields (value i in bits [12 i, 12 i + 12) of the byte
 * stream, ceil(1.5 count) bytes) for d <= 4096; *fits_out = 0 when a value
 * above 4095 was seen (the caller then uses the uint16 route for that chunk).
 * Host function, thread-safe. */
int qs_host_pack_u12(const uint32_t* src_host, uint8_t* dst_host, uint64_t count, int* fits_out);
/* dst_host[i] = (float)src_host[i]; *exact_out = 1 when every value widens
 * back to itself (then a float32 upload gives the chain the same samples),
 * 0 otherwise (NaN, overflow, inexact).  Host function, thread-safe. */
int qs_host_pack_f32(const double* src_host, float* dst_host, uint64_t count, int* exact_out);
/* dst_dev[i] = src_dev[i] (uint16 -> uint32), both 16-byte aligned. */
int qs_bits_widen_u16(const uint16_t* src_dev, uint32_t* dst_dev, uint64_t count, void* stream);
/* dst_dev[i] = field i of the 12-bit stream (src 4-byte, dst 16-byte aligned). */
int qs_bits_widen_u12(const uint8_t* src_dev, uint32_t* dst_dev, uint64_t count, void* stream);
int qs_memcpy_h2d_async(void* dst_dev, const void* src_host, size_t bytes, void* stream);
int qs_memcpy_d2h_async(void* dst_host, const void* src_dev, size_t bytes, void* stream);

/* ------------------------------------------------------------ Min-Max hash */

/* values_dev[x * n_funcs + j] = fmix64(((x + 1) * GOLDEN64) ^ (seed + j)).
 * Replaces minmax_hash.gen_hash_mapping (minmax_hash.py:73-90). */
int qs_gen_hash_mapping(uint64_t* values_dev, uint32_t d, uint32_t n_funcs,
                        uint64_t seed, void* stream);

/* Probe plan of a mapping: for every hash column the element indices in
 * ascending value order plus the sorted values (rank-major layout).  Built
 * once per mapping; consumed by qs_minmax_signatures. */
size_t qs_minmax_plan_bytes(uint32_t d, uint32_t n_funcs);
int qs_minmax_plan(const uint64_t* values_dev, uint32_t d, uint32_t n_funcs,
                   void* plan_dev, void* stream);

/* Min-Max signatures of rows [0, n) of bits_dev (n, K) uint32 -> out_dev (n, t)
 * uint64, bit-identical to _sigcore.gen_signatures_range (_sigcore.pyx:32-85):
 * out[r, i] = fold(min over set bits of V[:, i*kh + j] for j < kh, then max ...).
 * A bit index >= d sets *bad_dev (uint32, device) to 1 and that row is
 * unspecified (the Python layer validates first, minmax_hash.py:107-108). */
int qs_minmax_signatures(const uint32_t* bits_dev, uint64_t n, uint32_t K,
                         const void* plan_dev, uint32_t d, uint32_t t, uint32_t k_half,
                         uint64_t* out_dev, uint32_t* bad_dev, void* stream);

/* Same computation, search layout: keys_dev (t, n) uint64 table-major and
 * rkeys_dev (n, t) uint64 row-major hold mix64(sig) (a bijection of the
 * signature word, so bucket equality is unchanged) and tags_dev
 * [2][n][ceil(t/32)][8] uint32 the bit-sliced 16-bit tags (plane p of word w
 * = bit p of the tags of tables 32w..32w+31; planes 0-7 in the first half,
 * 8-15 in the second) used for exact first-colliding-table dedup.
 * sigs_dev (n, t) and keys_dev may be NULL (a table-sharded rank rebuilds
 * its own tables' keys from the gathered rkeys). */
int qs_minmax_signatures_search(const uint32_t* bits_dev, uint64_t n, uint32_t K,
                                const void* plan_dev, uint32_t d, uint32_t t,
                                uint32_t k_half, uint64_t* sigs_dev, uint64_t* keys_dev,
                                uint64_t* rkeys_dev, uint32_t* tags_dev, uint32_t* bad_dev,
                                void* stream);

/* The same for rows [row0, row0 + nrows) of the n-row layout (bits_dev,
 * keys_dev, rkeys_dev, tags_dev and sigs_dev all address the full n rows):
 * lets a caller overlap the signatures of landed rows with the host->device
 * copy of later ones. */
int qs_minmax_signatures_search_rows(const uint32_t* bits_dev, uint64_t n, uint64_t row0,
                                     uint64_t nrows, uint32_t K, const void* plan_dev,
                                     uint32_t d, uint32_t t, uint32_t k_half, uint64_t* sigs_dev,
                                     uint64_t* keys_dev, uint64_t* rkeys_dev, uint32_t* tags_dev,
                                     uint32_t* bad_dev, void* stream);

/* HOST-buffer drop-in for the reference's native plugin point
 * `_core.gen_signatures_range(bits, values, t, k_half, out, start, stop)`
 * (minmax_hash.py:24-30 selects it; _sigcore.pyx:32-36 defines it): fills
 * out[start:stop] (n_rows, t) from bits (n_rows, K) and values (d, F).
 * Stages through device memory on an internal stream; synchronous.  The
 * stream, device buffers and the uploaded mapping + probe plan persist
 * across calls (the reference calls once per worker chunk with one mapping):
 * the mapping is re-uploaded when its address, shape or a strided digest of
 * its values changes.  Calls are serialised internally (thread-safe). */
int qs_gen_signatures_range(const uint32_t* bits, uint64_t n_rows, uint32_t K,
                            const uint64_t* values, uint32_t d, uint32_t F,
                            int32_t t, int32_t k_half, uint64_t* out,
                            uint64_t start, uint64_t stop);

/* ------------------------------------------------------------- LSH search
 * The search (lsh_search.search_signatures, lsh_search.py:222-303) runs as the
 * stage sequence below, orchestrated by the Python host layer which owns all
 * buffers.  Layouts: keys (t, n) / rkeys (n, t) uint64 mixed signature words;
 * tags [2][n][W][8] uint32, W = ceil(t/32).  A bucket list is (bstart = offset
 * of the bucket's first member in the member-id array, bsize, btab = table). */

/* Row-major signatures (n, t) -> keys + rkeys + tags.  Used when the caller
 * hands in signatures (search_signatures) rather than bits. */
int qs_lsh_prep(const uint64_t* sigs_dev, uint64_t n, uint32_t t, uint64_t* keys_dev,
                uint64_t* rkeys_dev, uint32_t* tags_dev, void* stream);

/* Bucket construction: per table, sort (key, id) so equal keys are contiguous
 * with ascending ids (the stable argsort of lsh_search.py:157-164).
 * ids_out_dev (t, n) uint32; keys_out_dev (t, n) uint64 sorted keys. */
size_t qs_lsh_bucket_ws_bytes(uint64_t n, uint32_t t);
int qs_lsh_build_buckets(const uint64_t* keys_dev, uint64_t n, uint32_t t,
                         uint64_t* keys_out_dev, uint32_t* ids_out_dev,
                         void* ws_dev, size_t ws_bytes, void* stream);

/* Bucket listing (lsh_search.py:167-172 run lengths): non-singleton buckets
 * of all tables.  Call first with bstart_dev == NULL: counts_dev[0] = number
 * of non-singleton buckets, counts_dev[1] = number of buckets (all tables);
 * then with arrays of that capacity to fill them.  btab_dev receives each
 * bucket's table: table_ids_dev[local table] when table_ids_dev is given (a
 * table-sharded rank passes the global ids of its tables), else the local
 * index. */
size_t qs_lsh_list_ws_bytes(uint64_t n, uint32_t t);
int qs_lsh_list_buckets(const uint64_t* skeys_dev, uint64_t n, uint32_t t,
                        uint64_t* bstart_dev, uint32_t* bsize_dev, uint32_t* btab_dev,
                        const uint32_t* table_ids_dev, uint64_t* counts_dev, void* ws_dev,
                        size_t ws_bytes, void* stream);

/* Bucket construction for the search: the member ids of qs_lsh_build_buckets
 * in ids_out_dev (t, n) uint32, plus flags_out_dev (t, n) uint8 — bit 0:
 * first member of its bucket, bit 1: last member — in place of the sorted-key
 * array (the caller never sees it; it lives in the workspace). */
size_t qs_lsh_bucket_flags_ws_bytes(uint64_t n, uint32_t t);
int qs_lsh_build_bucket_flags(const uint64_t* keys_dev, uint64_t n, uint32_t t,
                              uint32_t* ids_out_dev, uint8_t* flags_out_dev,
                              void* ws_dev, size_t ws_bytes, void* stream);

/* qs_lsh_list_buckets over the flag bytes of qs_lsh_build_bucket_flags. */
size_t qs_lsh_list_flags_ws_bytes(uint64_t n, uint32_t t);
int qs_lsh_list_buckets_flags(const uint8_t* flags_dev, uint64_t n, uint32_t t,
                              uint64_t* bstart_dev, uint32_t* bsize_dev, uint32_t* btab_dev,
                              const uint32_t* table_ids_dev, uint64_t* counts_dev,
                              void* ws_dev, size_t ws_bytes, void* stream);

/* SearchStats bucket fields (lsh_search.py:70-109, 295-302): lookups_total
 * (counted before the canonical/dt/exclusion masks, :192-194), the sizes of
 * the per-partition-table buckets (histogram of sizes < hist_len into
 * hist_dev; larger sizes appended to big_dev), n_buckets and the max bucket.
 * out_dev: [0] lookups, [1] partition-table buckets from non-singleton lists,
 * [2] number of big sizes, [3] max size.  excluded_dev (n bytes) may be NULL;
 * edges_dev holds the partition_bounds edges (p + 1 values). */
int qs_lsh_bucket_stats(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                        const uint32_t* bsize_dev, uint64_t n_nonsingle,
                        const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p,
                        uint64_t* hist_dev, uint32_t hist_len, uint32_t* big_dev,
                        uint64_t big_cap, uint64_t* out_dev, void* stream);

/* Remove excluded members from every bucket (single partition only; an
 * excluded fingerprint can never be part of a counted pair there).  Writes
 * the compacted member ids and bucket list (buckets keeping >= 2 members);
 * counts_dev[0] = buckets kept, counts_dev[1] = members kept.  When hist_dev
 * is not NULL the same pass also produces the single-partition bucket
 * statistics of qs_lsh_bucket_stats (hist/big/stats_out_dev as there,
 * stats_out_dev zeroed by the caller). */
size_t qs_lsh_compact_ws_bytes(uint64_t n_nonsingle);
int qs_lsh_compact_buckets(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                           const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t nb,
                           const uint8_t* excluded_dev, uint32_t* sids2_dev,
                           uint64_t* bstart2_dev, uint32_t* bsize2_dev, uint32_t* btab2_dev,
                           uint64_t* counts_dev, uint64_t* hist_dev, uint32_t hist_len,
                           uint32_t* big_dev, uint64_t big_cap, uint64_t* stats_out_dev,
                           void* ws_dev, size_t ws_bytes, void* stream);

/* Candidate-pair enumeration + exact collision counting + >= m threshold
 * (replaces _collect_pairs + the count filter, lsh_search.py:175-219, 261, 281).
 * Every unordered pair sharing a bucket is handled only in the bucket of its
 * FIRST colliding table (exact dedup: bit-sliced tag comparison confirmed on
 * the 64-bit keys), so each distinct pair is seen once and sim = number of
 * tables whose keys agree.  Masks: canonical c < q, q - c > excl, exclusion /
 * partition rule of lsh_search.py:256-287.  mode 0: count distinct pairs and
 * emit sim >= m; 1: emit only; 2: count only.  Emitted records are
 * (sortkey = (q - c) << 32 | c, sim) into out_key/out_sim (capacity cap; the
 * true count is always added to counters_dev[1] so the caller can grow and
 * retry); counters_dev[0] += distinct pairs.
 * out_rest_dev (mode 1 only, may be NULL): lazy counts — a pair's count stops
 * being confirmed once it reaches m; the candidate tables left unexamined are
 * written as ceil(t/32) uint32 bit words per emitted pair and out_sim holds a
 * partial count (>= m) until qs_lsh_complete_sims finishes it. */
size_t qs_lsh_pairs_ws_bytes(uint64_t n_nonsingle);
int qs_lsh_pairs(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                 const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t n_nonsingle,
                 const uint64_t* rkeys_dev, const uint32_t* tags_dev, uint64_t n, uint32_t t,
                 uint32_t m, uint64_t excl, const uint8_t* excluded_dev,
                 const uint64_t* edges_dev, uint32_t p, int mode,
                 uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev,
                 uint64_t cap, unsigned long long* counters_dev, void* ws_dev, size_t ws_bytes,
                 void* stream);

/* qs_lsh_pairs restricted to the buckets of tables [table_lo, table_hi)
 * (t <= 128; the first-table rule still looks at every earlier table).  core_count_dev (mode 1 only, may be
 * NULL): the member lists are core-first (qs_lsh_core_first) and bucket b's
 * first core_count_dev[b] members are fingerprints already known to exceed
 * the occurrence limit; pairs of two of them are skipped — they change no
 * output of the occurrence-filtered search (partitions == 1): both endpoints
 * are core, hence excluded, whatever their count (lsh_search.py:256-287). */
int qs_lsh_pairs_ex(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                    const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t n_nonsingle,
                    const uint64_t* rkeys_dev, const uint32_t* tags_dev, uint64_t n, uint32_t t,
                    uint32_t m, uint64_t excl, const uint8_t* excluded_dev,
                    const uint64_t* edges_dev, uint32_t p, int mode,
                    uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev,
                    uint64_t cap, unsigned long long* counters_dev, void* ws_dev, size_t ws_bytes,
                    uint32_t table_lo, uint32_t table_hi, const uint32_t* core_count_dev,
                    void* stream);

/* Core-first member lists for qs_lsh_pairs_ex: for every bucket of a table
 * >= table_lo, a stable partition of its ids (core_dev[id] != 0 first) into
 * sids_out_dev at the same positions, and the number of core members in
 * core_count_dev[b] (0 for buckets of earlier tables, which are not copied). */
int qs_lsh_core_first(const uint32_t* sids_dev, const uint64_t* bstart_dev,
                      const uint32_t* bsize_dev, const uint32_t* btab_dev, uint64_t n_nonsingle,
                      uint32_t table_lo, const uint8_t* core_dev, uint32_t* sids_out_dev,
                      uint32_t* core_count_dev, void* stream);

/* Number of core-core pairs qs_lsh_pairs_ex (mode 1, core-first lists of
 * tables >= table_lo) leaves out, added to *out_dev (measurement: the pairs
 * the pass compares = all pairs of its buckets minus these). */
int qs_lsh_core_skipped(const uint32_t* bsize_dev, const uint32_t* btab_dev,
                        const uint32_t* core_count_dev, uint64_t n_nonsingle, uint32_t t,
                        uint32_t m, uint32_t table_lo, unsigned long long* out_dev, void* stream);

/* Exact counts of lazily counted pairs (see qs_lsh_pairs): pair_sim_dev[i] +=
 * the agreeing tables among rest_dev[i * ceil(t/32) ...]. */
int qs_lsh_complete_sims(const uint64_t* pair_key_dev, uint32_t* pair_sim_dev,
                         const uint32_t* rest_dev, uint64_t n_pairs, const uint64_t* rkeys_dev,
                         uint32_t t, void* stream);

/* Occurrence filter (lsh_search.py:256-274) from the matched pairs of a
 * filter-free enumeration: per partition, degree over within-partition
 * matched pairs, core = degree > thr * |partition|, excluded = core plus the
 * matched within-partition neighbours of core.  excluded_dev (n bytes) is
 * written; counters_dev[0] += number excluded.  Workspace: n * 4 bytes. */
int qs_lsh_occurrence_filter(const uint64_t* pair_key_dev, const uint32_t* pair_sim_dev,
                             uint64_t n_pairs, uint64_t n, double threshold,
                             const uint64_t* edges_dev, uint32_t p, uint8_t* excluded_dev,
                             unsigned long long* counters_dev, void* ws_dev, void* stream);

/* The same filter in three steps, for table-sharded searches whose matched
 * pairs are spread over ranks: (1) degree_dev (n uint32, zeroed by the caller)
 * += within-partition matched-pair degrees — sum it over ranks; (2) mark:
 * excluded_dev = 2 for core, 1 for matched neighbours of core, else 0 — take
 * the elementwise max over ranks; (3) finish: normalise to 0/1 and
 * counters_dev[0] += number excluded. */
int qs_lsh_occ_degree(const uint64_t* pair_key_dev, uint64_t n_pairs, const uint64_t* edges_dev,
                      uint32_t p, uint32_t* degree_dev, void* stream);
int qs_lsh_occ_mark(const uint64_t* pair_key_dev, uint64_t n_pairs, const uint32_t* degree_dev,
                    uint64_t n, double threshold, const uint64_t* edges_dev, uint32_t p,
                    uint8_t* excluded_dev, void* stream);
int qs_lsh_occ_finish(uint8_t* excluded_dev, uint64_t n, unsigned long long* counters_dev,
                      void* stream);

/* Matched pairs that survive the exclusion rule (pass-2 emission of
 * lsh_search.py:276-287), appended to out_* with *counter_dev as cursor.
 * rest_dev (may be NULL): the lazy-count words of each pair (rest_words per
 * pair), carried along into out_rest_dev. */
int qs_lsh_filter_pairs(const uint64_t* pair_key_dev, const uint32_t* pair_sim_dev,
                        const uint32_t* rest_dev, uint32_t rest_words, uint64_t n_pairs,
                        const uint8_t* excluded_dev, const uint64_t* edges_dev, uint32_t p,
                        uint64_t* out_key_dev, uint32_t* out_sim_dev, uint32_t* out_rest_dev,
                        unsigned long long* counter_dev, void* stream);

/* Sort matched pairs by (dt, idx1) (lsh_search.py:291) and pack them into
 * TRIPLET_DTYPE records (<u8 dt, <u8 idx1, <u4 sim; 20 bytes, :38).
 * key_bits = 32 + b where both dt and idx1 are < 2^b (b = bit length of n):
 * digits that are zero in both halves are not sorted on. */
size_t qs_sort_pairs_ws_bytes(uint64_t n);
int qs_lsh_finalize(uint64_t* pair_key_dev, uint32_t* pair_sim_dev, uint64_t n_pairs,
                    uint32_t key_bits, uint8_t* triplets_dev, void* ws_dev, size_t ws_bytes,
                    void* stream);

/* Channel combine / triplet sort (align.py:87-140): n packed TRIPLET_DTYPE
 * records (any order, several channels concatenated) are sorted by
 * (dt, idx1); equal window pairs have their sims summed and sums below
 * threshold dropped (threshold 0: plain sort, duplicates kept).  out_dev holds
 * up to n records; *count_dev receives the number written.  key_bits = bits of
 * (dt << 32 | idx1) that can be non-zero (64 if unknown).  QS_ERR_DATA when a
 * dt or idx1 does not fit 32 bits. */
size_t qs_triplets_combine_ws_bytes(uint64_t n);
int qs_triplets_combine(const uint8_t* triplets_dev, uint64_t n, uint32_t threshold,
                        uint32_t key_bits, uint8_t* out_dev, uint64_t* count_dev, void* ws_dev,
                        size_t ws_bytes, void* stream);

/* ------------------------------------------------- one-call search entries
 * The whole search in one call for non-Python callers: the same stage
 * sequence the Python host layer runs (lsh_search.py run_search), every
 * buffer carved from ONE caller workspace (no cudaMalloc inside), the stream
 * synchronised only where a count sizes the next stage.  Results are
 * identical to the stage-by-stage path and to the reference. */

/* SearchStats (lsh_search.py:70-109); lookups_per_query and selectivity are
 * derived (lookups_total / n_queries, 2 * distinct_pairs / n^2). */
typedef struct qs_search_stats {
    uint64_t n_fingerprints;
    uint64_t n_queries;
    uint64_t lookups_total;
    uint64_t distinct_pairs;
    uint64_t emitted_triplets;
    uint64_t filtered_fingerprints;
    uint64_t peak_table_entries;
    uint64_t n_buckets;
    uint64_t max_bucket;
    double top_bucket_mass;
    uint32_t n_partitions;  /* len(partition_bounds(n, partitions)) */
} qs_search_stats;

/* search_signatures(sigs, SearchConfig(tables=t, min_matches=m,
 * partitions=partitions, occurrence_threshold=occurrence_threshold or None
 * when <= 0), exclusion_windows) (lsh_search.py:222-303).  sigs_dev (n, t)
 * uint64 row-major; triplets_dev receives the emitted TRIPLET_DTYPE records
 * (20 B each, sorted by (dt, idx1)), stats->emitted_triplets of them.
 * pair_cap bounds the matched pairs of an enumeration pass (and the output):
 * QS_ERR_CAPACITY with *needed_out = the pairs found when it is too small.
 * Workspace: qs_lsh_search_ws_bytes(n, t, pair_cap, partitions). */
size_t qs_lsh_search_ws_bytes(uint64_t n, uint32_t t, uint64_t pair_cap, uint32_t partitions);
int qs_lsh_search(const uint64_t* sigs_dev, uint64_t n, uint32_t t, uint32_t m,
                  uint64_t exclusion_windows, double occurrence_threshold, uint32_t partitions,
                  uint8_t* triplets_dev, uint64_t pair_cap, uint64_t* needed_out,
                  qs_search_stats* stats, void* ws_dev, size_t ws_bytes, void* stream);

/* search_fingerprints(fps, cfg, mapping=None) (lsh_search.py:314-333) from
 * set-bit indices bits_dev (n, K) uint32: the hash mapping
 * gen_hash_mapping(d, t, 2 * k_half, seed) and its probe plan are built in the
 * workspace, signatures go straight into the search layout, then the search
 * as qs_lsh_search.  A bit index >= d -> QS_ERR_ARG (ParameterError).
 * Workspace: qs_lsh_search_bits_ws_bytes(n, d, t, k_half, pair_cap, partitions). */
size_t qs_lsh_search_bits_ws_bytes(uint64_t n, uint32_t d, uint32_t t, uint32_t k_half,
                                   uint64_t pair_cap, uint32_t partitions);
int qs_lsh_search_bits(const uint32_t* bits_dev, uint64_t n, uint32_t K, uint32_t d,
                       uint64_t seed, uint32_t t, uint32_t k_half, uint32_t m,
                       uint64_t exclusion_windows, double occurrence_threshold,
                       uint32_t partitions, uint8_t* triplets_dev, uint64_t pair_cap,
                       uint64_t* needed_out, qs_search_stats* stats, void* ws_dev,
                       size_t ws_bytes, void* stream);

/* Zero-phase band-pass (scipy.signal.sosfiltfilt with padtype "odd", as
 * reference ingest.py:74-84 calls it): sos_host (n_sections x 6, a0 == 1) and
 * zi_host (n_sections x 2, scipy.signal.sosfilt_zi) are small host arrays;
 * x_dev / out_dev hold n float64 samples; pad = the odd-extension length.
 * QS_ERR_ARG when n <= pad (scipy's ValueError). */
size_t qs_sosfiltfilt_ws_bytes(uint64_t n, uint64_t pad);
int qs_sosfiltfilt(const double* x_dev, uint64_t n, const double* sos_host, uint32_t n_sections,
                   const double* zi_host, uint64_t pad, double* out_dev, void* ws_dev,
                   size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ fingerprinting
 * Chain of fingerprint.fingerprint_series (fingerprint.py:581-623).  Float64
 * compute with float32 storage at the reference's rounding points
 * (spectrogram :148-149, images :239-241, coefficients :334). */

/* Band-limited log-power STFT (fingerprint.py:136-151 restricted to the band
 * rows): out[c, b] = float32(log10(|sum_j x[c*hop + j] tw[b, j]|^2 + 1e-12))
 * for c < n_cols, where tw (nb, frame, 2) float64 = hanning taper times the
 * DFT twiddles of the band bins.  Samples are float64 (x_is_f32 = 0) or
 * float32 widened exactly (x_is_f32 = 1). */
int qs_fp_band_stft(const void* x_dev, int x_is_f32, uint64_t n_samples, uint32_t frame,
                    uint32_t hop, uint64_t n_cols, uint32_t nb, const double* tw_dev,
                    float* out_dev, void* stream);

/* Per fingerprint window (iter_image_batches / iter_coeff_batches /
 * topk_bits, fingerprint.py:198-243, 271-335, 433-466): band rows ->
 * area-resampled image (CSR weights w_f over band rows, w_t per window width
 * in [wmin, wmax]) -> 2-D Haar (sched: n_levels (h, w, mode) triples, mode
 * bit 0 = row pass, bit 1 = column pass) -> coefficients.  Windows are
 * widx_dev[0..n_win) or win0 + [0, n_win).  mode 0: images (n_win, F, T) f32;
 * 1: coefficients (n_win, F*T) f32; 2: coefficients column-major (F*T, n_win);
 * 3: top_k sign bits (n_win, top_k) u32 using med/mad.  A non-finite
 * coefficient sets bit 0 of *flags_dev (-> DataError). */
int qs_fp_windows(const float* band_dev, uint64_t n_cols, uint32_t nb, const int64_t* widx_dev,
                  uint64_t win0, uint64_t n_win, uint64_t lag, uint64_t win, uint32_t frame,
                  uint32_t hop, const int32_t* wf_off, const int32_t* wf_idx, const double* wf_val,
                  const int32_t* wt_off, const int32_t* wt_idx, const double* wt_val,
                  uint32_t wmin, uint32_t wmax, uint32_t F, uint32_t T, const int32_t* sched_dev,
                  uint32_t n_levels, int mode, const double* med_dev, const double* mad_dev,
                  uint32_t top_k, void* out_dev, uint32_t* flags_dev, void* stream);

/* Median and MAD of each of n_coeffs columns of S float32 values (column-major
 * (n_coeffs, S)), float64 results exactly as np.median / np.median(|x - med|)
 * (estimate_mad, fingerprint.py:376-384).  ws_dev: 2 * n_coeffs doubles. */
int qs_fp_mad(const float* cols_dev, uint32_t n_coeffs, uint64_t S, double* med_dev,
              double* mad_dev, double* ws_dev, void* stream);

/* Transpose of a (rows, cols) float32 row-major matrix into (cols, rows): the
 * MAD sample pass writes one coefficient row per sampled window (coalesced)
 * and qs_fp_mad reads one column per coefficient (estimate_mad,
 * fingerprint.py:364-384 stacks the sampled windows the same way). */
int qs_fp_transpose_f32(const float* src_dev, uint64_t rows, uint32_t cols, float* dst_dev,
                        void* stream);

/* topk_bits (fingerprint.py:433-466) of B rows of n coefficients (float32, or
 * float64 with is_f64). */
int qs_fp_topk_bits(const void* coeffs_dev, int is_f64, uint64_t B, uint32_t n,
                    const double* med_dev, const double* mad_dev, uint32_t top_k, uint32_t* out_dev,
                    uint32_t* flags_dev, void* stream);

/* haar2d / ihaar2d (fingerprint.py:271-323) of B float64 (H, W) images in place. */
int qs_fp_haar2d(double* data_dev, uint64_t B, uint32_t H, uint32_t W, const int32_t* sched_dev,
                 uint32_t n_levels, int inverse, void* stream);

/* normalize (fingerprint.py:425-430): (c - median)/MAD in float64, 0 where
 * MAD == 0; B rows of n coefficients, float32 or float64 (is_f64).  med_dev /
 * mad_dev hold n values. */
int qs_fp_normalize(const void* coeffs_dev, int is_f64, uint64_t B, uint32_t n,
                    const double* med_dev, const double* mad_dev, double* out_dev, void* stream);

/* Fingerprint geometry (FingerprintParams + StftParams, fingerprint.py:44-88).
 * band_low_hz <= 0 and band_high_hz <= 0: the full band. */
typedef struct qs_fp_params {
    double window_len_s;
    double window_lag_s;
    uint32_t freq_bins;
    uint32_t time_bins;
    uint32_t top_k;
    double band_low_hz;
    double band_high_hz;
    double frame_len_s;
    double hop_s;
} qs_fp_params;

/* n_windows (fingerprint.py:189-195) after the same validation as
 * FingerprintParams.validate; QS_ERR_DATA for a series shorter than one window. */
int qs_fp_n_windows(uint64_t n_samples, double sample_rate_hz, const qs_fp_params* params,
                    uint64_t* n_windows_out);

/* fingerprint_series (fingerprint.py:581-623) in one call: band STFT, the MAD
 * pass over the windows mad_sample_dev[0 .. n_mad_sample) (sorted int64
 * window indices — the reference draws them with numpy's
 * default_rng(mad_seed).choice, fingerprint.py:356-362) writing med_dev /
 * mad_dev (n_coeffs float64 each), then the top_k sign bits of every window
 * into bits_dev (n_windows, top_k) uint32.  mad_sample_dev == NULL: med_dev /
 * mad_dev are inputs (fingerprint_series(stats=...)).  x_dev: float64 samples,
 * or float32 with x_is_f32 (widened exactly).  Errors as the reference:
 * ParameterError (QS_ERR_ARG) for geometry / top_k > eligible coefficients,
 * DataError (QS_ERR_DATA) for short series or non-finite coefficients.
 * Synchronises the stream twice (eligible count, non-finite flag). */
size_t qs_fingerprint_chain_ws_bytes(uint64_t n_samples, double sample_rate_hz,
                                     const qs_fp_params* params, uint64_t n_mad_sample);
int qs_fingerprint_chain(const void* x_dev, int x_is_f32, uint64_t n_samples,
                         double sample_rate_hz, const qs_fp_params* params,
                         const int64_t* mad_sample_dev, uint64_t n_mad_sample, double* med_dev,
                         double* mad_dev, uint32_t* bits_dev, uint64_t* n_windows_out, void* ws_dev,
                         size_t ws_bytes, void* stream);

/* .fp file records (fingerprint.py:529-551 layout: index u64 | epoch f64 |
 * bits u32[K], little endian, 16 + 4K bytes each) packed from / unpacked to
 * device columns, so fingerprint files stream through one D2H / H2D copy. */
int qs_fp_pack_records(const uint64_t* indices_dev, const double* epochs_dev,
                       const uint32_t* bits_dev, uint64_t n, uint32_t K, uint8_t* out_dev,
                       void* stream);
int qs_fp_unpack_records(const uint8_t* in_dev, uint64_t n, uint32_t K, uint64_t* indices_dev,
                         double* epochs_dev, uint32_t* bits_dev, void* stream);

/* Generic stable LSD radix sort of (uint64 key, uint32 value) pairs over
 * `segments` independent equal-length segments, on key bits [0, key_bits). */
size_t qs_radix_sort_ws_bytes(uint64_t seg_len, uint32_t segments);
int qs_radix_sort_pairs(uint64_t* keys_dev, uint32_t* vals_dev, uint64_t seg_len,
                        uint32_t segments, uint32_t key_bits, uint64_t* keys_alt_dev,
                        uint32_t* vals_alt_dev, void* ws_dev, size_t ws_bytes,
                        int* result_in_alt, void* stream);

/* CUDA-core throughput microbenchmarks for the rooflines:
 * kind 0 FP64 FMA, 1 FP32 FMA, 2 64-bit min/max compare-select; `blocks` x
 * 256 threads, 8 independent operations per thread and iteration;
 * *ops_out = operations launched (time the launch with events on `stream`).
 * scratch_dev: blocks x 256 x 8 bytes. */
int qs_peak_launch(int kind, uint32_t blocks, uint32_t iters, void* scratch_dev,
                   double* ops_out, void* stream);

/* The north-star design's pair-count table, as a measurement (DESIGN.md
 * §5.3): n inserts of `distinct` scattered 64-bit pair keys into an
 * open-addressed table of `slots` (power of two) 12-byte slots (keys u64 then
 * counts u32, zeroed by the caller); *probes_dev += probes made. */
int qs_bench_pair_table(uint64_t n, uint64_t distinct, void* table_dev, uint64_t slots,
                        uint64_t* probes_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QUAKESCAN_B200_H */
