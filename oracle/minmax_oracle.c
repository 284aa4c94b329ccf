/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * Plain-C restatement of the reference's Min-Max signature arithmetic, used by
 * tests/ and bench.py's cpu_baseline leg as the CPU checker.  It follows:
 *   fmix64         reference pkg/src/quakescan/_sigcore.pyx:18-24 (murmur3 finalizer)
 *   combine step   reference pkg/src/quakescan/_sigcore.pyx:27-29 (boost-style fold)
 *   mapping        reference pkg/src/quakescan/minmax_hash.py:86-89
 *                  values[x, j] = fmix64(((x + 1) * GOLDEN64) ^ (seed + j))
 *   signatures     reference pkg/src/quakescan/_sigcore.pyx:32-85
 *                  per row: running min/max over the F = t*k/2 mapping columns of
 *                  every set bit, then per table fold k/2 minima then k/2 maxima.
 * All arithmetic is modular uint64, exactly as the reference.
 *
 * The implementation here is deliberately "function-major per row" (loop over
 * columns outside, set bits inside), the traversal used by the reference's
 * own slow oracle (bench.py:51-73), so it shares no loop structure with the
 * element-major Cython kernel nor with the CUDA probe kernel it checks.
 */
#include <stdint.h>
#include <stddef.h>
#include <pthread.h>
#include <stdlib.h>

#define GOLDEN64 0x9E3779B97F4A7C15ULL

uint64_t qso_fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDULL;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ULL;
    x ^= x >> 33;
    return x;
}

uint64_t qso_hash(uint64_t x, uint64_t salt) {
    return qso_fmix64(((x + 1ULL) * GOLDEN64) ^ salt);
}

uint64_t qso_combine(const uint64_t *words, size_t n) {
    uint64_t acc = 0;
    for (size_t i = 0; i < n; ++i)
        acc ^= qso_fmix64(words[i]) + GOLDEN64 + (acc << 6) + (acc >> 2);
    return acc;
}

void qso_gen_mapping(uint64_t *values, size_t d, size_t n_funcs, uint64_t seed) {
    for (size_t x = 0; x < d; ++x)
        for (size_t j = 0; j < n_funcs; ++j)
            values[x * n_funcs + j] = qso_hash((uint64_t)x, seed + (uint64_t)j);
}

/* rows [start, stop) of bits (n, K) -> out (n, t); values is (d, t*k_half). */
int qso_signatures_range(const uint32_t *bits, size_t K, const uint64_t *values,
                         size_t F, int t, int k_half, uint64_t *out,
                         size_t start, size_t stop) {
    if ((size_t)t * (size_t)k_half != F || K < 1 || k_half < 1) return 1;
    uint64_t *words = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)k_half);
    if (!words) return 2;
    for (size_t row = start; row < stop; ++row) {
        const uint32_t *b = bits + row * K;
        for (int i = 0; i < t; ++i) {
            for (int j = 0; j < k_half; ++j) {
                size_t col = (size_t)i * k_half + j;
                uint64_t lo = UINT64_MAX, hi = 0;
                for (size_t kk = 0; kk < K; ++kk) {
                    uint64_t v = values[(size_t)b[kk] * F + col];
                    if (v < lo) lo = v;
                    if (v > hi) hi = v;
                }
                words[j] = lo;
                words[k_half + j] = hi;
            }
            out[row * (size_t)t + i] = qso_combine(words, 2 * (size_t)k_half);
        }
    }
    free(words);
    return 0;
}

typedef struct {
    const uint32_t *bits; size_t K; const uint64_t *values; size_t F;
    int t; int k_half; uint64_t *out; size_t start, stop; int rc;
} qso_job;

static void *qso_worker(void *p) {
    qso_job *j = (qso_job *)p;
    j->rc = qso_signatures_range(j->bits, j->K, j->values, j->F, j->t, j->k_half,
                                 j->out, j->start, j->stop);
    return NULL;
}

/* Row ranges split over `threads` pthreads (the reference's ThreadPoolExecutor
 * split, minmax_hash.py:113-128). */
int qso_signatures(const uint32_t *bits, size_t n, size_t K, const uint64_t *values,
                   size_t F, int t, int k_half, uint64_t *out, int threads) {
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = n ? (int)n : 1;
    qso_job *jobs = (qso_job *)calloc((size_t)threads, sizeof(qso_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !tid) { free(jobs); free(tid); return 2; }
    for (int w = 0; w < threads; ++w) {
        jobs[w] = (qso_job){bits, K, values, F, t, k_half, out,
                            n * (size_t)w / threads, n * (size_t)(w + 1) / threads, 0};
        pthread_create(&tid[w], NULL, qso_worker, &jobs[w]);
    }
    int rc = 0;
    for (int w = 0; w < threads; ++w) {
        pthread_join(tid[w], NULL);
        if (jobs[w].rc) rc = jobs[w].rc;
    }
    free(jobs);
    free(tid);
    return rc;
}
