/*
 * datagen/gen.c -- seeded, counter-based synthetic inputs (YET, ELT records, event pool).
 *
 * This module is shared by the oracle side and the CUDA side as their ONLY common code.
 * It holds none of the method's arithmetic: no lookups, no financial/occurrence/aggregate
 * terms, no sums over trials.  It only draws random numbers.
 *
 * Generator: SplitMix64 finaliser (constants 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9,
 * 0x94D049BB133111EB), used counter-style:
 *     key(seed, stream) = mix64(seed * GOLDEN + stream)
 *     rng(seed, stream, i) = mix64(key(seed, stream) + (i + 1) * GOLDEN)
 * so every entity (pool slot, ELT record, trial) draws from its own substream and any slice
 * of trials is generated identically alone or as part of the whole YET.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

#define S_POOL (1ULL << 56)
#define S_ELT_MEMBER (2ULL << 56)
#define S_ELT_LOSS (3ULL << 56)
#define S_LEN (6ULL << 56)
#define S_YET (7ULL << 56)

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t key64(uint64_t seed, uint64_t stream) { return mix64(seed * GOLDEN + stream); }

uint64_t gen_rng(uint64_t seed, uint64_t stream, uint64_t index)
{
    return mix64(key64(seed, stream) + (index + 1) * GOLDEN);
}

/* uniform in [0, 1) from the top 53 bits */
double gen_uniform(uint64_t seed, uint64_t stream, uint64_t index)
{
    return (double)(gen_rng(seed, stream, index) >> 11) * (1.0 / 9007199254740992.0);
}

/* F distinct event ids uniform in [1, C] (draw order; duplicates skipped). */
int gen_pool(uint64_t seed, uint32_t catalogue_size, uint32_t pool_size, uint32_t *pool)
{
    if (pool_size > catalogue_size) return -1;
    uint8_t *seen = (uint8_t *)calloc((size_t)catalogue_size + 1, 1);
    if (!seen) return -2;
    uint64_t i = 0;
    for (uint32_t f = 0; f < pool_size; ++i) {
        uint32_t e = (uint32_t)(gen_rng(seed, S_POOL, i) % catalogue_size) + 1;
        if (seen[e]) continue;
        seen[e] = 1;
        pool[f++] = e;
    }
    free(seen);
    return 0;
}

/*
 * ELT j takes R distinct members of the pool (partial Fisher-Yates over pool slots) with
 * truncated-Pareto(alpha = 1) losses on [a, b]:  l = a / (1 - u (1 - a/b)).
 * Writes ids[j*R + r], losses[j*R + r] for j < n_elts, r < R.
 */
int gen_elt_records(uint64_t seed, const uint32_t *pool, uint32_t pool_size, uint32_t n_elts,
                    uint32_t records_per_elt, double loss_min, double loss_max, uint32_t *ids,
                    double *losses)
{
    if (records_per_elt > pool_size) return -1;
    uint32_t *slot = (uint32_t *)malloc((size_t)pool_size * sizeof(uint32_t));
    if (!slot) return -2;
    double shape = 1.0 - loss_min / loss_max;
    for (uint32_t j = 0; j < n_elts; ++j) {
        for (uint32_t f = 0; f < pool_size; ++f) slot[f] = f;
        for (uint32_t r = 0; r < records_per_elt; ++r) {
            uint32_t pick = r + (uint32_t)(gen_rng(seed, S_ELT_MEMBER | j, r) % (pool_size - r));
            uint32_t tmp = slot[r]; slot[r] = slot[pick]; slot[pick] = tmp;
            ids[(size_t)j * records_per_elt + r] = pool[slot[r]];
            double u = (double)(gen_rng(seed, S_ELT_LOSS | j, r) >> 11) *
                       (1.0 / 9007199254740992.0);
            losses[(size_t)j * records_per_elt + r] = loss_min / (1.0 - u * shape);
        }
    }
    free(slot);
    return 0;
}

static inline uint64_t trial_len(uint64_t seed, uint64_t t, uint32_t kmin, uint32_t kmax)
{
    if (kmax <= kmin) return kmin;
    return kmin + gen_rng(seed, S_LEN, t) % ((uint64_t)kmax - kmin + 1);
}

/* offsets[0..n] of trials [t0, t0+n), rebased to offsets[0] = 0. */
void gen_trial_offsets(uint64_t seed, uint64_t t0, uint64_t n, uint32_t kmin, uint32_t kmax,
                       uint64_t *offsets)
{
    offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + trial_len(seed, t0 + i, kmin, kmax);
}

typedef struct {
    uint64_t seed, t0, i0, i1;
    double hit;
    uint32_t catalogue_size, pool_size;
    const uint32_t *pool;
    const uint64_t *offsets;
    uint32_t *events;
} yet_job;

/* Occurrence d of trial t: x = rng(seed, S_YET|t, d); the top 24 bits decide a pool hit
 * (probability hit), the low 40 bits pick the id: pool[x40 % F] or 1 + x40 % C. */
static void *yet_run(void *arg)
{
    yet_job *j = (yet_job *)arg;
    uint64_t thresh = (uint64_t)(j->hit * 16777216.0);
    for (uint64_t i = j->i0; i < j->i1; ++i) {
        uint64_t key = key64(j->seed, S_YET | (j->t0 + i));
        uint32_t *out = j->events + j->offsets[i];
        uint64_t k = j->offsets[i + 1] - j->offsets[i];
        for (uint64_t d = 0; d < k; ++d) {
            uint64_t x = mix64(key + (d + 1) * GOLDEN);
            uint64_t low = x & 0xFFFFFFFFFFULL;
            if ((x >> 40) < thresh)
                out[d] = j->pool[low % j->pool_size];
            else
                out[d] = (uint32_t)(low % j->catalogue_size) + 1;
        }
    }
    return NULL;
}

/* Event ids of trials [t0, t0+n) into events[offsets[i] ..] (offsets rebased to 0). */
int gen_yet_events(uint64_t seed, uint64_t t0, uint64_t n, const uint64_t *offsets, double hit,
                   uint32_t catalogue_size, const uint32_t *pool, uint32_t pool_size,
                   uint32_t *events, int n_threads)
{
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > n) n_threads = n ? (int)n : 1;
    yet_job *jobs = (yet_job *)calloc((size_t)n_threads, sizeof(yet_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -2; }
    for (int i = 0; i < n_threads; ++i) {
        yet_job *j = &jobs[i];
        j->seed = seed; j->t0 = t0; j->hit = hit;
        j->catalogue_size = catalogue_size; j->pool_size = pool_size; j->pool = pool;
        j->offsets = offsets; j->events = events;
        j->i0 = n * (uint64_t)i / (uint64_t)n_threads;
        j->i1 = n * (uint64_t)(i + 1) / (uint64_t)n_threads;
    }
    for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, yet_run, &jobs[i]);
    yet_run(&jobs[0]);
    for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(jobs); free(th);
    return 0;
}
