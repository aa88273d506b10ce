/*
 * bm_oracle.c — CPU restatement of the Big-means hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see bm_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so that every `a - b`, `a * b`, `a + b` rounds
 * separately, exactly as the reference's default x86-64 build (no -march,
 * hence no FMA contraction) does.  File:line citations are relative to
 * /root/reference/proj.
 */
#include "bm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_BLOCK 1024u /* kReductionBlock threading.hpp:15 */

/* ---------------------------------------------------------------------------
 * std::mt19937_64 (common.hpp:13); parameters of the C++ standard
 * [rand.predef] (w=64 n=312 m=156 r=31 ...), seeding per [rand.eng.mers].
 * ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (uint64_t i = 1; i < MT_N; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
    }
    r->mti = MT_N;
}

static void mt_twist(orc_rng* r) {
    for (uint64_t i = 0; i < MT_N; ++i) {
        const uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= MT_A;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->mti >= MT_N) mt_twist(r);
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* uniform_int_distribution<size_t>(a,b): libstdc++ 13 downscaling through
 * Lemire's nearly divisionless method with a 128-bit product
 * (uniform_int_dist.h:252-331), then + a. */
uint64_t orc_uniform_int(orc_rng* r, uint64_t a, uint64_t b) {
    const uint64_t urange = b - a;
    if (urange == UINT64_MAX) return orc_rng_next(r) + a;
    const uint64_t erange = urange + 1;
    unsigned __int128 product = (unsigned __int128)orc_rng_next(r) * erange;
    uint64_t low = (uint64_t)product;
    if (low < erange) {
        const uint64_t threshold = (0 - erange) % erange;
        while (low < threshold) {
            product = (unsigned __int128)orc_rng_next(r) * erange;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64) + a;
}

/* uniform_real_distribution<double>(a,b): generate_canonical<double,53> with
 * one 64-bit engine call (random.tcc:3349-3381), then canon*(b-a)+a
 * (random.h:1904-1910). */
double orc_uniform_real(orc_rng* r, double a, double b) {
    const double sum = (double)orc_rng_next(r);
    double canon = sum / 18446744073709551616.0; /* 2^64 */
    if (canon >= 1.0) canon = nextafter(1.0, 0.0);
    return canon * (b - a) + a;
}

/* ---------------------------------------------------------------------------
 * sample_chunk big_means.cpp:39-56
 * ------------------------------------------------------------------------- */
static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

int orc_sample_chunk(uint64_t m, uint64_t s, orc_rng* r, uint64_t* out) {
    if (s < 1 || s > m) return ORC_CONFIG_ERROR; /* :41-43 */
    if (s == m) {                                 /* :46-48, no draws */
        for (uint64_t i = 0; i < m; ++i) out[i] = i;
        return ORC_OK;
    }
    uint64_t* idx = (uint64_t*)malloc(m * sizeof(uint64_t)); /* iota :44-45 */
    for (uint64_t i = 0; i < m; ++i) idx[i] = i;
    for (uint64_t i = 0; i < s; ++i) { /* partial Fisher-Yates :49-52 */
        const uint64_t j = orc_uniform_int(r, i, m - 1);
        const uint64_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    memcpy(out, idx, s * sizeof(uint64_t));
    free(idx);
    qsort(out, s, sizeof(uint64_t), cmp_u64); /* :53-54 */
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * core.cpp
 * ------------------------------------------------------------------------- */
static uint64_t active_count(const uint8_t* mask, uint64_t k) {
    uint64_t a = 0;
    for (uint64_t j = 0; j < k; ++j) a += mask[j] ? 0 : 1;
    return a;
}

/* assign_nearest core.cpp:106-161; distance loop core.cpp:142-146. */
int orc_assign_nearest(const double* X, uint64_t m, uint64_t n, const double* C,
                       const uint8_t* mask, uint64_t k, int32_t* labels, double* dists,
                       uint64_t* evals) {
    const uint64_t active = active_count(mask, k);
    if (active == 0) return ORC_STATE_ERROR; /* :115-118 */
    for (uint64_t i = 0; i < m; ++i) {
        const double* x = X + i * n;
        double best = INFINITY;
        int32_t best_j = -1;
        for (uint64_t j = 0; j < k; ++j) {
            if (mask[j]) continue;
            const double* c = C + j * n;
            double sum = 0.0;
            for (uint64_t d = 0; d < n; ++d) {
                const double diff = x[d] - c[d];
                sum += diff * diff;
            }
            if (sum < best) { /* strict: lowest index wins ties, :147 */
                best = sum;
                best_j = (int32_t)j;
            }
        }
        labels[i] = best_j;
        if (dists) dists[i] = best;
    }
    if (evals) *evals += m * active; /* :157-159 */
    return ORC_OK;
}

/* block_sum core.cpp:163-175. */
double orc_block_sum(const double* v, uint64_t m) {
    double total = 0.0;
    for (uint64_t begin = 0; begin < m; begin += ORC_BLOCK) {
        const uint64_t end = begin + ORC_BLOCK < m ? begin + ORC_BLOCK : m;
        double partial = 0.0;
        for (uint64_t i = begin; i < end; ++i) partial += v[i];
        total += partial;
    }
    return total;
}

/* update_centroids core.cpp:183-244. */
int orc_update_centroids(const double* X, uint64_t m, uint64_t n, const int32_t* labels,
                         uint64_t k, double* C, uint8_t* mask) {
    for (uint64_t i = 0; i < m; ++i) {
        if (labels[i] < 0 || (uint64_t)labels[i] >= k) return ORC_CONFIG_ERROR; /* :189-193 */
    }
    const uint64_t blocks = (m + ORC_BLOCK - 1) / ORC_BLOCK;
    double* sums = (double*)calloc(k * n, sizeof(double));
    uint64_t* counts = (uint64_t*)calloc(k, sizeof(uint64_t));
    double* psum = (double*)malloc(k * n * sizeof(double));
    uint64_t* pcnt = (uint64_t*)malloc(k * sizeof(uint64_t));
    for (uint64_t b = 0; b < blocks; ++b) {
        /* per-block partials, points in index order (:200-215) */
        memset(psum, 0, k * n * sizeof(double));
        memset(pcnt, 0, k * sizeof(uint64_t));
        const uint64_t begin = b * ORC_BLOCK;
        const uint64_t end = begin + ORC_BLOCK < m ? begin + ORC_BLOCK : m;
        for (uint64_t i = begin; i < end; ++i) {
            const uint64_t j = (uint64_t)labels[i];
            const double* x = X + i * n;
            double* row = psum + j * n;
            for (uint64_t d = 0; d < n; ++d) row[d] += x[d];
            ++pcnt[j];
        }
        /* merged in block index order (:217-229) */
        for (uint64_t j = 0; j < k; ++j) {
            for (uint64_t d = 0; d < n; ++d) sums[j * n + d] += psum[j * n + d];
            counts[j] += pcnt[j];
        }
    }
    for (uint64_t j = 0; j < k; ++j) { /* all_degenerate start, :231-242 */
        if (counts[j] == 0) {
            for (uint64_t d = 0; d < n; ++d) C[j * n + d] = 0.0;
            mask[j] = 1;
            continue;
        }
        const double inv = 1.0 / (double)counts[j];
        for (uint64_t d = 0; d < n; ++d) C[j * n + d] = sums[j * n + d] * inv;
        mask[j] = 0;
    }
    free(sums);
    free(counts);
    free(psum);
    free(pcnt);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * init.cpp
 * ------------------------------------------------------------------------- */
/* distances_to_row init.cpp:19-43 */
static void distances_to_row(const double* P, uint64_t m, uint64_t n, const double* c, double* out,
                             uint64_t* evals) {
    for (uint64_t i = 0; i < m; ++i) {
        const double* x = P + i * n;
        double sum = 0.0;
        for (uint64_t d = 0; d < n; ++d) {
            const double diff = x[d] - c[d];
            sum += diff * diff;
        }
        out[i] = sum;
    }
    if (evals) *evals += m;
}

/* lower_to_row init.cpp:46-70; std::min(a,b) keeps a unless b < a. */
static void lower_to_row(const double* P, uint64_t m, uint64_t n, const double* c, double* d2,
                         uint64_t* evals) {
    for (uint64_t i = 0; i < m; ++i) {
        const double* x = P + i * n;
        double sum = 0.0;
        for (uint64_t d = 0; d < n; ++d) {
            const double diff = x[d] - c[d];
            sum += diff * diff;
        }
        if (sum < d2[i]) d2[i] = sum;
    }
    if (evals) *evals += m;
}

/* pick_by_mass init.cpp:73-79: upper_bound, clamped to the last index. */
static uint64_t pick_by_mass(const double* cum, uint64_t m, double u) {
    uint64_t lo = 0, hi = m; /* first index with cum[idx] > u */
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (u < cum[mid]) hi = mid;
        else lo = mid + 1;
    }
    return lo == m ? m - 1 : lo;
}

/* prefix_sums init.cpp:81-88 (sequential) */
static void prefix_sums(const double* v, uint64_t m, double* cum) {
    double running = 0.0;
    for (uint64_t i = 0; i < m; ++i) {
        running += v[i];
        cum[i] = running;
    }
}

/* kmeanspp_fill init.cpp:123-201 */
int orc_kmeanspp_fill(const double* P, uint64_t m, uint64_t n, double* C, uint8_t* mask,
                      uint64_t k, int candidates, orc_rng* r, uint64_t* evals) {
    if (candidates < 1) return ORC_CONFIG_ERROR; /* :129-131 */
    uint64_t* degenerate = (uint64_t*)malloc(k * sizeof(uint64_t));
    uint64_t n_deg = 0;
    for (uint64_t j = 0; j < k; ++j)
        if (mask[j]) degenerate[n_deg++] = j; /* :133-138 */
    if (n_deg == 0) {
        free(degenerate);
        return ORC_OK;
    }
    double* dist2 = (double*)malloc(m * sizeof(double));
    for (uint64_t i = 0; i < m; ++i) dist2[i] = INFINITY;
    uint64_t first_slot_index = 0;
    if (active_count(mask, k) == 0) { /* :144-150 */
        const uint64_t first = orc_uniform_int(r, 0, m - 1);
        const uint64_t slot = degenerate[0];
        memcpy(C + slot * n, P + first * n, n * sizeof(double));
        mask[slot] = 0;
        first_slot_index = 1;
        distances_to_row(P, m, n, C + slot * n, dist2, evals);
    } else { /* :151-164 */
        int first_row = 1;
        for (uint64_t j = 0; j < k; ++j) {
            if (mask[j]) continue;
            if (first_row) {
                distances_to_row(P, m, n, C + j * n, dist2, evals);
                first_row = 0;
            } else {
                lower_to_row(P, m, n, C + j * n, dist2, evals);
            }
        }
    }
    double* cum = (double*)malloc(m * sizeof(double));
    double* trial = (double*)malloc(m * sizeof(double));
    double* best_trial = (double*)malloc(m * sizeof(double));
    for (uint64_t q = first_slot_index; q < n_deg; ++q) { /* :171-199 */
        const uint64_t slot = degenerate[q];
        prefix_sums(dist2, m, cum);
        const double total = cum[m - 1];
        if (total <= 0.0) { /* uniform fallback :174-180 */
            const uint64_t pick = orc_uniform_int(r, 0, m - 1);
            memcpy(C + slot * n, P + pick * n, n * sizeof(double));
            mask[slot] = 0;
            continue;
        }
        double best_potential = INFINITY;
        uint64_t best_index = 0;
        for (int c = 0; c < candidates; ++c) { /* :183-196 */
            const double u = orc_uniform_real(r, 0.0, total);
            const uint64_t index = pick_by_mass(cum, m, u);
            distances_to_row(P, m, n, P + index * n, trial, evals);
            for (uint64_t i = 0; i < m; ++i)
                if (dist2[i] < trial[i]) trial[i] = dist2[i]; /* std::min(trial, dist2) */
            const double potential = orc_block_sum(trial, m);
            if (potential < best_potential) {
                best_potential = potential;
                best_index = index;
                double* t = trial;
                trial = best_trial;
                best_trial = t;
            }
        }
        memcpy(C + slot * n, P + best_index * n, n * sizeof(double)); /* :197 */
        mask[slot] = 0;
        double* t = dist2; /* :198 */
        dist2 = best_trial;
        best_trial = t;
    }
    free(degenerate);
    free(dist2);
    free(cum);
    free(trial);
    free(best_trial);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * lloyd local_search.cpp:16-60
 * ------------------------------------------------------------------------- */
int orc_lloyd(const double* X, uint64_t m, uint64_t n, double* C, uint8_t* mask, uint64_t k,
              uint64_t max_iterations, double rel_tolerance, int32_t* labels, double* history,
              uint64_t history_cap, orc_lloyd_out* out) {
    if (max_iterations < 1) return ORC_CONFIG_ERROR; /* :18-20 */
    if (rel_tolerance < 0.0) return ORC_CONFIG_ERROR; /* :21-23 */
    memset(out, 0, sizeof(*out));
    double* dists = (double*)malloc(m * sizeof(double));
    int32_t* new_labels = (int32_t*)malloc(m * sizeof(int32_t));
    double* next = (double*)malloc(k * n * sizeof(double));
    uint8_t* next_mask = (uint8_t*)malloc(k);
    int rc = orc_assign_nearest(X, m, n, C, mask, k, labels, dists, &out->evals); /* :26 */
    if (rc != ORC_OK) goto done;
    double f = orc_block_sum(dists, m); /* :27 */
    if (out->history_len < history_cap) history[out->history_len] = f;
    out->history_len++;
    double last = f;
    while (out->iterations < max_iterations) { /* :32 */
        orc_update_centroids(X, m, n, labels, k, next, next_mask);                    /* :33 */
        rc = orc_assign_nearest(X, m, n, next, next_mask, k, new_labels, dists, &out->evals); /* :34 */
        if (rc != ORC_OK) goto done;
        const double f_new = orc_block_sum(dists, m); /* :35 */
        ++out->iterations;                            /* :36 */
        if (out->history_len < history_cap) history[out->history_len] = f_new;
        out->history_len++;
        last = f_new;
        const int unchanged = memcmp(new_labels, labels, m * sizeof(int32_t)) == 0; /* :39 */
        memcpy(C, next, k * n * sizeof(double));                                   /* :40 */
        memcpy(mask, next_mask, k);
        memcpy(labels, new_labels, m * sizeof(int32_t)); /* :41 */
        if (unchanged) break;                            /* :42-44 */
        if (f <= 0.0) break;                             /* :45-47 */
        if (rel_tolerance > 0.0 && (f - f_new) / f < rel_tolerance) break; /* :48-50 */
        f = f_new;                                       /* :51 */
    }
    out->objective = last; /* history.back() :54 */
done:
    free(dists);
    free(new_labels);
    free(next);
    free(next_mask);
    return rc;
}

/* ---------------------------------------------------------------------------
 * big_means big_means.cpp:16-112
 * ------------------------------------------------------------------------- */
int orc_big_means(const double* X, uint64_t m, uint64_t n, const orc_config* cfg, double* C,
                  uint8_t* mask, int32_t* labels, orc_record* trace, orc_outcome* out) {
    /* validate :16-35 (chunk budget only in the restatement) */
    if (cfg->k < 1 || cfg->chunk_size < cfg->k || cfg->chunk_size > m || cfg->max_chunks < 1)
        return ORC_CONFIG_ERROR;
    const uint64_t k = cfg->k, s = cfg->chunk_size;
    memset(out, 0, sizeof(*out));
    orc_rng* rng = (orc_rng*)malloc(sizeof(orc_rng));
    orc_rng_seed(rng, cfg->seed); /* :62 */
    /* incumbent all-degenerate, f_opt = +inf (:63-64) */
    for (uint64_t i = 0; i < k * n; ++i) C[i] = 0.0;
    for (uint64_t j = 0; j < k; ++j) mask[j] = 1;
    double f_opt = INFINITY;
    uint64_t* idx = (uint64_t*)malloc(s * sizeof(uint64_t));
    double* portion = (double*)malloc(s * n * sizeof(double));
    double* start = (double*)malloc(k * n * sizeof(double));
    uint8_t* start_mask = (uint8_t*)malloc(k);
    int32_t* chunk_labels = (int32_t*)malloc(s * sizeof(int32_t));
    int rc = ORC_OK;
    for (uint64_t chunk = 0; chunk < cfg->max_chunks; ++chunk) { /* :70-95 */
        orc_sample_chunk(m, s, rng, idx);                 /* :79 */
        for (uint64_t i = 0; i < s; ++i)                  /* gather :80, core.cpp:34-44 */
            memcpy(portion + i * n, X + idx[i] * n, n * sizeof(double));
        memcpy(start, C, k * n * sizeof(double)); /* :82 */
        memcpy(start_mask, mask, k);
        const uint64_t repaired = k - active_count(start_mask, k); /* :83 */
        rc = orc_kmeanspp_fill(portion, s, n, start, start_mask, k, cfg->candidates_per_step, rng,
                               &out->evals); /* :84 */
        if (rc != ORC_OK) goto done;
        orc_lloyd_out lo;
        rc = orc_lloyd(portion, s, n, start, start_mask, k, cfg->max_iterations,
                       cfg->rel_tolerance, chunk_labels, NULL, 0, &lo); /* :86 */
        if (rc != ORC_OK) goto done;
        out->evals += lo.evals; /* lloyd accumulate local_search.cpp:55-58 */
        out->iterations += lo.iterations;
        const int accepted = lo.objective < f_opt; /* :89 strict */
        if (accepted) {
            f_opt = lo.objective;
            memcpy(C, start, k * n * sizeof(double));
            memcpy(mask, start_mask, k);
        }
        if (trace) {
            trace[chunk].chunk_index = chunk;
            trace[chunk].candidate_objective = lo.objective;
            trace[chunk].incumbent_objective = f_opt;
            trace[chunk].accepted = (uint64_t)accepted;
            trace[chunk].degenerate_repaired = repaired;
        }
        out->chunks++;
    }
    if (cfg->final_assignment) { /* :102-107 */
        double* dists = (double*)malloc(m * sizeof(double));
        int32_t* lab = labels ? labels : (int32_t*)malloc(m * sizeof(int32_t));
        rc = orc_assign_nearest(X, m, n, C, mask, k, lab, dists, &out->evals);
        out->objective = orc_block_sum(dists, m);
        if (!labels) free(lab);
        free(dists);
    } else {
        out->objective = f_opt; /* :108-110 */
    }
done:
    free(rng);
    free(idx);
    free(portion);
    free(start);
    free(start_mask);
    free(chunk_labels);
    return rc;
}

/* kmeans local_search.cpp:62-94 (kmeans_pp branch). */
int orc_kmeans_pp(const double* X, uint64_t m, uint64_t n, uint64_t k, int candidates,
                  uint64_t seed, uint64_t max_iterations, double rel_tolerance, double* C,
                  uint8_t* mask, int32_t* labels, orc_outcome* out) {
    if (k < 1 || m < k) return ORC_CONFIG_ERROR;
    memset(out, 0, sizeof(*out));
    orc_rng* rng = (orc_rng*)malloc(sizeof(orc_rng));
    orc_rng_seed(rng, seed);
    for (uint64_t i = 0; i < k * n; ++i) C[i] = 0.0;
    for (uint64_t j = 0; j < k; ++j) mask[j] = 1;
    uint64_t init_evals = 0;
    int rc = orc_kmeanspp_fill(X, m, n, C, mask, k, candidates, rng, &init_evals);
    free(rng);
    if (rc != ORC_OK) return rc;
    orc_lloyd_out lo;
    rc = orc_lloyd(X, m, n, C, mask, k, max_iterations, rel_tolerance, labels, NULL, 0, &lo);
    if (rc != ORC_OK) return rc;
    out->objective = lo.objective;
    out->iterations = lo.iterations;
    out->evals = lo.evals + init_evals;
    out->chunks = 1;
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * forgy_init init.cpp:92-115: partial Fisher-Yates over the row indices; the
 * first k slots (in slot order) are the centroids.  No distance evaluations.
 * ------------------------------------------------------------------------- */
int orc_forgy_init(const double* X, uint64_t m, uint64_t n, uint64_t k, orc_rng* r, double* C) {
    if (k < 1 || m < k) return ORC_CONFIG_ERROR; /* :95-100 */
    uint64_t* idx = (uint64_t*)malloc(m * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) idx[i] = i; /* :101-102 */
    for (uint64_t i = 0; i < k; ++i) {          /* :104-107 */
        const uint64_t j = orc_uniform_int(r, i, m - 1);
        const uint64_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    for (uint64_t i = 0; i < k; ++i) memcpy(C + i * n, X + idx[i] * n, n * sizeof(double)); /* :108-113 */
    free(idx);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * kmeans_parallel_init init.cpp:209-347.
 * ------------------------------------------------------------------------- */
int orc_kmeans_parallel_init(const double* X, uint64_t m, uint64_t n, uint64_t k, const orc_init* cfg,
                             orc_rng* r, double* C, uint64_t* evals) {
    if (k < 1 || m < k) return ORC_CONFIG_ERROR;       /* :213-218 */
    const uint64_t first = orc_uniform_int(r, 0, m - 1); /* :220-221 */
    if (k == 1) {                                        /* :222-225 */
        memcpy(C, X + first * n, n * sizeof(double));
        return ORC_OK;
    }
    const double l = cfg->oversampling_l > 0 ? (double)cfg->oversampling_l : 2.0 * (double)k; /* :227-228 */
    uint64_t cap = 1024, nc = 0;
    uint64_t* cand = (uint64_t*)malloc(cap * sizeof(uint64_t));
    cand[nc++] = first;
    double* dist2 = (double*)malloc(m * sizeof(double));
    distances_to_row(X, m, n, X + first * n, dist2, evals); /* :232 */
    int rounds = cfg->rounds_r;                             /* :234-238 */
    if (cfg->rounds_rule == 1) {
        const double phi1 = orc_block_sum(dist2, m);
        rounds = phi1 > 1.0 ? (int)floor(log(phi1)) : 1;
        if (rounds < 1) rounds = 1;
    }
    if (rounds < 1) { /* :239-241 */
        free(cand);
        free(dist2);
        return ORC_CONFIG_ERROR;
    }
    uint64_t* fresh = (uint64_t*)malloc(m * sizeof(uint64_t));
    for (int round = 0; round < rounds; ++round) { /* :244-263 */
        const double phi = orc_block_sum(dist2, m);
        if (phi <= 0.0) break;
        uint64_t nf = 0;
        for (uint64_t i = 0; i < m; ++i) { /* one draw per point, index order :251-258 */
            const double u = orc_uniform_real(r, 0.0, 1.0);
            double p = l * dist2[i] / phi;
            if (p > 1.0) p = 1.0; /* std::min(1.0, .) */
            if (u < p) fresh[nf++] = i;
        }
        for (uint64_t f = 0; f < nf; ++f) { /* :259-262 */
            if (nc == cap) {
                cap *= 2;
                cand = (uint64_t*)realloc(cand, cap * sizeof(uint64_t));
            }
            cand[nc++] = fresh[f];
            lower_to_row(X, m, n, X + fresh[f] * n, dist2, evals);
        }
    }
    free(fresh);
    if (nc < k) { /* top-up with distinct uniform rows :266-278 */
        uint8_t* used = (uint8_t*)calloc(m, 1);
        for (uint64_t i = 0; i < nc; ++i) used[cand[i]] = 1;
        if (cap < k) {
            cap = k;
            cand = (uint64_t*)realloc(cand, cap * sizeof(uint64_t));
        }
        while (nc < k) {
            const uint64_t i = orc_uniform_int(r, 0, m - 1);
            if (!used[i]) {
                used[i] = 1;
                cand[nc++] = i;
            }
        }
        free(used);
    }
    /* the candidate set (data.gather :280) and its weights: points nearest each :287-295 */
    double* cr = (double*)malloc(nc * n * sizeof(double));
    for (uint64_t q = 0; q < nc; ++q) memcpy(cr + q * n, X + cand[q] * n, n * sizeof(double));
    uint8_t* cmask = (uint8_t*)calloc(nc, 1);
    int32_t* lab = (int32_t*)malloc(m * sizeof(int32_t));
    double* dd = (double*)malloc(m * sizeof(double));
    int rc = orc_assign_nearest(X, m, n, cr, cmask, nc, lab, dd, evals);
    double* weight = (double*)calloc(nc, sizeof(double));
    if (rc == ORC_OK)
        for (uint64_t i = 0; i < m; ++i) weight[lab[i]] += 1.0;
    free(lab);
    free(dd);
    free(cmask);
    if (rc != ORC_OK) {
        free(cand);
        free(dist2);
        free(cr);
        free(weight);
        return rc;
    }
    /* weighted greedy k-means++ over the candidates :297-339 */
    double* wcum = (double*)malloc(nc * sizeof(double));
    prefix_sums(weight, nc, wcum);
    const uint64_t chosen_first = pick_by_mass(wcum, nc, orc_uniform_real(r, 0.0, wcum[nc - 1]));
    uint64_t* chosen = (uint64_t*)malloc(k * sizeof(uint64_t));
    uint64_t nch = 0;
    chosen[nch++] = chosen_first;
    double* cdist2 = (double*)malloc(nc * sizeof(double));
    distances_to_row(cr, nc, n, cr + chosen_first * n, cdist2, evals);
    const int candidates = cfg->candidates_per_step > 1 ? cfg->candidates_per_step : 1;
    double* mass = (double*)malloc(nc * sizeof(double));
    double* cum = (double*)malloc(nc * sizeof(double));
    double* trial = (double*)malloc(nc * sizeof(double));
    double* best_trial = (double*)malloc(nc * sizeof(double));
    while (nch < k) {
        for (uint64_t q = 0; q < nc; ++q) mass[q] = weight[q] * cdist2[q];
        prefix_sums(mass, nc, cum);
        const double total = cum[nc - 1];
        if (total <= 0.0) { /* :318-322 */
            chosen[nch++] = orc_uniform_int(r, 0, nc - 1);
            continue;
        }
        double best_potential = INFINITY;
        uint64_t best_index = 0;
        for (int c = 0; c < candidates; ++c) { /* :323-336 */
            const uint64_t index = pick_by_mass(cum, nc, orc_uniform_real(r, 0.0, total));
            distances_to_row(cr, nc, n, cr + index * n, trial, evals);
            double potential = 0.0;
            for (uint64_t q = 0; q < nc; ++q) {
                if (cdist2[q] < trial[q]) trial[q] = cdist2[q]; /* std::min(trial, cdist2) */
                potential += weight[q] * trial[q];
            }
            if (potential < best_potential) {
                best_potential = potential;
                best_index = index;
                double* t = trial;
                trial = best_trial;
                best_trial = t;
            }
        }
        chosen[nch++] = best_index;
        double* t = cdist2; /* std::swap(cdist2, best_trial) :338 */
        cdist2 = best_trial;
        best_trial = t;
    }
    for (uint64_t j = 0; j < k; ++j) memcpy(C + j * n, cr + chosen[j] * n, n * sizeof(double)); /* :341-346 */
    free(cand);
    free(dist2);
    free(cr);
    free(weight);
    free(wcum);
    free(chosen);
    free(cdist2);
    free(mass);
    free(cum);
    free(trial);
    free(best_trial);
    return ORC_OK;
}

/* kmeans local_search.cpp:62-94: init per method (seeded by init.seed), then lloyd. */
int orc_kmeans(const double* X, uint64_t m, uint64_t n, uint64_t k, const orc_init* init,
               uint64_t max_iterations, double rel_tolerance, double* C, uint8_t* mask, int32_t* labels,
               orc_outcome* out) {
    if (k < 1 || m < k) return ORC_CONFIG_ERROR; /* :64-69 */
    memset(out, 0, sizeof(*out));
    orc_rng* rng = (orc_rng*)malloc(sizeof(orc_rng));
    orc_rng_seed(rng, init->seed); /* :71 */
    for (uint64_t i = 0; i < k * n; ++i) C[i] = 0.0;
    for (uint64_t j = 0; j < k; ++j) mask[j] = 1;
    uint64_t init_evals = 0;
    int rc = ORC_CONFIG_ERROR;
    if (init->method == 0) {
        rc = orc_forgy_init(X, m, n, k, rng, C);
        if (rc == ORC_OK) memset(mask, 0, k);
    } else if (init->method == 1) {
        rc = orc_kmeanspp_fill(X, m, n, C, mask, k, init->candidates_per_step, rng, &init_evals);
    } else if (init->method == 2) {
        rc = orc_kmeans_parallel_init(X, m, n, k, init, rng, C, &init_evals);
        if (rc == ORC_OK) memset(mask, 0, k);
    }
    free(rng);
    if (rc != ORC_OK) return rc;
    orc_lloyd_out lo;
    rc = orc_lloyd(X, m, n, C, mask, k, max_iterations, rel_tolerance, labels, NULL, 0, &lo);
    if (rc != ORC_OK) return rc;
    out->objective = lo.objective;
    out->iterations = lo.iterations;
    out->evals = lo.evals + init_evals;
    out->chunks = 1;
    return ORC_OK;
}
