/*
 * bm_oracle.h — CPU restatement of the Big-means hot path (TEST INFRASTRUCTURE).
 *
 * This is the CHECKER, not the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * (paper_2204_07485_b200/, the CUDA C-ABI) never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj) in plain C11, in the same arithmetic order, so that
 * results are bit-identical to the reference's g++ -O3 (no -march, no FMA)
 * build.  The restatement is pinned against the compiled reference
 * (oracle/_ref/libbigmeans_ref.so, built by oracle/Makefile from the
 * read-only sources) and against the committed golden vectors in
 * tests/golden/ generated from that build (tests/golden/make_golden.py).
 *
 * RNG: the reference uses std::mt19937_64 + libstdc++-13
 * uniform_int_distribution (Lemire nearly-divisionless, 128-bit product,
 * /usr/include/c++/13/bits/uniform_int_dist.h:252-331) and
 * uniform_real_distribution (generate_canonical<double,53>, one engine call,
 * /usr/include/c++/13/bits/random.tcc:3349-3381).  Those are third-party
 * (GCC 13.3 libstdc++); their published algorithms are restated here.
 */
#ifndef BM_ORACLE_H
#define BM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_CONFIG_ERROR 1
#define ORC_STATE_ERROR 2

/* std::mt19937_64 (common.hpp:13). */
typedef struct orc_rng {
    uint64_t mt[312];
    uint64_t mti;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
/* uniform_int_distribution<size_t>(a, b)(rng), inclusive bounds. */
uint64_t orc_uniform_int(orc_rng* r, uint64_t a, uint64_t b);
/* uniform_real_distribution<double>(a, b)(rng). */
double orc_uniform_real(orc_rng* r, double a, double b);

/* sample_chunk big_means.cpp:39-56: s distinct sorted indices of [0,m). */
int orc_sample_chunk(uint64_t m, uint64_t s, orc_rng* r, uint64_t* out);

/* assign_nearest core.cpp:106-161 (labels int32, dists f64). */
int orc_assign_nearest(const double* X, uint64_t m, uint64_t n, const double* C,
                       const uint8_t* mask, uint64_t k, int32_t* labels, double* dists,
                       uint64_t* evals);
/* block_sum core.cpp:163-175. */
double orc_block_sum(const double* v, uint64_t m);
/* update_centroids core.cpp:183-244; C (k*n) and mask (k) are outputs. */
int orc_update_centroids(const double* X, uint64_t m, uint64_t n, const int32_t* labels,
                         uint64_t k, double* C, uint8_t* mask);
/* kmeanspp_fill init.cpp:123-201; C/mask are in/out. */
int orc_kmeanspp_fill(const double* P, uint64_t m, uint64_t n, double* C, uint8_t* mask,
                      uint64_t k, int candidates, orc_rng* r, uint64_t* evals);

typedef struct orc_lloyd_out {
    double objective;
    uint64_t evals;
    uint64_t iterations;
    uint64_t history_len;
} orc_lloyd_out;

/* lloyd local_search.cpp:16-60.  C/mask in/out (start -> final centroids),
 * labels (m) out, history (cap entries) out. */
int orc_lloyd(const double* X, uint64_t m, uint64_t n, double* C, uint8_t* mask, uint64_t k,
              uint64_t max_iterations, double rel_tolerance, int32_t* labels, double* history,
              uint64_t history_cap, orc_lloyd_out* out);

typedef struct orc_config {
    uint64_t k;
    uint64_t chunk_size;
    uint64_t max_chunks; /* required (>=1) in the restatement; time budgets are host-only */
    uint64_t max_iterations;
    double rel_tolerance;
    int candidates_per_step;
    uint64_t seed;
    int final_assignment;
} orc_config;

typedef struct orc_record {
    uint64_t chunk_index;
    double candidate_objective;
    double incumbent_objective;
    uint64_t accepted;
    uint64_t degenerate_repaired;
} orc_record;

typedef struct orc_outcome {
    double objective;
    uint64_t evals;
    uint64_t iterations;
    uint64_t chunks;
} orc_outcome;

/* big_means big_means.cpp:58-112.  C (k*n), mask (k) out; labels (m) out when
 * final_assignment (may be NULL); trace (max_chunks records) out (may be NULL). */
int orc_big_means(const double* X, uint64_t m, uint64_t n, const orc_config* cfg, double* C,
                  uint8_t* mask, int32_t* labels, orc_record* trace, orc_outcome* out);

/* kmeans local_search.cpp:62-94 with kmeans_pp init (init.seed), used for the
 * s == m identity (test_big_means.cpp:177-195). */
int orc_kmeans_pp(const double* X, uint64_t m, uint64_t n, uint64_t k, int candidates,
                  uint64_t seed, uint64_t max_iterations, double rel_tolerance, double* C,
                  uint8_t* mask, int32_t* labels, orc_outcome* out);

/* InitConfig (init.hpp:16-27): method 0 forgy, 1 kmeans_pp, 2 kmeans_parallel;
 * rounds_rule 0 fixed, 1 log_phi. */
typedef struct {
    int method;
    int candidates_per_step;
    int oversampling_l;
    int rounds_r;
    int rounds_rule;
    uint64_t seed;
} orc_init;

/* forgy_init init.cpp:92-115: k distinct rows by partial Fisher-Yates. */
int orc_forgy_init(const double* X, uint64_t m, uint64_t n, uint64_t k, orc_rng* r, double* C);

/* kmeans_parallel_init init.cpp:209-347 (all k rows active on return). */
int orc_kmeans_parallel_init(const double* X, uint64_t m, uint64_t n, uint64_t k, const orc_init* cfg,
                             orc_rng* r, double* C, uint64_t* evals);

/* kmeans local_search.cpp:62-94, any init method. */
int orc_kmeans(const double* X, uint64_t m, uint64_t n, uint64_t k, const orc_init* init,
               uint64_t max_iterations, double rel_tolerance, double* C, uint8_t* mask, int32_t* labels,
               orc_outcome* out);

#ifdef __cplusplus
}
#endif
#endif
