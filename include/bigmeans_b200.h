/*
 * bigmeans_b200.h — C-ABI of the B200-native Big-means hot path.
 *
 * Drop-in boundary for the reference's C++ library (libbigmeans.a,
 * /root/reference/proj/src/CMakeLists.txt:1-13).  Every entry point below
 * replaces one reference function; the citation names it (paths relative to
 * /root/reference/proj).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * Semantics: results are bit-identical to the reference built with its own
 * Release flags (g++ -O3, no -march): same RNG stream (std::mt19937_64 +
 * libstdc++ 13 distributions), same per-1024-point reduction order, same
 * first-minimum tie rule, same n_d accounting.
 *
 * Errors: every function returns a bm_status.  BM_CONFIG_ERROR maps to the
 * reference's ConfigError (CLI exit 2), BM_STATE_ERROR to StateError, anything
 * else to std::runtime_error (CLI exit 1; bigmeans_cli.cpp:379-385).  The
 * message of the last failure on the calling thread is bm_last_error().
 *
 * Threading: one host thread per (dataset handle, device) at a time; distinct
 * handles may be driven concurrently from distinct threads.
 */
#ifndef BIGMEANS_B200_H
#define BIGMEANS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 1

typedef enum bm_status {
    BM_OK = 0,
    BM_CONFIG_ERROR = 1,   /* ConfigError  common.hpp:21-24 */
    BM_STATE_ERROR = 2,    /* StateError   common.hpp:46-49 */
    BM_CUDA_ERROR = 3,     /* device failure (runtime_error) */
    BM_INTERNAL_ERROR = 4, /* anything else (runtime_error) */
    BM_PARSE_ERROR = 5     /* ParseError   common.hpp:28-42 (bm_last_parse_location) */
} bm_status;

/* io::Format io.hpp:14. */
typedef enum bm_format {
    BM_FORMAT_CSV = 0,
    BM_FORMAT_WHITESPACE = 1,
    BM_FORMAT_TSPLIB = 2
} bm_format;

typedef enum bm_dtype {
    BM_F64 = 0, /* reference storage type (core.hpp:34) */
    BM_F32 = 1  /* fp32 storage, promoted exactly to fp64 before any arithmetic */
} bm_dtype;

/* Opaque device-resident, immutable dataset (Dataset core.hpp:13-37). */
typedef struct bm_dataset bm_dataset;
/* Opaque RNG (Rng = std::mt19937_64, common.hpp:13). */
typedef struct bm_rng bm_rng;

/* Reference configuration surface (BigMeansConfig big_means.hpp:11-26,
 * SearchConfig local_search.hpp:10-16, InitConfig::candidates_per_step
 * init.hpp:18).  Defaults: bm_config_init(). */
typedef struct bm_config {
    uint64_t k;
    uint64_t chunk_size;          /* s */
    int32_t has_max_cpu_seconds;  /* std::optional<double> max_cpu_seconds */
    double max_cpu_seconds;
    int32_t has_max_chunks;       /* std::optional<uint64_t> max_chunks */
    uint64_t max_chunks;
    uint64_t max_iterations;      /* search.max_iterations (300) */
    double rel_tolerance;         /* search.rel_tolerance (1e-4) */
    int32_t candidates_per_step;  /* init.candidates_per_step (3) */
    uint64_t seed;                /* cfg.seed (kDefaultSeed 123456789) */
    int32_t final_assignment;     /* cfg.final_assignment (true) */
} bm_config;

/* ClusteringOutcome (local_search.hpp:24-30) + EvalCounter (core.hpp:89-101).
 * Caller-owned output buffers: centroids k*n f64 (row-major), mask k bytes
 * (1 = degenerate), labels m int32 (may be NULL: assignment not copied back). */
typedef struct bm_outcome {
    double* centroids;
    uint8_t* mask;
    int32_t* labels;
    double objective;
    uint64_t distance_evals;
    uint64_t iterations;
    double cpu_init; /* chunk-loop wall seconds (big_means.cpp:96) */
    double cpu_full; /* final-pass wall seconds (big_means.cpp:103-107) */
    uint64_t chunks; /* trace.chunks() */
} bm_outcome;

/* ChunkRecord big_means.hpp:28-34. */
typedef struct bm_chunk_record {
    uint64_t chunk_index;
    double candidate_objective;
    double incumbent_objective;
    uint64_t accepted;
    uint64_t degenerate_repaired;
} bm_chunk_record;

const char* bm_last_error(void);
int bm_abi_version(void);
void bm_config_init(bm_config* cfg);
/* Number of CUDA devices; BM_CUDA_ERROR when none. */
bm_status bm_device_count(int* count);

/* Dataset(values, m, n) core.hpp:19 + core.cpp:19-32 (shape and finiteness
 * checks -> BM_CONFIG_ERROR).  Uploads to `device`. */
bm_status bm_dataset_create(const void* values, uint64_t m, uint64_t n, bm_dtype dtype,
                            int device, bm_dataset** out);
bm_status bm_dataset_destroy(bm_dataset* data);
bm_status bm_dataset_shape(const bm_dataset* data, uint64_t* m, uint64_t* n);
/* Device storage type: fp64 input whose every value is exactly representable
 * in fp32 is stored as fp32 (lossless; results unchanged). */
bm_status bm_dataset_storage(const bm_dataset* data, bm_dtype* storage);
/* io::min_max_normalize io.hpp:38 / io.cpp:245-264 on the device: per column
 * (x - min) / (max - min), constant columns 0.0; a new dataset. */
bm_status bm_dataset_min_max_normalize(const bm_dataset* data, bm_dataset** out);
/* Exact-sum property (no reference counterpart; it changes no result): every
 * value is an integer multiple of 2^exponent and m * max|x| < 2^52 * 2^exponent,
 * so the ordered fp64 sums of update_centroids (core.cpp:206-229) are exact and
 * the device keeps per-label integer sums instead of re-summing each round. */
bm_status bm_dataset_sum_mode(const bm_dataset* data, int32_t* exact, int32_t* exponent);
/* Dataset::gather core.hpp:30 / core.cpp:34-44: new dataset with the listed
 * rows in the listed order (index >= m -> BM_CONFIG_ERROR). */
bm_status bm_dataset_gather(const bm_dataset* data, const uint64_t* rows, uint64_t count,
                            bm_dataset** out);
/* Copy the (promoted-to-f64) rows back to the host, m*n f64. */
bm_status bm_dataset_download(const bm_dataset* data, double* out);

/* RNG (Rng rng(seed), common.hpp:13). */
bm_status bm_rng_create(uint64_t seed, bm_rng** out);
bm_status bm_rng_destroy(bm_rng* rng);
uint64_t bm_rng_next(bm_rng* rng);
/* uniform_int_distribution<size_t>(a,b)(rng) / uniform_real_distribution<double>(a,b)(rng)
 * with libstdc++ 13 semantics (host only). */
uint64_t bm_rng_uniform_int(bm_rng* rng, uint64_t a, uint64_t b);
double bm_rng_uniform_real(bm_rng* rng, double a, double b);

/* sample_chunk big_means.hpp:46 / big_means.cpp:39-56.  out: s indices,
 * ascending.  Draws from rng on the host; resolution and sort on the device. */
bm_status bm_sample_chunk(const bm_dataset* data, uint64_t s, bm_rng* rng, uint64_t* out);

/* sample_chunk with the draws made ON THE DEVICE from rng's state (the path
 * big_means uses); rng advances exactly as the host draws would advance it.
 * force_sequential=1 exercises the exact sequential Lemire-rejection path. */
bm_status bm_sample_chunk_device(const bm_dataset* data, uint64_t s, bm_rng* rng, int force_sequential,
                                 uint64_t* out);

/* sample_chunk with caller-side draws: draws[i] = uniform_int(i, m-1) taken
 * from the caller's own Rng (big_means.cpp:49-51); the Fisher-Yates
 * resolution and the ascending sort run on `device`.  s < m required. */
bm_status bm_sample_chunk_draws(uint64_t m, uint64_t s, const uint32_t* draws, int device,
                                uint64_t* out);

/* assign_nearest core.hpp:112-114 / core.cpp:106-161.  centroids k*n f64,
 * mask k (1 = degenerate).  labels (m) and dists (m, may be NULL) out;
 * *evals += m * active when evals != NULL.  All-degenerate -> BM_STATE_ERROR. */
bm_status bm_assign_nearest(const bm_dataset* data, const double* centroids, const uint8_t* mask,
                            uint64_t k, int32_t* labels, double* dists, uint64_t* evals);
/* objective core.hpp:118 / core.cpp:177-181. */
bm_status bm_objective(const bm_dataset* data, const double* centroids, const uint8_t* mask,
                       uint64_t k, double* objective, uint64_t* evals);
/* block_sum core.hpp:122 / core.cpp:163-175 (host values, device reduction). */
bm_status bm_block_sum(const double* values, uint64_t count, int device, double* out);
/* update_centroids core.hpp:126 / core.cpp:183-244: centroids k*n and mask k out. */
bm_status bm_update_centroids(const bm_dataset* data, const int32_t* labels, uint64_t k,
                              double* centroids, uint8_t* mask);
/* kmeanspp_fill init.hpp:40-41 / init.cpp:123-201 (centroids/mask in-out). */
bm_status bm_kmeanspp_fill(const bm_dataset* pool, double* centroids, uint8_t* mask, uint64_t k,
                           int32_t candidates_per_step, bm_rng* rng, uint64_t* evals);
/* lloyd local_search.hpp:38-39 / local_search.cpp:16-60.  centroids/mask in
 * (start) and out (final); labels m out; history (capacity entries) out with
 * its full length in *history_len; objective/evals/iterations out. */
bm_status bm_lloyd(const bm_dataset* data, double* centroids, uint8_t* mask, uint64_t k,
                   uint64_t max_iterations, double rel_tolerance, int32_t* labels,
                   double* history, uint64_t history_capacity, uint64_t* history_len,
                   double* objective, uint64_t* evals, uint64_t* iterations);
/* kmeans local_search.hpp:44 / local_search.cpp:62-94, kmeans_pp init only
 * (the s == m identity partner of big_means, test_big_means.cpp:177-195). */
bm_status bm_kmeans_pp(const bm_dataset* data, uint64_t k, int32_t candidates_per_step,
                       uint64_t seed, uint64_t max_iterations, double rel_tolerance,
                       bm_outcome* out);

/* InitConfig init.hpp:16-27: method 0 forgy, 1 kmeans_pp, 2 kmeans_parallel
 * (InitMethod); rounds_rule 0 fixed, 1 log_phi (RoundsRule). */
typedef struct {
    int32_t method;
    int32_t candidates_per_step; /* 3 */
    int32_t oversampling_l;      /* 0: 2k */
    int32_t rounds_r;            /* 5 */
    int32_t rounds_rule;
    uint64_t seed;
} bm_init_config;

/* kmeans local_search.hpp:44 / local_search.cpp:62-94 with any InitMethod:
 * forgy_init (init.cpp:92-115), kmeanspp_fill (:123-201) or
 * kmeans_parallel_init (:209-347), then lloyd.  out->labels may be NULL. */
bm_status bm_kmeans(const bm_dataset* data, uint64_t k, const bm_init_config* init,
                    uint64_t max_iterations, double rel_tolerance, bm_outcome* out);
/* The initialization stage of kmeans alone (local_search.cpp:66-83):
 * forgy_init init.cpp:92-115, kmeanspp_fill from an all-degenerate start
 * :123-201, kmeans_parallel_init :209-347, seeded by init->seed.  Writes the
 * start centroids (k*n f64) and mask (k bytes); *evals = the init's distance
 * evaluations.  kmeans == bm_init_centroids + bm_lloyd (the drop-in's
 * local_search shim composes them exactly as local_search.cpp:62-94 does). */
bm_status bm_init_centroids(const bm_dataset* data, uint64_t k, const bm_init_config* init,
                            double* centroids, uint8_t* mask, uint64_t* evals);

/* choose_chunk_size_hint big_means.hpp:72-73 / big_means.cpp:114-160 (ChunkHintConfig
 * :60-68): ladder NULL / empty = m/64 .. m; best mean objective of
 * runs_per_candidate big_means probes (seeds seed + run) wins, ties to the
 * smaller size.  best_mean may be NULL. */
bm_status bm_choose_chunk_size_hint(bm_dataset* data, uint64_t k, const uint64_t* ladder,
                                    uint64_t ladder_len, uint64_t chunks_per_candidate,
                                    uint64_t runs_per_candidate, uint64_t max_iterations,
                                    double rel_tolerance, int32_t candidates_per_step,
                                    uint64_t seed, uint64_t* chunk_size, double* best_mean);

/* big_means big_means.hpp:56-57 / big_means.cpp:58-112.  trace may be NULL;
 * at most trace_capacity records are written, out->chunks holds the count. */
bm_status bm_big_means(bm_dataset* data, const bm_config* cfg, bm_outcome* out,
                       bm_chunk_record* trace, uint64_t trace_capacity);

/* Multi-GPU Big-means in one process (paper parallel mode 2, PAPER.md:216;
 * the reference runs one chain: big_means.hpp:56).  data[g] is chain g's
 * handle of the SAME matrix (normally one handle per GPU).  Chain g runs
 * big_means with seed + g and floor(N/G) (+1 for g < N mod G) of the
 * cfg->max_chunks = N chunks (a time budget applies to every chain), without
 * its own final pass; one host thread per device drives that device's chains.
 * The lowest-index chain with the minimum f_opt wins (*winner); its incumbent
 * is the result; with cfg->final_assignment the final pass is row-sharded over
 * the distinct devices on 1024-row tiles, the tile partials folded in row
 * order (== block_sum over all rows, core.cpp:165-175).  n_d / iterations /
 * chunks sum over the chains (+ the final pass); cpu_init is the slowest
 * chain's loop.  trace: the chains' records in chain order (chain_chunks[g]
 * of them each; both may be NULL). */
bm_status bm_big_means_multi(bm_dataset* const* data, int32_t chains, const bm_config* cfg,
                             bm_outcome* out, bm_chunk_record* trace, uint64_t trace_capacity,
                             uint64_t* chain_chunks, int32_t* winner);

/* Every chunk record of the last bm_big_means call on this thread (the trace
 * is never truncated here: *count is the full chunk count, at most `capacity`
 * records are copied).  Lets a caller with a time budget size its trace from
 * the result (BigMeansTrace big_means.hpp:36-40). */
bm_status bm_last_trace(bm_chunk_record* out, uint64_t capacity, uint64_t* count);

/* Dataset ingestion: io::load io.hpp:31-37 / io.cpp:224-243 (DatasetSpec
 * io.hpp:18-25: path, format, has_header, columns, normalize).  Parses the file
 * on the host (delimited formats in parallel over line ranges; threads <= 0:
 * all cores), with the reference's cell rules, ragged-row check, errors and
 * 1-based line / column (BM_PARSE_ERROR; bm_last_parse_location), the Dataset
 * finiteness check (BM_CONFIG_ERROR) and the column selection (columns NULL:
 * all; an empty selection is BM_CONFIG_ERROR), then uploads it and, with
 * normalize, min-max normalises it on the device (io.cpp:245-264). */
bm_status bm_dataset_load(const char* path, int32_t format, int32_t has_header, int32_t normalize,
                          const uint64_t* columns, uint64_t ncolumns, int32_t threads, int device,
                          bm_dataset** out);
/* The host part of bm_dataset_load alone (no device): *values (malloc'd,
 * release with bm_free_values) holds m x n row-major f64. */
bm_status bm_parse_file(const char* path, int32_t format, int32_t has_header, const uint64_t* columns,
                        uint64_t ncolumns, int32_t threads, double** values, uint64_t* m, uint64_t* n);
void bm_free_values(double* values);
/* 1-based line and column of the last BM_PARSE_ERROR on this thread. */
bm_status bm_last_parse_location(uint64_t* line, uint64_t* column);

/* Multi-GPU pieces.  Row-sharded final pass: assign rows
 * [row_begin, row_end) (row_begin a multiple of 1024) against the centroids,
 * write their labels (row_end-row_begin, may be NULL) and the per-1024-row
 * tile partial sums (ceil((row_end-row_begin)/1024) f64); the caller
 * concatenates all shards' partials in row order and folds them left to right
 * (block_sum's outer loop, core.cpp:172), which reproduces block_sum exactly. */
bm_status bm_assign_rows(const bm_dataset* data, const double* centroids, const uint8_t* mask,
                         uint64_t k, uint64_t row_begin, uint64_t row_end, int32_t* labels,
                         double* tile_partials, uint64_t* evals);

/* Device timing of the last bm_big_means call on this thread (for roofline
 * reporting): average assignment-kernel duration in ms measured with CUDA
 * events, number of assignment launches, and rows*n of one average launch. */
typedef struct bm_profile {
    double assign_ms_total;
    uint64_t assign_launches;
    uint64_t assign_rows_total;
    uint64_t kernel_launches;
    double final_ms;
    uint64_t final_rows;
    uint64_t screen_candidates; /* exact rechecks issued by the screened assignment */
    uint64_t screen_rows;       /* rows that went through the screened assignment */
    /* per launch group: 0 assign (chunk loop), 1 final pass, 2 update, 3 sample,
     * 4 gather, 5 k-means++ distances, 6 Lloyd control */
    double phase_ms[8];
    uint64_t phase_count[8];
    /* persistent chunk kernel (one launch per chunk; device globaltimer stamps
     * taken inside the timed run itself): summed launch durations, launches,
     * assignment passes (first assignment + one per Lloyd round) and update
     * passes over the chunk, rows per chunk, gaps between launches */
    double chunk_ms_total;
    uint64_t chunk_launches;
    uint64_t chunk_assign_passes;
    uint64_t chunk_update_passes;
    uint64_t chunk_rows;
    /* summed idle time between consecutive chunk kernels (one's end stamp to
     * the next one's start stamp) */
    double chunk_gap_ms_total;
} bm_profile;
bm_status bm_set_profiling(int enabled);
/* Debug builds (-DBM_KTRACE): per-CTA phase timestamps of the screened assignment. */
bm_status bm_debug_ktrace(uint64_t* out, uint64_t count);
/* Debug (BM_CHUNK_DBG=1): phase stamps of the persistent chunk kernel,
 * [chunk % 4][round 0..6, 7 = tail][16] globaltimer ns. */
bm_status bm_debug_chunk_phases(uint64_t* out);
/* Debug builds (-DBM_WIDE_DBG, BM_WIDE_DBG=1): k_wide_screen CTA (0,0)'s per-atom
 * globaltimer stamps [4][64]: TMA issued, data landed, MMAs issued, stage retired. */
bm_status bm_debug_wide_stamps(uint64_t* out);
bm_status bm_last_profile(bm_profile* out);

#ifdef __cplusplus
}
#endif
#endif /* BIGMEANS_B200_H */
