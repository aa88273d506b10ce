// ref_capi.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the read-only reference sources /root/reference/proj/src/{core,threading,
// init,local_search,big_means}.cpp (reference flags: -std=c++20 -O3 -DNDEBUG
// -fopenmp, no -march) into oracle/_ref/libbigmeans_ref.so.  It lets the
// Python tests and bench.py call the reference's own public API
// (big_means.hpp:46,56; local_search.hpp:38,44; init.hpp:40; core.hpp:112-126)
// with plain buffers, to pin the C restatement (bm_oracle.c) and to time the
// reference CPU path.  Nothing here is reference source; it only calls it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bigmeans/big_means.hpp"
#include "bigmeans/core.hpp"
#include "bigmeans/init.hpp"
#include "bigmeans/local_search.hpp"
#include "bigmeans/threading.hpp"

using namespace bigmeans;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const StateError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Dataset make_dataset(const double* X, uint64_t m, uint64_t n) {
    return Dataset(std::vector<double>(X, X + m * n), m, n);
}

Centroids make_centroids(const double* C, const uint8_t* mask, uint64_t k, uint64_t n) {
    Centroids c = Centroids::all_degenerate(k, n);
    for (uint64_t j = 0; j < k; ++j) {
        if (!mask[j]) c.set_row(j, std::span<const double>(C + j * n, n));
    }
    return c;
}

void export_centroids(const Centroids& c, double* C, uint8_t* mask) {
    std::memcpy(C, c.values().data(), c.values().size() * sizeof(double));
    std::memcpy(mask, c.mask().data(), c.mask().size());
}

}  // namespace

extern "C" {

struct ref_config {
    uint64_t k;
    uint64_t chunk_size;
    int has_max_chunks;
    uint64_t max_chunks;
    int has_max_cpu_seconds;
    double max_cpu_seconds;
    uint64_t max_iterations;
    double rel_tolerance;
    int candidates_per_step;
    uint64_t seed;
    int final_assignment;
};

struct ref_record {
    uint64_t chunk_index;
    double candidate_objective;
    double incumbent_objective;
    uint64_t accepted;
    uint64_t degenerate_repaired;
};

struct ref_outcome {
    double objective;
    uint64_t evals;
    uint64_t iterations;
    uint64_t chunks;
    double cpu_init;
    double cpu_full;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_worker_count(unsigned count) { set_worker_count(count); }
unsigned ref_worker_count() { return worker_count(); }

void* ref_rng_create(uint64_t seed) { return new Rng(seed); }
void ref_rng_destroy(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<Rng*>(r))(); }
uint64_t ref_uniform_int(void* r, uint64_t a, uint64_t b) {
    std::uniform_int_distribution<std::size_t> d(a, b);
    return d(*static_cast<Rng*>(r));
}
double ref_uniform_real(void* r, double a, double b) {
    std::uniform_real_distribution<double> d(a, b);
    return d(*static_cast<Rng*>(r));
}

int ref_sample_chunk(uint64_t m, uint64_t s, void* rng, uint64_t* out) {
    return guarded([&] {
        Dataset d(std::vector<double>(m, 0.0), m, 1);
        std::vector<std::size_t> idx = sample_chunk(d, s, *static_cast<Rng*>(rng));
        for (std::size_t i = 0; i < idx.size(); ++i) out[i] = idx[i];
    });
}

int ref_assign_nearest(const double* X, uint64_t m, uint64_t n, const double* C,
                       const uint8_t* mask, uint64_t k, int32_t* labels, double* dists,
                       uint64_t* evals) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        Centroids c = make_centroids(C, mask, k, n);
        EvalCounter counter;
        auto [asg, ds] = assign_nearest(d, c, &counter);
        std::memcpy(labels, asg.labels.data(), m * sizeof(int32_t));
        if (dists) std::memcpy(dists, ds.data(), m * sizeof(double));
        if (evals) *evals += counter.distance_evals;
    });
}

double ref_block_sum(const double* v, uint64_t m) {
    return block_sum(std::vector<double>(v, v + m));
}

int ref_update_centroids(const double* X, uint64_t m, uint64_t n, const int32_t* labels,
                         uint64_t k, double* C, uint8_t* mask) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        Assignment a;
        a.labels.assign(labels, labels + m);
        export_centroids(update_centroids(d, a, k), C, mask);
    });
}

int ref_kmeanspp_fill(const double* P, uint64_t m, uint64_t n, double* C, uint8_t* mask,
                      uint64_t k, int candidates, void* rng, uint64_t* evals) {
    return guarded([&] {
        Dataset d = make_dataset(P, m, n);
        InitConfig cfg;
        cfg.candidates_per_step = candidates;
        EvalCounter counter;
        Centroids out = kmeanspp_fill(d, make_centroids(C, mask, k, n), cfg,
                                      *static_cast<Rng*>(rng), &counter);
        export_centroids(out, C, mask);
        if (evals) *evals += counter.distance_evals;
    });
}

int ref_lloyd(const double* X, uint64_t m, uint64_t n, double* C, uint8_t* mask, uint64_t k,
              uint64_t max_iterations, double rel_tolerance, int32_t* labels, double* history,
              uint64_t history_cap, double* objective, uint64_t* evals, uint64_t* iterations,
              uint64_t* history_len) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        SearchConfig cfg;
        cfg.max_iterations = max_iterations;
        cfg.rel_tolerance = rel_tolerance;
        ClusteringOutcome out = lloyd(d, make_centroids(C, mask, k, n), cfg);
        export_centroids(out.centroids, C, mask);
        std::memcpy(labels, out.assignment.labels.data(), m * sizeof(int32_t));
        for (std::size_t i = 0; i < out.objective_history.size() && i < history_cap; ++i)
            history[i] = out.objective_history[i];
        *history_len = out.objective_history.size();
        *objective = out.objective;
        *evals = out.counter.distance_evals;
        *iterations = out.counter.iterations;
    });
}

int ref_big_means(const double* X, uint64_t m, uint64_t n, const ref_config* cfg, double* C,
                  uint8_t* mask, int32_t* labels, ref_record* trace, uint64_t trace_cap,
                  ref_outcome* out) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        BigMeansConfig c;
        c.k = cfg->k;
        c.chunk_size = cfg->chunk_size;
        if (cfg->has_max_chunks) c.max_chunks = cfg->max_chunks;
        if (cfg->has_max_cpu_seconds) c.max_cpu_seconds = cfg->max_cpu_seconds;
        c.search.max_iterations = cfg->max_iterations;
        c.search.rel_tolerance = cfg->rel_tolerance;
        c.init.candidates_per_step = cfg->candidates_per_step;
        c.seed = cfg->seed;
        c.final_assignment = cfg->final_assignment != 0;
        auto [o, t] = big_means(d, c);
        export_centroids(o.centroids, C, mask);
        if (labels && !o.assignment.labels.empty())
            std::memcpy(labels, o.assignment.labels.data(), m * sizeof(int32_t));
        for (std::size_t i = 0; i < t.records.size() && i < trace_cap; ++i) {
            trace[i].chunk_index = t.records[i].chunk_index;
            trace[i].candidate_objective = t.records[i].candidate_objective;
            trace[i].incumbent_objective = t.records[i].incumbent_objective;
            trace[i].accepted = t.records[i].accepted ? 1 : 0;
            trace[i].degenerate_repaired = t.records[i].degenerate_repaired;
        }
        out->objective = o.objective;
        out->evals = o.counter.distance_evals;
        out->iterations = o.counter.iterations;
        out->chunks = t.chunks();
        out->cpu_init = o.counter.cpu_init;
        out->cpu_full = o.counter.cpu_full;
    });
}

int ref_kmeans_pp(const double* X, uint64_t m, uint64_t n, uint64_t k, int candidates,
                  uint64_t seed, uint64_t max_iterations, double rel_tolerance, double* C,
                  uint8_t* mask, int32_t* labels, ref_outcome* out) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        InitConfig init;
        init.seed = seed;
        init.candidates_per_step = candidates;
        SearchConfig search;
        search.max_iterations = max_iterations;
        search.rel_tolerance = rel_tolerance;
        ClusteringOutcome o = kmeans(d, k, init, search);
        export_centroids(o.centroids, C, mask);
        std::memcpy(labels, o.assignment.labels.data(), m * sizeof(int32_t));
        out->objective = o.objective;
        out->evals = o.counter.distance_evals;
        out->iterations = o.counter.iterations;
        out->chunks = 1;
        out->cpu_init = o.counter.cpu_init;
        out->cpu_full = o.counter.cpu_full;
    });
}

struct ref_init {  // InitConfig init.hpp:16-27 (method / rounds_rule as their enum values)
    int method;
    int candidates_per_step;
    int oversampling_l;
    int rounds_r;
    int rounds_rule;
    uint64_t seed;
};

static InitConfig to_init(const ref_init* c) {
    InitConfig init;
    init.method = static_cast<InitMethod>(c->method);
    init.candidates_per_step = c->candidates_per_step;
    init.oversampling_l = c->oversampling_l;
    init.rounds_r = c->rounds_r;
    init.rounds_rule = static_cast<RoundsRule>(c->rounds_rule);
    init.seed = c->seed;
    return init;
}

// forgy_init init.hpp:31 (explicit stream)
int ref_forgy_init(const double* X, uint64_t m, uint64_t n, uint64_t k, Rng* rng, double* C) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        Centroids c = forgy_init(d, k, *rng);
        std::memcpy(C, c.values().data(), k * n * sizeof(double));
    });
}

// kmeans_parallel_init init.hpp:50 (explicit stream)
int ref_kmeans_parallel_init(const double* X, uint64_t m, uint64_t n, uint64_t k, const ref_init* cfg, Rng* rng,
                             double* C, uint64_t* evals) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        EvalCounter counter;
        Centroids c = kmeans_parallel_init(d, k, to_init(cfg), *rng, &counter);
        std::memcpy(C, c.values().data(), k * n * sizeof(double));
        *evals = counter.distance_evals;
    });
}

// kmeans local_search.hpp:44 (any init method)
int ref_kmeans(const double* X, uint64_t m, uint64_t n, uint64_t k, const ref_init* init, uint64_t max_iterations,
               double rel_tolerance, double* C, uint8_t* mask, int32_t* labels, ref_outcome* out) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        SearchConfig search;
        search.max_iterations = max_iterations;
        search.rel_tolerance = rel_tolerance;
        ClusteringOutcome o = kmeans(d, k, to_init(init), search);
        export_centroids(o.centroids, C, mask);
        std::memcpy(labels, o.assignment.labels.data(), m * sizeof(int32_t));
        out->objective = o.objective;
        out->evals = o.counter.distance_evals;
        out->iterations = o.counter.iterations;
        out->chunks = 1;
        out->cpu_init = o.counter.cpu_init;
        out->cpu_full = o.counter.cpu_full;
    });
}

// choose_chunk_size_hint big_means.hpp:72-73
int ref_choose_chunk_size_hint(const double* X, uint64_t m, uint64_t n, uint64_t k, const uint64_t* ladder,
                               uint64_t ladder_len, uint64_t chunks_per, uint64_t runs_per, uint64_t max_iterations,
                               double rel_tolerance, int candidates, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        Dataset d = make_dataset(X, m, n);
        ChunkHintConfig cfg;
        cfg.ladder.assign(ladder, ladder + ladder_len);
        cfg.chunks_per_candidate = chunks_per;
        cfg.runs_per_candidate = runs_per;
        cfg.search.max_iterations = max_iterations;
        cfg.search.rel_tolerance = rel_tolerance;
        cfg.init.candidates_per_step = candidates;
        cfg.seed = seed;
        *out = choose_chunk_size_hint(d, k, cfg);
    });
}

}  // extern "C"
