// local_search_b200.cpp — drop-in replacement for the reference's
// src/local_search.cpp (/root/reference/proj/src/local_search.cpp): the two
// functions local_search.hpp declares, with their exact types, on a B200.
//   lloyd   local_search.hpp:38-39 / local_search.cpp:16-60  -> bm_lloyd
//   kmeans  local_search.hpp:44-45 / local_search.cpp:62-94  -> bm_init_centroids + bm_lloyd
// With this file and big_means_b200.cpp in place of the reference's two
// translation units, every bench cell (bench.cpp:25-86: big_means and the
// forgy / kmeans_pp / kmeans_parallel baselines) runs on the device.  Errors
// map back to ConfigError / StateError as in dropin_common.hpp.
#include <chrono>
#include <utility>
#include <vector>

#include "bigmeans/local_search.hpp"
#include "dropin_common.hpp"

namespace bigmeans {
using namespace dropin;

namespace {

double seconds_since(std::chrono::steady_clock::time_point start) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
}

// Centroids -> (k*n values, mask) buffers and back (core.hpp:42-74: degenerate
// rows hold 0.0, operator== compares them).
Centroids to_centroids(const std::vector<double>& values, const std::vector<std::uint8_t>& mask, std::size_t k,
                       std::size_t n) {
    Centroids c = Centroids::all_degenerate(k, n);
    for (std::size_t j = 0; j < k; ++j)
        if (!mask[j]) c.set_row(j, std::span<const double>(values.data() + j * n, n));
    return c;
}

}  // namespace

ClusteringOutcome lloyd(const Dataset& data, Centroids start, const SearchConfig& cfg, EvalCounter* accumulate) {
    if (cfg.max_iterations < 1) throw ConfigError("lloyd: max_iterations must be at least 1");  // :18-23
    if (cfg.rel_tolerance < 0.0) throw ConfigError("lloyd: rel_tolerance must be nonnegative");
    if (start.n() != data.n()) throw ConfigError("squared_distance: length mismatch");
    const std::shared_ptr<Handle> dd = device_dataset(data);
    const std::size_t k = start.k(), n = start.n();
    std::vector<double> values(start.values());
    std::vector<std::uint8_t> mask(start.mask());
    ClusteringOutcome out;
    out.assignment.labels.resize(data.m());
    out.objective_history.resize(cfg.max_iterations + 1);
    std::uint64_t hlen = 0, evals = 0, iterations = 0;
    double objective = 0.0;
    rethrow(bm_lloyd(dd->h, values.data(), mask.data(), k, cfg.max_iterations, cfg.rel_tolerance,
                     out.assignment.labels.data(), out.objective_history.data(), out.objective_history.size(),
                     &hlen, &objective, &evals, &iterations));
    out.objective_history.resize(hlen);
    out.centroids = to_centroids(values, mask, k, n);
    out.objective = objective;  // history.back() (:54)
    out.counter.distance_evals = evals;
    out.counter.iterations = iterations;
    if (accumulate != nullptr) {  // :55-58
        accumulate->distance_evals += evals;
        accumulate->iterations += iterations;
    }
    return out;
}

ClusteringOutcome kmeans(const Dataset& data, std::size_t k, const InitConfig& init, const SearchConfig& search) {
    if (k < 1) throw ConfigError("kmeans: k must be at least 1");  // :64-69
    if (data.m() < k) throw ConfigError("kmeans: dataset has fewer points than clusters");
    const std::shared_ptr<Handle> dd = device_dataset(data);
    bm_init_config ic{};
    ic.method = init.method == InitMethod::forgy ? 0 : init.method == InitMethod::kmeans_pp ? 1 : 2;
    ic.candidates_per_step = init.candidates_per_step;
    ic.oversampling_l = init.oversampling_l;
    ic.rounds_r = init.rounds_r;
    ic.rounds_rule = init.rounds_rule == RoundsRule::fixed ? 0 : 1;
    ic.seed = init.seed;  // Rng rng(init.seed) (:71)
    const std::size_t n = data.n();
    std::vector<double> values(k * n);
    std::vector<std::uint8_t> mask(k);
    std::uint64_t init_evals = 0;
    const auto t_init = std::chrono::steady_clock::now();
    rethrow(bm_init_centroids(dd->h, k, &ic, values.data(), mask.data(), &init_evals));  // :74-83
    const double cpu_init = seconds_since(t_init);
    const auto t_search = std::chrono::steady_clock::now();
    ClusteringOutcome out = lloyd(data, to_centroids(values, mask, k, n), search);  // :86
    out.counter.cpu_init = cpu_init;
    out.counter.cpu_full = seconds_since(t_search);
    out.counter.distance_evals += init_evals;  // :90
    return out;
}

}  // namespace bigmeans
