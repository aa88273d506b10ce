// big_means_b200.cpp — drop-in replacement for the reference's
// src/big_means.cpp (/root/reference/proj/src/big_means.cpp) that runs the
// hot path on a B200 through the C-ABI (include/bigmeans_b200.h).
//
// Compiled against the REFERENCE's own headers (include/bigmeans/*.hpp), it
// defines the three functions big_means.hpp declares with their exact types:
//   sample_chunk            big_means.hpp:46  -> host draws + bm_sample_chunk_draws
//   big_means               big_means.hpp:56  -> bm_big_means
//   choose_chunk_size_hint  big_means.hpp:72  -> unchanged logic over big_means
// Errors are rethrown as the reference's ConfigError / StateError /
// std::runtime_error (common.hpp:21-49), so callers (CLI exit codes,
// bench failure accounting, acceptance gate) behave as before.
#include <algorithm>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "bigmeans/big_means.hpp"
#include "dropin_common.hpp"

namespace bigmeans {
using namespace dropin;

std::vector<std::size_t> sample_chunk(const Dataset& data, std::size_t s, Rng& rng) {
    const std::size_t m = data.m();
    if (s < 1 || s > m) throw ConfigError("sample_chunk: chunk size must be in [1, m]");
    std::vector<std::size_t> idx(s);
    if (s == m) {  // the unique m-subset; no draws (big_means.cpp:46-48)
        std::iota(idx.begin(), idx.end(), 0);
        return idx;
    }
    // The caller's stream, consumed exactly as the reference does (:49-52).
    std::vector<uint32_t> draws(s);
    for (std::size_t i = 0; i < s; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, m - 1);
        draws[i] = static_cast<uint32_t>(pick(rng));
    }
    std::vector<uint64_t> out(s);
    rethrow(bm_sample_chunk_draws(m, s, draws.data(), device_of_thread(), out.data()));
    for (std::size_t i = 0; i < s; ++i) idx[i] = static_cast<std::size_t>(out[i]);
    return idx;
}

std::pair<ClusteringOutcome, BigMeansTrace> big_means(const Dataset& data, const BigMeansConfig& cfg) {
    bm_config c;
    bm_config_init(&c);
    c.k = cfg.k;
    c.chunk_size = cfg.chunk_size;
    c.has_max_cpu_seconds = cfg.max_cpu_seconds.has_value();
    c.max_cpu_seconds = cfg.max_cpu_seconds.value_or(0.0);
    c.has_max_chunks = cfg.max_chunks.has_value();
    c.max_chunks = cfg.max_chunks.value_or(0);
    c.max_iterations = cfg.search.max_iterations;
    c.rel_tolerance = cfg.search.rel_tolerance;
    c.candidates_per_step = cfg.init.candidates_per_step;
    c.seed = cfg.seed;
    c.final_assignment = cfg.final_assignment ? 1 : 0;
    if (data.m() < 1) throw ConfigError("big_means: empty dataset");

    const std::shared_ptr<Handle> dd = device_dataset(data);
    const std::size_t k = cfg.k, n = data.n();
    std::vector<double> centers(std::max<std::size_t>(k, 1) * n);
    std::vector<std::uint8_t> mask(std::max<std::size_t>(k, 1));
    std::vector<std::int32_t> labels(cfg.final_assignment ? data.m() : 0);
    bm_outcome o{};
    o.centroids = centers.data();
    o.mask = mask.data();
    o.labels = cfg.final_assignment ? labels.data() : nullptr;
    rethrow(bm_big_means(dd->h, &c, &o, nullptr, 0));
    // the whole trace, sized from the chunk count (time budgets: unknown up front)
    uint64_t nrec = 0;
    rethrow(bm_last_trace(nullptr, 0, &nrec));
    std::vector<bm_chunk_record> recs(nrec);
    rethrow(bm_last_trace(recs.data(), nrec, &nrec));

    Centroids inc = Centroids::all_degenerate(k, n);
    for (std::size_t j = 0; j < k; ++j)
        if (!mask[j]) inc.set_row(j, std::span<const double>(centers.data() + j * n, n));
    ClusteringOutcome out;
    out.centroids = std::move(inc);
    out.assignment.labels = std::move(labels);
    out.objective = o.objective;
    out.counter.distance_evals = o.distance_evals;
    out.counter.iterations = o.iterations;
    out.counter.cpu_init = o.cpu_init;
    out.counter.cpu_full = o.cpu_full;
    BigMeansTrace trace;
    for (uint64_t i = 0; i < recs.size(); ++i)
        trace.records.push_back({recs[i].chunk_index, recs[i].candidate_objective,
                                 recs[i].incumbent_objective, recs[i].accepted != 0,
                                 static_cast<std::size_t>(recs[i].degenerate_repaired)});
    return {std::move(out), std::move(trace)};
}

// Advisory chunk-size probe (big_means.hpp:63-73): every candidate size on the
// geometric ladder m/64 .. m (or the caller's ladder, clamped to [k, m]) gets
// runs_per_candidate short runs; the smallest size with the lowest mean final
// objective wins.  The probes themselves are B200 big_means runs.
std::size_t choose_chunk_size_hint(const Dataset& data, std::size_t k, const ChunkHintConfig& cfg) {
    const std::size_t m = data.m();
    if (k < 1 || m < k) throw ConfigError("choose_chunk_size_hint: need at least k points");
    if (cfg.chunks_per_candidate < 1 || cfg.runs_per_candidate < 1)
        throw ConfigError("choose_chunk_size_hint: probe budget must be positive");
    std::vector<std::size_t> sizes = cfg.ladder;
    if (sizes.empty()) {
        for (std::size_t shift = 6;; --shift) {
            sizes.push_back(std::max(k, m >> shift));
            if (shift == 0) break;
        }
    }
    for (auto& v : sizes) v = std::min(std::max(v, k), m);
    std::sort(sizes.begin(), sizes.end());
    sizes.erase(std::unique(sizes.begin(), sizes.end()), sizes.end());
    auto mean_objective = [&](std::size_t s) {
        double acc = 0.0;
        for (std::uint64_t r = 0; r < cfg.runs_per_candidate; ++r) {
            BigMeansConfig p;
            p.k = k;
            p.chunk_size = s;
            p.max_chunks = cfg.chunks_per_candidate;
            p.search = cfg.search;
            p.init = cfg.init;
            p.seed = cfg.seed + r;
            acc += big_means(data, p).first.objective;
        }
        return acc / static_cast<double>(cfg.runs_per_candidate);
    };
    std::size_t chosen = sizes.front();
    double chosen_mean = std::numeric_limits<double>::infinity();
    for (std::size_t s : sizes) {
        const double v = mean_objective(s);
        if (v < chosen_mean) {  // strict: ties keep the smaller size
            chosen_mean = v;
            chosen = s;
        }
    }
    return chosen;
}

}  // namespace bigmeans
