// plan_main.cpp — minimal driver of the reference's experiment harness
// (bench::load_plan / run_plan / result_to_json, bench.hpp:80-88,
// bench.cpp:252-424): `plan <plan.json>` prints the result document.
// tools/dropin/Makefile links it twice from the same unmodified reference
// sources: plan_ref with src/big_means.cpp + src/local_search.cpp (CPU),
// plan_b200 with the drop-in shims in their place (every cell on the B200).
#include <cstdio>
#include <exception>
#include <iostream>

#include "bigmeans/bench.hpp"

int main(int argc, char** argv) {
    if (argc != 2) {
        std::fprintf(stderr, "usage: %s <plan.json>\n", argv[0]);
        return 2;
    }
    try {
        const auto plan = bigmeans::bench::load_plan(argv[1]);
        const auto result = bigmeans::bench::run_plan(plan);
        std::cout << bigmeans::bench::result_to_json(result, plan);
        return result.any_failed ? 1 : 0;
    } catch (const bigmeans::ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
