// common.cuh — error taxonomy, CUDA checks and shared constants.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace bm {

// kReductionBlock threading.hpp:15 — every fp64 total is a left fold over
// 1024-point tiles followed by a left fold over tile partials (core.cpp:163-175).
constexpr int kTile = 1024;

// Mirrors of the reference exception types (common.hpp:21-24, 46-49).
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct StateError : std::runtime_error {
    explicit StateError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                        std::to_string(line) + ")");
    }
}

#define BM_CUDA(x) ::bm::cuda_check((x), #x, __FILE__, __LINE__)
#define BM_LAUNCH() ::bm::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t tiles_of(uint64_t rows) { return ceil_div(rows, kTile); }

}  // namespace bm
