// finaltc.h — the final full-data assignment on the tensor core (finaltc.cu):
// fp32 rows exact in tf32, n <= 88, k <= 32.  Host-visible args + launch entry.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"

namespace bm {
namespace dev {

struct FinalTcArgs {
    CUtensorMap xmap;       // rows [rows][n] fp32 (stride ld), box 32 dims x 128 rows, 128-byte swizzle
    uint64_t rows;
    int n;
    const double* Cact;     // compacted active centroids (fp64), row stride ldc
    int ldc;
    const int* act;         // compacted rank -> label
    const int* n_active;
    ScreenConsts cst;       // the chunk kernel's tensor-core bound (chunk_screen_consts(n, true, true))
    int32_t* labels;        // [rows]
    double* dists;          // [rows]
};

}  // namespace dev

bool final_tc_supported(int n, int k);
CUtensorMap final_tc_map(const void* X, uint64_t rows, int n, uint64_t ld);
void launch_final_tc(cudaStream_t st, int device, const dev::FinalTcArgs& a, bool pdl);

}  // namespace bm
