// wide.h — tensor-core pre-screen of wide rows (wide.cu): split-K partial dot
// products x.c and squared norms of 128-point tiles, consumed by k_assign_tma's
// pre-screened mode (kernels_assign.cuh).  Host-visible plan + launch entry.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device_common.cuh"

namespace bm {
namespace dev {

struct WideArgs {
    CUtensorMap xmap;      // rows [rows][n] fp32 (stride ld), box 32 dims x 128 rows, 128-byte swizzle
    const double* Cact;    // compacted active centroids (fp64), row stride ldc
    int ldc;
    const int* n_active;
    uint64_t rows;
    int n;
    int na;                // 32-dim atoms per split; split ks covers atoms [ks*na, min(ks*na+na, natoms))
    int bpa;               // atoms per TMEM accumulator block (1 or 2)
    int natoms;            // ceil(n / 32)
    float* dot;            // [KS][rows][NP] partial dot products
    float* nx;             // [KS][rows][2]  partial squared norms of the rows (rounded down, up)
    float* nc;             // [natoms][NP][2] per-atom partial squared norms of the centroids (k_wide_prep)
    float* bops;           // [natoms][2][NP][32] B operands (hi, lo), UMMA K-major 128-byte swizzle (k_wide_prep)
    const int* stop;       // nothing to do when *stop (a finished Lloyd loop) ...
    const int* go;         // ... or when go && !*go (a chunk that waits for a repair)
    unsigned long long* dbg;  // diagnostics (-DBM_WIDE_DBG): CTA (0,0)'s per-atom globaltimer stamps
};

// k_wide_recheck: the candidates of 32 points per CTA from the split-K
// partials (certified bounds), their exact fp64 distances (direct form, dims
// streamed through shared memory), and each point's minimum (ascending j,
// strict <): compacted rank and distance.
struct RecheckArgs {
    CUtensorMap xmap;      // rows [rows][n] fp32, box 32 dims x 32 rows, 128-byte swizzle
    CUtensorMap cmap;      // Cact [k][n] fp64 (stride ldc), box 16 dims x NP rows, 128-byte swizzle
    const float* X;        // rows [rows][ld] fp32
    uint64_t ld;
    uint64_t rows;
    int n;
    const double* Cact;
    int ldc;
    const int* n_active;
    const float* dot;      // k_wide_screen's partials (WideArgs)
    const float* nx;
    const float* nc;
    int ks;
    int natoms;
    int np;
    ScreenConsts cst;
    double* best;          // [rows] exact distance to the nearest active centroid
    int* bj;               // [rows] its compacted rank
    const int* stop;
    const int* go;
};

// What k_assign_tma reads in its pre-screened mode (best == nullptr: its own screen).
struct PreDots {
    const double* best;
    const int* bj;
};

}  // namespace dev

struct WidePlan {
    bool ok = false;
    int np = 16;        // UMMA N: centroid slots (16 for k <= 16, else 32)
    int natoms = 0, na = 0, ks = 0;
    int bpa = 1;        // atoms per accumulator block
    unsigned tiles = 0; // 128-point tiles
    size_t smem = 0;
    size_t dot_floats() const { return static_cast<size_t>(ks) * tiles * 128 * np; }
    size_t nx_floats() const { return static_cast<size_t>(ks) * tiles * 128 * 2; }
    size_t nc_floats() const { return static_cast<size_t>(natoms) * np * 2; }
    size_t bops_floats() const { return static_cast<size_t>(natoms) * 2 * np * 32; }
    unsigned recheck_ctas(uint64_t rows) const { return static_cast<unsigned>((rows + 31) / 32); }
};

WidePlan wide_plan(int device, uint64_t rows, int n, int k);
dev::ScreenConsts wide_screen_consts(const WidePlan& p, int n);
CUtensorMap wide_rows_map(const void* X, uint64_t rows, int n, uint64_t ld, int box_rows = 128);
CUtensorMap wide_cent_map(const double* Cact, int k, int n, int ldc, int np);
void launch_wide_screen(cudaStream_t st, const WidePlan& p, const dev::WideArgs& a, bool pdl);
void launch_wide_recheck(cudaStream_t st, const WidePlan& p, const dev::RecheckArgs& a, bool pdl);

}  // namespace bm
