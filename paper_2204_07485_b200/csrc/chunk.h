// chunk.h — the persistent chunk kernel (chunk.cu): one cooperative launch
// runs a whole Big-means chunk on the device — lloyd (local_search.cpp:16-60:
// the first assignment, every update/assign round, the stop tests) and the
// accept (big_means.cpp:89-94) with its record — with the chunk's rows held
// in shared memory across all rounds.  Host-visible plan + launch entry.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "bigmeans_b200.h"
#include "device_common.cuh"

namespace bm {
namespace dev {

// The deferred exact objective of one chunk (k_chunk -> k_chunk_fix, per
// chunk buffer): block_sum of its final distances (core.cpp:165-175) is folded
// by a small kernel on a side stream while the next chunk runs.
struct FixJob {
    unsigned long long chunk;
    double fo;        // exact f_opt before this chunk's accept
    int slot;         // distance slot of the final assignment
    int accepted;
    int have_exact;   // the accept needed the exact objective: record / f_opt already final
    int valid;
};

// Everything one chunk launch reads and writes (pointers into the Workspace).
struct ChunkArgs {
    // tensor map of the gathered chunk (2-D [rows][n], stride ld): the rows
    // land in shared memory by TMA — tensor-core screen: 32-dim x 128-row
    // boxes in the UMMA K-major 128-byte-swizzle layout; otherwise xld-wide x
    // chunk_box_rows(B)-row boxes, row-major (dims n..xld-1 and rows past the
    // chunk zero-filled)
    CUtensorMap xmap;
    const void* X;            // the gathered chunk: rows x ld, storage T
    uint64_t rows;            // s
    int n;
    uint64_t ld;              // global row stride (elements)
    int k;
    int threads;              // working threads per CTA (the launch may be padded beyond them)
    int B;                    // points per CTA (ordered mode: 1024 = one reduction tile)
    int xld;                  // shared-memory row stride (elements)
    int ordered;              // 1: real-valued data, CTA = 1024-tile, tile-order merge; 0: exact sums
    int rows_tf32_exact;      // every dataset value is exactly a tf32 (no per-CTA check needed)
    double* C;                // working centroids k x n (the start; then every update)
    uint8_t* mask;            // their degenerate mask
    double* part;             // update partials [G][k*n] (CTA g's fold of label j, dim d)
    unsigned* pcnt;           // member counts [G][k]
    double* dists;            // [2][rows]: the distances of the last two assignments
    double* tiles;            // [2][ntiles]: exact 1024-tile partials (tolerance fallback, accept)
    unsigned* bar;            // grid barrier: [0] arrivals, [1] generation; [2] CTAs past their last control read
    double* rsum;             // [3] per-round fast distance sums (slot = round & 1; red mode: round % 3)
    int* rchg;                // [3] per-round "a label changed" flags
    // red mode (exact-sum data, one grid barrier per round): label-sum deltas
    // of round r's assignment, added by RED into dsum[r % 3] / dcnt[r % 3];
    // every CTA keeps the running sums in shared memory and forms the
    // centroids itself (any order of exact sums gives the reference's bits)
    int red;
    double* dsum;             // [3][k*n], all zero between launches
    int* dcnt;                // [3][k]
    ScreenConsts cst;         // screen bounds: packed-FFMA (fp64 rows) / tensor core, rows exact in tf32
    ScreenConsts cst_loose;   // tensor core, rows not exact in tf32 (truncated by the MMA)
    unsigned long long max_iterations;
    double rel_tolerance;
    int force_exact;          // test hook: every interval decision takes the exact path
    // accept (big_means.cpp:89-94) and chain state
    double* f_opt;
    double* Cinc;
    uint8_t* maskinc;
    Record* rec_base;
    unsigned long long* chunk_ctr;
    GState* gs;
    LloydStatus* st;          // this chunk buffer's status
    LloydStatus* host_st;     // mapped host copy of it
    unsigned long long* timing;  // optional [2 * timing_cap]: per chunk, globaltimer at CTA 0's start and the accept's end
    unsigned long long timing_cap;
    unsigned long long* dbg;  // optional [4][8][16] phase stamps (BM_CHUNK_DBG)
    int dbg_mma;              // diagnostics (BM_CHUNK_DBG=2): max observed MMA dot error into dbg
    FixJob* job;              // this chunk buffer's deferred exact objective
    unsigned long long* fix_seq;  // chunks whose exact objective is final (k_chunk_fix)
};

// k_chunk_fix: grid = tiles of the chunk, one CTA per 1024-row tile.
struct FixArgs {
    FixJob* job;
    const double* dists;      // the chunk buffer's [2][rows] distances
    uint64_t rows;
    double* tiles;            // [ntiles]
    unsigned* counter;
    Record* rec_base;
    double* f_opt;
    GState* gs;
    unsigned long long* fix_seq;
};

}  // namespace dev

// Launch geometry for one (s, n, k, storage) — ok == false: use the
// multi-launch path (engine.cu).
struct ChunkPlan {
    bool ok = false;
    bool tc = false;  // tensor-core screen (fp32 rows, swizzled layout)
    int B = 0, threads = 0, ppt = 0, nd = 0, xld = 0, ordered = 0;
    int red = 0;      // exact sums by RED deltas, one grid barrier per round
    unsigned grid = 0;
    size_t smem = 0;
};

ChunkPlan chunk_plan(int device, uint64_t s, int n, int k, bm_dtype storage, bool exact_sums, bool tc, bool red = true);
// The row tensor map of one gathered chunk buffer for a plan.
CUtensorMap chunk_rows_map(const ChunkPlan& p, bm_dtype storage, const void* X, uint64_t rows, int n, uint64_t ld);
// Enqueue one chunk (cooperative launch, capturable into a graph).
void launch_chunk(cudaStream_t st, const ChunkPlan& p, bm_dtype storage, const dev::ChunkArgs& a);
// k_chunk_fix prefers the maximum shared-memory carveout (current device).
void chunk_fix_prefer_max_smem();
// Enqueue the deferred exact objective of the chunk just launched (side stream).
void launch_chunk_fix(cudaStream_t st, const dev::FixArgs& f);
// The certified-screen constants of the chunk kernel's dot products: the
// packed-FFMA screen (tc = false) or the tensor-core screen (tc = true, with
// rows exactly representable in tf32 or not).
dev::ScreenConsts chunk_screen_consts(int n, bool tc = false, bool rows_tf32_exact = true);

}  // namespace bm
