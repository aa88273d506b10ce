// device_common.cuh — device-side types and small helpers shared by the
// kernel translation units (kernels.cuh via engine.cu, chunk.cu): loop/chain
// state, the chunk record, the exact distance step, the certified-screen
// constants and packed-fp32 helpers.  Header-only, ODR-safe (inline only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace bm {
namespace dev {

// ---------------------------------------------------------------------------
// Device-side Lloyd status (one per workspace).  Mirrors the loop state of
// lloyd() local_search.cpp:16-60 so that the loop can run without host trips.
// ---------------------------------------------------------------------------
struct LloydStatus {
    double f;            // f of the previous round (local_search.cpp:27,51)
    double objective;    // history.back() (:54)
    unsigned long long evals;       // this run's distance evals (core.cpp:157-159)
    unsigned long long iterations;  // ++iterations (:36)
    int parity;          // labels[parity] holds the current assignment (slot 2: a graph-mode begin)
    int stop;            // loop finished
    int changed;         // set by the assignment when a label differs (:39)
    int state_error;     // assign against all-degenerate centroids (core.cpp:115-118)
    int inc_degenerate;  // host copy: degenerate rows of the incumbent after the accept step
    int bad_label;       // update saw a label outside [0,k) (core.cpp:189-193)
    // fast-sum control (graph mode): the stop test runs on certified intervals
    // of the objectives, the exact block_sum only when the interval test cannot
    // decide (and for the final objective, in k_accept)
    double f_lo, f_hi;   // interval of the exact f around the fast sum kept in `f`
    double fsum;         // accumulator of the current launch's CTA distance sums
    unsigned ctas_done;  // CTAs of the current launch that have added their sum
    int exact_checks;    // decisions that needed the exact sums (diagnostics)
    int incomplete;      // the graph's unrolled rounds ended without a stop: the host continues
    int sum_sel;         // exact-sum mode: which half of the chunk buffer's label sums is live (1: the redo begin's)
    long long begin_version;  // incumbent version the begin's assignment used (-1: none / stale)
    long long bv_min;         // lowest version its CTAs saw when they started (atomicMin; host resets)
};

// Chain state shared by the two chunk buffers (big_means.cpp:62-94).
struct GState {
    double fopt_exact;   // exact f_opt of the chunks whose records are final (deferred exact objectives)
    long long inc_version;  // bumped whenever the next chunk's start stops being the incumbent's copy
    int n_active;        // active rows of the working compacted centroids (Cact / CT32 / act)
    int n_active_inc;    // active rows of the incumbent's compacted copy (CactI / CT32I / actI)
    int inc_degenerate;  // degenerate rows of the incumbent
    int go;              // the next chunk starts from the incumbent as is (no repair, :83-85)
    int pending_fix;     // chunk whose record awaits its exact objective (-1: none)
    int fix_par;         // distance slot of that chunk's final assignment
    int fix_acc;         // that chunk's accept decision
    int pad;
};
static_assert(sizeof(LloydStatus) % 8 == 0, "status is copied as 8-byte words");

constexpr int kSMaxK = 32;  // centroids handled by the screened path
constexpr int kStateBufs = 4;  // graph mode: chunk c's data, labels / distances / bounds / status live in buffer c % 4

// Per-chunk accept record (ChunkRecord big_means.hpp:28-34).
struct Record {
    unsigned long long chunk_index;
    double candidate_objective;
    double incumbent_objective;
    unsigned long long accepted;
    unsigned long long degenerate_repaired;
};

// Exact promotion of the storage type (P11).
__device__ __forceinline__ double to_f64(double v) { return v; }
__device__ __forceinline__ double to_f64(float v) { return static_cast<double>(v); }

// One step of the reference distance loop core.cpp:144-145 / init.cpp:34-35:
// diff = x - c; sum += diff * diff  (three separately rounded operations).
// Programmatic dependent launch: wait for the previous kernel's completion and
// memory (no-op when not launched as a dependent); allow the next kernel to launch.
// (The assignment and the update do not trigger early: dependents that wait
// on SM slots starve the prep and speculative kernels on the other streams.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ double dist_step(double sum, double x, double c) {
    const double diff = __dsub_rn(x, c);
    return __dadd_rn(sum, __dmul_rn(diff, diff));
}

struct ScreenConsts {
    float K;      // g_b/2 + 2u' + u'^2, rounded up
    float dabs;   // absolute slack for fp32 underflow
    float lo64;   // 1-g64, rounded down
    float hi64;   // 1+g64, rounded up
};

__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
    unsigned long long d;
    const float2 bb = make_float2(b, b);
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
          "l"(*reinterpret_cast<const unsigned long long*>(&bb)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}

// Certified interval of the exact blocked sum around an unordered sum `s` of
// the same nonnegative terms: both differ from the real sum by at most
// gamma_(additions on the longest path) times that sum.
__device__ __forceinline__ void sum_interval(double s, uint64_t rows, unsigned ctas, double* lo, double* hi) {
    const double adds = static_cast<double>(tiles_of(rows) + ctas + kTile + 16);
    const double rel = __dmul_ru(adds, 0x1.02p-53);  // (1 - n u)^-1 <= 1.01 for n u < 0.01
    const double e = __dadd_ru(__dmul_ru(s, rel), 0x1p-1000);
    *lo = __dsub_rd(s, e);
    *hi = __dadd_ru(s, e);
}


}  // namespace dev
}  // namespace bm
