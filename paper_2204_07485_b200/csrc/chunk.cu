// chunk.cu — persistent chunk kernel: one cooperative launch per Big-means
// chunk (lloyd local_search.cpp:16-60 + accept big_means.cpp:89-94).
//
// Why: the multi-launch path (engine.cu) streams the chunk from L2 through a
// TMA ring on every round and pays two launches and CTA-wide phase barriers
// per round; on B200 that left the chunk-loop assignment at 0.05-0.15 of the
// HBM roofline.  Here the chunk's rows are loaded into shared memory ONCE
// (148 SMs x 227 KB holds a c2/c3 chunk) and every round reuses them; rounds
// are separated by two grid barriers instead of kernel boundaries.
//
// Layout.  CTA g owns rows [g*B, g*B+B) of the chunk.  Real-valued data
// ("ordered" mode): B = 1024, so CTA g IS reduction tile g and every
// per-tile fold of the reference (update partials core.cpp:200-215, block_sum
// core.cpp:165-173) is CTA-local and sequential in index order; partials are
// merged in tile order (core.cpp:217-229).  Exact-sum data (every value an
// integer multiple of 2^e, m*max|x| < 2^52*2^e: DESIGN §3.2b): all sums are
// exact in fp64 whatever the order, so B is chosen to spread the chunk over
// the SMs.
//
// One round (r >= 1):  [load centroids C from global -> compacted fp32/fp64
// copies + norms]  assign (certified fp32 screen with the point rows in
// registers, exact fp64 direct-form recheck of the candidates in ascending j,
// strict <: reproduces assign_nearest core.cpp:129-155 bit for bit) ->
// speculative update partials of the new labels (stable member lists, one
// thread per (label, dim) folding the members in index order) -> grid
// barrier A (fast distance sums and "changed" flags arrive with it) -> the
// stop tests of local_search.cpp:39-50, decided identically by every CTA on
// certified intervals of the unordered sums (exact block sums only when the
// interval cannot decide) -> merge of the partials (one thread per (label,
// dim), tile order, sum * (1.0/count): core.cpp:231-242) -> grid barrier B.
// After the stop: exact block_sum of the final distances (tile folds, tile
// order), the strict accept against f_opt, the record, the next start.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <mutex>
#include <utility>
#include <vector>

#include "chunk.h"
#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace bm {
namespace dev {
namespace {

constexpr int kCMaxT = 512;  // threads per CTA
constexpr int kCKMax = 32;   // centroids (labels) per chunk kernel

__device__ __forceinline__ float2 ffma2x(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

__device__ __forceinline__ unsigned long long u2(float2 a) { return *reinterpret_cast<const unsigned long long*>(&a); }
__device__ __forceinline__ float2 f2(unsigned long long v) { return *reinterpret_cast<const float2*>(&v); }
#define BM_F2OP2(name, ins)                                                    \
    __device__ __forceinline__ float2 name(float2 a, float2 b) {              \
        unsigned long long d;                                                  \
        asm(ins " %0, %1, %2;" : "=l"(d) : "l"(u2(a)), "l"(u2(b)));            \
        return f2(d);                                                          \
    }
BM_F2OP2(add2_rd, "add.rm.f32x2")
BM_F2OP2(add2_ru, "add.rp.f32x2")
BM_F2OP2(sub2_rd, "sub.rm.f32x2")
BM_F2OP2(sub2_ru, "sub.rp.f32x2")
BM_F2OP2(mul2_rd, "mul.rm.f32x2")
BM_F2OP2(mul2_ru, "mul.rp.f32x2")
BM_F2OP2(mul2_rn, "mul.rn.f32x2")
BM_F2OP2(add2_rn, "add.rn.f32x2")
#undef BM_F2OP2
__device__ __forceinline__ float2 fma2_ru(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rp.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(u2(a)), "l"(u2(b)), "l"(u2(c)));
    return f2(d);
}
__device__ __forceinline__ float2 ffma2s(float2 a, float b, float2 c) { return ffma2x(a, make_float2(b, b), c); }

// Certified bounds of two (point, centroid) pairs at once (the screen's error
// model, DESIGN §3.1 / chunk_screen_consts): dot = fp32 dot products, nx* / nc*
// the fp32 norms (sum of squares rounded down / up, sqrt of the upper rounded
// up; out-of-range rows carry (0, inf, inf), which yields L = 0 and a U that
// never lowers the minimum).
__device__ __forceinline__ void bounds2(float2 dot, float2 nxl, float2 nxh, float2 nxr, float2 ncl, float2 nch,
                                        float2 ncr, const ScreenConsts& c, float2& L, float2& U) {
    const float2 t2 = mul2_rn(dot, make_float2(2.f, 2.f));  // exact
    const float2 Sn = add2_ru(nxr, ncr);
    const float2 D = fma2_ru(mul2_ru(Sn, make_float2(c.K, c.K)), Sn, make_float2(c.dabs, c.dabs));
    const float2 Al = add2_rd(nxl, ncl), Ah = add2_ru(nxh, nch);
    const float2 Lr = mul2_rd(sub2_rd(sub2_rd(Al, t2), D), make_float2(c.lo64, c.lo64));
    L = make_float2(fmaxf(Lr.x, 0.f), fmaxf(Lr.y, 0.f));
    U = mul2_ru(add2_ru(sub2_ru(Ah, t2), D), make_float2(c.hi64, c.hi64));
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier (all CTAs co-resident: cooperative launch).  Generation
// counting: the arrival counter returns to 0 at every barrier, the generation
// only grows, so the state carries over between launches.  The CTA's writes
// are ordered before thread 0's release arrival by the CTA barrier (release is
// cumulative); the waiters' acquire loads order everything after.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(bar + 1);
        unsigned arrived;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
        if (arrived == G - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
            while (ld_acquire(bar + 1) == gen) {
            }
        }
    }
    __syncthreads();
}

// One lane of the (converged) calling warp.
__device__ __forceinline__ bool elect_one() {
    unsigned pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xFFFFFFFF;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Left fold from 0.0 of `len` doubles (global, L2; loads issued ahead of the adds).
__device__ double fold_global(const double* v, int len) {
    double a = 0.0;
    int i = 0;
    for (; i + 16 <= len; i += 16) {
        double t[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) t[r] = __ldcg(v + i + r);
#pragma unroll
        for (int r = 0; r < 16; ++r) a = __dadd_rn(a, t[r]);
    }
    for (; i < len; ++i) a = __dadd_rn(a, __ldcg(v + i));
    return a;
}

// Direct-form squared distance (core.cpp:142-146): x row (storage T, shared
// memory, 16-byte aligned), c row fp64 (shared, 16-byte aligned).
template <typename T>
__device__ __forceinline__ double exact_dist(const T* __restrict__ x, const double* __restrict__ c, int n) {
    double s = 0.0;
    int d = 0;
    if constexpr (sizeof(T) == 4) {
        for (; d + 4 <= n; d += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(x + d);
            const double2 c0 = *reinterpret_cast<const double2*>(c + d);
            const double2 c1 = *reinterpret_cast<const double2*>(c + d + 2);
            s = dist_step(s, static_cast<double>(xv.x), c0.x);
            s = dist_step(s, static_cast<double>(xv.y), c0.y);
            s = dist_step(s, static_cast<double>(xv.z), c1.x);
            s = dist_step(s, static_cast<double>(xv.w), c1.y);
        }
    } else {
        for (; d + 2 <= n; d += 2) {
            const double2 xv = *reinterpret_cast<const double2*>(x + d);
            const double2 c0 = *reinterpret_cast<const double2*>(c + d);
            s = dist_step(s, xv.x, c0.x);
            s = dist_step(s, xv.y, c0.y);
        }
    }
    for (; d < n; ++d) s = dist_step(s, to_f64(x[d]), c[d]);
    return s;
}

// ---- tcgen05 / TMEM helpers (umma.cuh) under the names used below ----
using umma::smem_addr;
using umma::mbar_wait_parity;
using umma::tf32_rna;
using umma::tmem_ld32;
__device__ __forceinline__ unsigned long long umma_desc_sw128_units(unsigned u) { return umma::desc_sw128(u); }
constexpr unsigned kTcIdesc = umma::idesc_tf32<64>();  // N = 64: 32 hi slots, then 32 lo slots
__device__ __forceinline__ void umma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db, int acc) {
    umma::mma_tf32(tmem_d, da, db, kTcIdesc, acc);
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) { umma::commit(bar); }
__device__ __forceinline__ void tc_fence_before() { umma::fence_before(); }
__device__ __forceinline__ void tc_fence_after() { umma::fence_after(); }
__device__ __forceinline__ void fence_proxy_async_smem() { umma::fence_proxy_async_smem(); }

// Global -> shared copies with U loads in flight per thread (a plain
// load-then-store loop would wait one L2 round trip per element).
template <int U, class Load, class Store>
__device__ __forceinline__ void batched_copy(int count, int tid, int NT, Load ld, Store st) {
    for (int e0 = tid; e0 < count; e0 += U * NT) {
        decltype(ld(0)) v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * NT;
            if (e < count) v[u] = ld(e);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * NT;
            if (e < count) st(e, v[u]);
        }
    }
}

// Left fold from 0.0 of `len` doubles in shared memory (16-byte aligned).
__device__ __forceinline__ double fold_smem(const double* v, int len) {
    double a = 0.0;
    int i = 0;
    for (; i + 8 <= len; i += 8) {
        const double2 v0 = *reinterpret_cast<const double2*>(v + i);
        const double2 v1 = *reinterpret_cast<const double2*>(v + i + 2);
        const double2 v2 = *reinterpret_cast<const double2*>(v + i + 4);
        const double2 v3 = *reinterpret_cast<const double2*>(v + i + 6);
        a = __dadd_rn(a, v0.x);
        a = __dadd_rn(a, v0.y);
        a = __dadd_rn(a, v1.x);
        a = __dadd_rn(a, v1.y);
        a = __dadd_rn(a, v2.x);
        a = __dadd_rn(a, v2.y);
        a = __dadd_rn(a, v3.x);
        a = __dadd_rn(a, v3.y);
    }
    for (; i < len; ++i) a = __dadd_rn(a, v[i]);
    return a;
}

}  // namespace

// Shared-memory carve-up (host and device agree).
struct CLayout {
    size_t xs, cb, u, cf, cd, ssum, scnt, nrm, act, lab, dist, red, total;
    int cdld;         // fp64 centroid row stride: even, an odd number of 16-byte units
};

__host__ __device__ inline int chunk_cdld(int n) {
    int c = n + (n & 1);
    if (((c / 2) & 1) == 0) c += 2;
    return c;
}

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Rows per TMA box of the row-major (non tensor-core) layout: the CTA's B rows
// in the fewest boxes of <= 256 rows, all of one size.
__host__ __device__ inline int chunk_box_rows(int B) {
    const int nb = (B + 255) / 256;
    return ((B + nb - 1) / nb + 7) / 8 * 8;  // a multiple of 8 rows: 128-byte aligned boxes
}

// Tensor-core layout of the fp32 rows (tc): UMMA K-major, 128-byte swizzle.
// K-atoms of 32 dims; atom `ka` holds Mpad rows x 128 B (rows 8-grouped into
// 1024 B core-matrix groups, 16-byte chunks XOR-swizzled by row & 7).
__host__ __device__ inline int tc_mpad(int B) { return (B + 127) / 128 * 128; }
__host__ __device__ inline int tc_katoms(int nd) { return (nd + 31) / 32; }

__host__ __device__ inline CLayout chunk_layout(int B, int xld, int es, int k, int nd, int n, unsigned G,
                                                bool tc = false, bool redm = false) {
    CLayout L{};
    size_t o = 0;
    L.xs = o;
    if (tc) {  // rows (A operand) + centroid hi / lo parts (B operands), 1024-aligned
        o += (size_t)tc_katoms(nd) * tc_mpad(B) * 128;
        L.cb = o;
        o += (size_t)2 * tc_katoms(nd) * kCKMax * 128;
    } else {  // whole TMA boxes of chunk_box_rows(B) rows
        o = al16(o + (size_t)chunk_box_rows(B) * ((B + chunk_box_rows(B) - 1) / chunk_box_rows(B)) * xld * es);
        L.cb = o;
    }
    // region U (aliased): screen lower bounds Ls[k][B] (FFMA screen) | member
    // lists for the update | staging of this CTA's merge pairs | staged
    // distance / tile partials
    const size_t ls = tc ? 0 : (size_t)k * B * 4;
    const int nc = (B + 31) / 32;
    const size_t sort = al16((size_t)B * 2) + al16((size_t)B) + al16((size_t)nc * k * 4) + al16((size_t)(2 * k + 2) * 4);
    const size_t kn = (size_t)k * n, ppc = (kn + G - 1) / G;
    // (red mode: no merge staging — every CTA keeps the label sums, below)
    const size_t merge = redm ? 0 : al16(ppc * G * 8) + al16((ppc / (size_t)n + 2) * G * 4);
    // exact-sum mode: a staged 1024-row tile of distances (red mode: in the rows' region when it is large enough)
    const size_t tailf = redm && L.cb - L.xs >= (size_t)kTile * 8 ? 0 : (size_t)kTile * 8;
    size_t u = ls > sort ? ls : sort;
    u = u > merge ? u : merge;
    u = u > tailf ? u : tailf;
    L.cdld = chunk_cdld(n);
    L.u = o;
    o = al16(o + u);
    L.cf = o;
    if (!tc) o = al16(o + (size_t)kCKMax * nd * 4);
    L.cd = o;
    o = al16(o + (size_t)k * chunk_cdld(n) * 8);
    L.ssum = o;  // red mode: running label sums [k][cdld] (fp64) and member counts
    if (redm) o = al16(o + (size_t)k * chunk_cdld(n) * 8);
    L.scnt = o;  // [kCKMax] 1.0 / count (fp64), then [2][kCKMax] counts (by round parity)
    if (redm) o = al16(o + (size_t)kCKMax * 16);
    L.nrm = o;
    o = al16(o + 3 * kCKMax * 4);
    L.act = o;
    o = al16(o + (kCKMax + 4) * 4);
    L.lab = o;
    o = al16(o + (size_t)B * 4);
    L.dist = o;
    o = al16(o + (size_t)B * 8);
    L.red = o;
    o = al16(o + 64 * 8);
    L.total = o + (tc ? 1024 : 128);  // slack to align the base (tc: 1024 B for the swizzle atoms; TMA boxes: 128 B)
    return L;
}

// Per-CTA control state, identical in every CTA (computed from the same
// global values after each barrier).
struct CCtl {
    double f, f_lo, f_hi;
    unsigned long long evals, iterations;
    int stop, undecided, ka, state_error;
    unsigned gdirty;  // labels whose membership changed in some tile this round
    double s_last, lo_last, hi_last;  // fast sum (and its interval) of the last assignment
    double fo;                        // exact f_opt before the accept
    int decision;                     // accept: 1 / 0, -1: the interval cannot decide (exact fold)
};

// Debug phase stamps (ChunkArgs::dbg, BM_CHUNK_DBG=1): CTA 0's globaltimer at
// the phase boundaries of rounds 0..6 (row 7: the tail), chunk % 4.
#define CDBG(row, ph)                                                                        \
    do {                                                                                     \
        if (a.dbg && cta == 0 && tid == 0 && (row) < 8)                                      \
            a.dbg[((s_chunk & 3ull) * 8 + (row)) * 16 + (ph)] = gtimer();                    \
    } while (0)

template <typename T, int ND, int PPT, bool TC, bool RED>
__global__ void __launch_bounds__(kCMaxT, 1) k_chunk(const __grid_constant__ ChunkArgs a) {
    // RED: exact-sum data, label-sum deltas by RED and one grid barrier per round (ChunkArgs::red)
    // TC (fp32 rows): tensor-core screen (tcgen05.mma kind::tf32, TMEM
    // accumulators) over rows in the swizzled K-major layout; otherwise the
    // packed-FFMA screen with the rows in registers (row-major shared rows)
    static_assert(!TC || sizeof(T) == 4, "the tensor-core screen reads fp32 rows");
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const unsigned long long t_entry = gtimer();
    // (a.threads < blockDim.x: the launch is padded with warps that leave at once — their
    // registers stay allocated, so no side kernel's CTA fits beside this one; BM_CHUNK_OWN_SM=1)
    if (static_cast<int>(threadIdx.x) >= a.threads) return;
    const int tid = threadIdx.x, NT = a.threads, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
    const unsigned G = gridDim.x, cta = blockIdx.x;
    const int B = a.B, n = a.n, k = a.k, xld = a.xld;
    const uint64_t p0 = static_cast<uint64_t>(cta) * B;
    const int np = static_cast<int>(min(static_cast<uint64_t>(B), a.rows - p0));
    const CLayout L = chunk_layout(B, xld, (int)sizeof(T), k, ND, n, G, TC, RED);
    // tc: operand tiles need a 1024-byte aligned base (128-byte swizzle atoms)
    unsigned char* sm = TC ? sm_raw + ((1024u - (smem_addr(sm_raw) & 1023u)) & 1023u)
                           : sm_raw + ((128u - (smem_addr(sm_raw) & 127u)) & 127u);
    const int cdld = L.cdld;
    const int MP = tc_mpad(B), NKA = tc_katoms(ND);
    const size_t ASZ = static_cast<size_t>(MP) * 128;  // bytes of one K-atom of the rows
    T* xs = reinterpret_cast<T*>(sm + L.xs);
    float* Ls = reinterpret_cast<float*>(sm + L.u);
    float* cf = reinterpret_cast<float*>(sm + L.cf);
    double* cd = reinterpret_cast<double*>(sm + L.cd);
    float* ncl = reinterpret_cast<float*>(sm + L.nrm);
    float* nch = ncl + kCKMax;
    float* ncr = nch + kCKMax;
    int* act = reinterpret_cast<int*>(sm + L.act);
    int* lab = reinterpret_cast<int*>(sm + L.lab);
    double* dist = reinterpret_cast<double*>(sm + L.dist);
    double* red = reinterpret_cast<double*>(sm + L.red);
    double* ssum = reinterpret_cast<double*>(sm + L.ssum);  // red mode
    double* sinv = reinterpret_cast<double*>(sm + L.scnt);
    int* scnt = reinterpret_cast<int*>(sm + L.scnt + kCKMax * 8);
    const int kn = k * n;
    __shared__ CCtl ctl;
    __shared__ int s_any;
    __shared__ unsigned s_tmem;
    __shared__ __align__(8) unsigned long long s_mbar;
    __shared__ __align__(8) uint64_t s_xbar;  // the rows' TMA boxes
    const float finf = __int_as_float(0x7F800000);
    const double dinf = __longlong_as_double(0x7FF0000000000000LL);
    __shared__ unsigned long long s_chunk;
    // (no repair before this chunk: its start is the incumbent's copy — red mode leaves C / mask untouched)
    bool start_is_inc = false;
    // 16-byte chunk q of row p (fp32: dims 4q..4q+3; fp64: 2q, 2q+1):
    // tc rows in the swizzled K-major layout, else row-major with stride xld
    auto xchunk = [&](int p, int q) -> unsigned char* {
        if constexpr (TC) {
            const int ka = q >> 3, c = q & 7;  // (p >> 3) * 1024 + (p & 7) * 128 == p * 128
            return sm + L.xs + static_cast<size_t>(ka) * ASZ + static_cast<size_t>(p) * 128 + ((c ^ (p & 7)) << 4);
        } else {
            return sm + L.xs + static_cast<size_t>(p) * xld * sizeof(T) + static_cast<size_t>(q) * 16;
        }
    };
    constexpr int EPC = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte chunk
    auto xat = [&](int p, int d) -> T { return reinterpret_cast<const T*>(xchunk(p, d / EPC))[d % EPC]; };
    // direct-form squared distance of row p to compacted fp64 row j (core.cpp:142-146)
    auto exact = [&](int p, int j) -> double {
        const double* c = cd + j * cdld;
        double s = 0.0;
        int d = 0;
        if constexpr (TC) {
            const unsigned char* rowb = sm + L.xs + static_cast<size_t>(p) * 128;
            const int sw = p & 7;
            for (; d + 4 <= n; d += 4) {
                const int q = d >> 2;
                const float4 xv = *reinterpret_cast<const float4*>(rowb + static_cast<size_t>(q >> 3) * ASZ +
                                                                    (((q & 7) ^ sw) << 4));
                const double2 c0 = *reinterpret_cast<const double2*>(c + d);
                const double2 c1 = *reinterpret_cast<const double2*>(c + d + 2);
                s = dist_step(s, static_cast<double>(xv.x), c0.x);
                s = dist_step(s, static_cast<double>(xv.y), c0.y);
                s = dist_step(s, static_cast<double>(xv.z), c1.x);
                s = dist_step(s, static_cast<double>(xv.w), c1.y);
            }
            for (; d < n; ++d) s = dist_step(s, static_cast<double>(xat(p, d)), c[d]);
            return s;
        } else {
            return exact_dist(xs + static_cast<size_t>(p) * xld, c, n);
        }
    };

    // Tensor-core screen: a whole (converged) warp calls this, its elected lane
    // issues the tile MMAs and their commit: D[tile] = rows . (hi + lo)^T over K
    // (inside a one-thread branch the compiler wraps every MMA in an election loop)
    auto issue_mma = [&]() {
        tc_fence_after();
        if (!elect_one()) return;
        // descriptors from their 14-bit start-address field (units of
        // 16 B); k-steps outer, tiles inner: consecutive MMAs feed
        // different accumulators
        const unsigned ua0 = smem_addr(sm + L.xs) >> 4;  // start addresses, 16-byte units
        const unsigned ub0 = smem_addr(sm + L.cb) >> 4;
        const int ntl = MP / 128;
        // k-steps of 8 dims (dims n..ND-1 are zero in both operands);
        // D[tile] (64 columns) = rows . [hi | lo]^T
        constexpr int KSTEPS = ND / 8;
        for (int ks = 0; ks < KSTEPS; ++ks) {
            const unsigned ko = ((ks & 3) * 32) >> 4;
            const unsigned bo = (((ks >> 2) * 2 * kCKMax * 128) >> 4) + ko;
            const unsigned ao = static_cast<unsigned>((static_cast<size_t>(ks >> 2) * ASZ) >> 4) + ko;
            const unsigned long long db = umma_desc_sw128_units(ub0 + bo);
            for (int t = 0; t < ntl; ++t) {
                const unsigned long long da = umma_desc_sw128_units(ua0 + ao + static_cast<unsigned>(t) * (16384 >> 4));
                umma_tf32(s_tmem + 64u * t, da, db, ks > 0);
            }
        }
        umma_commit(&s_mbar);
    };
    int prevKA = 0;  // tc: B operand rows holding values (the rest are 0)
    // C (global) -> compacted active rows: fp64 (exact recheck) and the screen's
    // fp32 / tf32 hi+lo copies, then their certified fp32 norms
    auto load_centroids = [&](int rr, unsigned long long r) {
        const bool own = RED && r > 0;  // centroids from this CTA's label sums (core.cpp:231-242)
        // B operand of K-atom ka: 64 rows = [hi of slots 0..31][lo of slots 0..31] (one N = 64 MMA per k-step)
        unsigned char* cbhi = sm + L.cb;
        unsigned char* cblo = cbhi + kCKMax * 128;
        auto boff = [&](int rk, int d) -> size_t {
            return static_cast<size_t>(d >> 5) * (2 * kCKMax * 128) + rk * 128 + ((((d >> 2) & 7) ^ (rk & 7)) << 4) +
                   (d & 3) * 4;
        };
        // compacted row rk, dim d := v (fp64 for the recheck, the screen's fp32 / tf32 hi + lo copy)
        auto put = [&](int rk, int d, double v) {
            cd[rk * cdld + d] = v;
            const float f = __double2float_rn(v);
            if constexpr (TC) {
                const float hi = tf32_rna(f);
                const size_t off = boff(rk, d);
                *reinterpret_cast<float*>(cbhi + off) = hi;
                *reinterpret_cast<float*>(cblo + off) = f - hi;
            } else {
                cf[rk * ND + d] = f;
            }
        };
        int KA;
        if (own) {
            // One pass, no CTA barrier inside: every warp takes the member
            // counts (previous counts + the deltas), their reciprocals
            // (:237-239) and the active mask; every thread adds the deltas of
            // the previous assignment to its elements of the label sums (exact
            // sums: any order) and writes the centroid sum * (1.0 / count) into
            // the compacted row of its label.
            const int pr = static_cast<int>((r - 1) % 3);
            int cj = 0;
            double inv = 0.0;
            if (lane < k) {
                cj = scnt[((r - 1) & 1) * kCKMax + lane] + __ldcg(a.dcnt + pr * k + lane);
                inv = cj > 0 ? __ddiv_rn(1.0, static_cast<double>(cj)) : 0.0;
            }
            const unsigned live = __ballot_sync(0xFFFFFFFFu, lane < k && cj > 0);
            KA = __popc(live);
            if (warp == 0) {  // (scnt is double-buffered by round parity: the other warps read the previous counts)
                if (lane < k) {
                    scnt[(r & 1) * kCKMax + lane] = cj;
                    sinv[lane] = inv;
                    if (cj > 0) act[__popc(live & ((1u << lane) - 1u))] = lane;
                }
                if (lane == 0) act[kCKMax] = KA;
            }
            const double* dsrc = a.dsum + static_cast<size_t>(pr) * kn;
            for (int e0 = 0; e0 < kn; e0 += 4 * NT) {  // (warp-uniform trip count: shuffles inside)
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * NT + tid;
                    v[u] = e < kn ? __ldcg(dsrc + e) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * NT + tid;
                    const bool ok = e < kn;
                    const int j = ok ? e / n : 0, d = ok ? e - j * n : 0;
                    const double invj = __shfl_sync(0xFFFFFFFFu, inv, j);
                    if (ok) {
                        double* sp = ssum + j * cdld + d;
                        const double S = __dadd_rn(*sp, v[u]);
                        *sp = S;
                        if ((live >> j) & 1u) put(__popc(live & ((1u << j) - 1u)), d, __dmul_rn(S, invj));
                    }
                }
            }
            CDBG(rr, 10);
            CDBG(rr, 11);
        } else {
            CDBG(rr, 10);
            // the active list from the mask, then the active rows with every load
            // of a thread in flight at once (U = 4)
            if (warp == 0) {
                const bool live = lane < k && !__ldcg(a.mask + lane);
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, live);
                if (live) act[__popc(bal & ((1u << lane) - 1u))] = lane;
                if (lane == 0) act[kCKMax] = __popc(bal);
            }
            __syncthreads();
            CDBG(rr, 11);
            KA = act[kCKMax];
            batched_copy<4>(
                KA * n, tid, NT,
                [&](int e) {
                    const int rk = e / n;
                    return __ldcg(a.C + static_cast<size_t>(act[rk]) * n + (e - rk * n));
                },
                [&](int e, double v) {
                    const int rk = e / n;
                    put(rk, e - rk * n, v);
                });
        }
        if constexpr (TC) {
            for (int e = KA * n + tid; e < prevKA * n; e += NT) {  // rows that held values last round
                const int rk = e / n, d = e - rk * n;
                const size_t off = boff(rk, d);
                *reinterpret_cast<float*>(cbhi + off) = 0.f;
                *reinterpret_cast<float*>(cblo + off) = 0.f;
            }
            prevKA = KA;
            fence_proxy_async_smem();
        }
        __syncthreads();
        if (rr > 0) CDBG(rr, 13);
        // tensor core, rounds >= 1 (round 0 waits for the rows): the last warp
        // issues the MMAs while the other warps take the norms
        const bool split = TC && r > 0 && NW > 1;
        if constexpr (TC) {
            if (r > 0 && warp == (NW > 1 ? NW - 1 : 0)) issue_mma();
        }
        const int NWN = split ? NW - 1 : NW;
        for (int rk = warp; rk < KA && warp < NWN; rk += NWN) {
            float lo = 0.f, hi = 0.f;
            for (int d = lane; d < n; d += 32) {
                const float f = TC ? __double2float_rn(cd[rk * cdld + d]) : cf[rk * ND + d];
                lo = __fmaf_rd(f, f, lo);
                hi = __fmaf_ru(f, f, hi);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo = __fadd_rd(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
                hi = __fadd_ru(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
            }
            if (lane == 0) {
                const bool ok = hi <= 1.0e36f;  // beyond: (0, inf, inf), see bounds2
                ncl[rk] = ok ? lo : 0.f;
                nch[rk] = ok ? hi : finf;
                ncr[rk] = ok ? __fsqrt_ru(hi) : finf;
            }
        }
        CDBG(rr, 15);
    };
    // ---- the chunk's rows -> shared memory (once for all rounds) ----
    int xinexact = 0;  // tc: some row value is not exactly a tf32 (looser screen bound)
    {
        // TMA boxes of the chunk's rows, completion on s_xbar (one thread issues)
        if (tid == 0) {
            mbar_init(&s_xbar, 1);
            fence_mbar_init();
            tma_prefetch_map(&a.xmap);
            if constexpr (TC) {
                const int ntl = MP / 128;
                mbar_expect_tx(&s_xbar, static_cast<unsigned>(ntl * NKA * 16384));
                for (int t = 0; t < ntl; ++t)
                    for (int ka = 0; ka < NKA; ++ka)
                        tma_load_2d(sm + L.xs + static_cast<size_t>(ka) * ASZ + static_cast<size_t>(t) * 16384, &a.xmap,
                                    &s_xbar, ka * 32, static_cast<int>(p0) + 128 * t);
            } else {
                const int RB = chunk_box_rows(B), nb = (B + RB - 1) / RB;
                mbar_expect_tx(&s_xbar, static_cast<unsigned>(nb * RB * xld * sizeof(T)));
                for (int i = 0; i < nb; ++i)
                    tma_load_2d(sm + L.xs + static_cast<size_t>(i) * RB * xld * sizeof(T), &a.xmap, &s_xbar, 0,
                                static_cast<int>(p0) + RB * i);
            }
        }
        // while the rows are in flight: the round-0 centroids (start of the chunk)
        if constexpr (!TC) {
            for (int e = tid; e < kCKMax * ND; e += NT) cf[e] = 0.f;  // padding rows / dims stay 0
        } else {
            for (int e = tid; e < NKA * kCKMax * 8 * 2; e += NT)  // the B operands start at 0
                reinterpret_cast<float4*>(sm + L.cb)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (RED) {
            for (int e = tid; e < k * cdld; e += NT) ssum[e] = 0.0;
            for (int e = tid; e < 2 * kCKMax; e += NT) scnt[e] = 0;
        }
        if constexpr (TC) {  // the accumulators (TMEM) and the MMA-completion barrier, while the rows are in flight
            if (warp == 0) {
                const unsigned cols = umma::tmem_cols(static_cast<unsigned>(MP / 128) * 64);
                asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                             "r"(cols)
                             : "memory");
                asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
            }
            if (tid == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_mbar)) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            tc_fence_before();
        }
        __syncthreads();
        if constexpr (TC) tc_fence_after();
        // ---- Everything above is independent of the previous chunk kernel (under a
        // programmatic dependent launch it overlaps that kernel's accept); from here
        // on its results are read.  The three values its accept left, one L2 round trip:
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int go_ = __ldcg(&a.gs->go);
        const int incdeg_ = __ldcg(&a.gs->inc_degenerate);
        const unsigned long long chunk_ = __ldcg(a.chunk_ctr);
        if (!go_) {  // a chunk queued behind one that needs a repair: nothing to do
            mbar_wait(&s_xbar, 0);  // (no exit with the rows' copies in flight)
            if constexpr (TC) {
                tc_fence_before();
                __syncthreads();
                if (warp == 0) {
                    tc_fence_after();
                    const unsigned cols = umma::tmem_cols(static_cast<unsigned>(MP / 128) * 64);
                    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(cols) : "memory");
                }
            }
            return;
        }
        start_is_inc = incdeg_ == 0;
        if (tid == 0) {
            s_chunk = chunk_;  // every CTA: stable until CTA 0's accept (after a grid barrier)
            if (cta == 0 && a.timing && s_chunk < a.timing_cap) a.timing[2 * s_chunk] = t_entry;
        }
        CDBG(7, 13);
        load_centroids(0, 0);
        mbar_wait(&s_xbar, 0);
        CDBG(0, 13);
#ifdef BM_CHUNK_MMA_DIAG
        if (a.dbg_mma && a.dbg && TC) {  // diagnostics: the landed rows against global memory
            unsigned bad = 0;
            for (int e = tid; e < np * 32 * NKA; e += NT) {
                const int pp = e / (32 * NKA), d = e % (32 * NKA);
                const T want = d < n ? static_cast<const T*>(a.X)[(p0 + pp) * a.ld + d] : T(0);
                const T got = reinterpret_cast<const T*>(xchunk(pp, d / EPC))[d % EPC];
                if (!(got == want)) {
                    ++bad;
                    unsigned long long* sl = &a.dbg[(1 * 8 + 7) * 16];
                    if (cta == 0 && atomicCAS(sl, 0ull, 1ull) == 0ull) {
                        sl[1] = pp;
                        sl[2] = d;
                        sl[3] = __double_as_longlong(static_cast<double>(got));
                        sl[4] = __double_as_longlong(static_cast<double>(want));
                    }
                }
            }
            if (bad) atomicAdd(&a.dbg[(2 * 8 + 7) * 16 + 15], static_cast<unsigned long long>(bad));
            // the B operands (hi / lo parts of the compacted fp32 centroids, zero elsewhere)
            unsigned bbad = 0;
            const int KA0 = act[kCKMax];
            for (int e = tid; e < 2 * 32 * 32 * NKA; e += NT) {
                const int part = e / (32 * 32 * NKA), rem = e % (32 * 32 * NKA), rk = rem / (32 * NKA), d = rem % (32 * NKA);
                float want = 0.f;
                if (rk < KA0 && d < n) {
                    const float f = __double2float_rn(cd[rk * cdld + d]), hi = tf32_rna(f);
                    want = part ? f - hi : hi;
                }
                const size_t off = static_cast<size_t>(d >> 5) * (2 * kCKMax * 128) + rk * 128 +
                                   ((((d >> 2) & 7) ^ (rk & 7)) << 4) + (d & 3) * 4 + (part ? kCKMax * 128 : 0);
                const float got = *reinterpret_cast<const float*>(sm + L.cb + off);
                if (!(got == want)) ++bbad;
            }
            if (bbad) atomicAdd(&a.dbg[(3 * 8 + 7) * 16 + 15], static_cast<unsigned long long>(bbad));
        }
#endif
        if constexpr (TC) {
            // the MMA reads whole atoms: TMA zero-filled dims n..ND-1 and rows past
            // the chunk (rows np..MP-1 of an inner CTA hold the next CTA's rows:
            // finite, and their dot products are never read).  tf32 exactness of
            // this CTA's values unless the dataset is known to be exact
            if (!a.rows_tf32_exact) {
                const int zq = (n + 3) >> 2;  // 16-byte chunks holding data values
                for (int e = tid; e < np * zq; e += NT) {
                    const float4 v = *reinterpret_cast<const float4*>(xchunk(e / zq, e % zq));
                    xinexact |= ((__float_as_uint(v.x) | __float_as_uint(v.y) | __float_as_uint(v.z) |
                                  __float_as_uint(v.w)) & 0x1FFFu) != 0u;
                }
            }
            xinexact = __syncthreads_or(xinexact);
            fence_proxy_async_smem();
            // round 0's MMAs go out now (their operands are in place); the
            // rows' norms below are taken while they run
            if (warp == 0) issue_mma();
        }
    }
    const ScreenConsts cst = TC && xinexact ? a.cst_loose : a.cst;
    unsigned mma_phase = 0;
    // this thread's points: p = tid + i*NT; fp32 rows in registers, norms (rd/ru)
    // PPT == 2: xp[d] = (x_p0[d], x_p1[d]) (point pairs share every centroid
    // load); PPT == 1: xp[h] = (x[2h], x[2h+1]) (dimension pairs).  Norms as
    // (p0, p1) pairs (PPT == 1: both halves p0's).
    constexpr int NX = PPT == 2 ? ND : ND / 2;
    // this thread's rows, fp32, into registers (dimensions >= n read as 0).
    // Reloaded for every screen so that the registers are free in the other phases.
    auto load_xp = [&](float2 (&xp)[NX]) {
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int p = tid + i * NT;
            const int pp = p < np ? p : 0;
#pragma unroll
            for (int q = 0; q < ND / 4; ++q) {
                float v[4];
                if constexpr (sizeof(T) == 4) {
                    const float4 t = *reinterpret_cast<const float4*>(xchunk(pp, q));
                    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
                } else {
                    const double2 t0 = *reinterpret_cast<const double2*>(xchunk(pp, 2 * q));
                    const double2 t1 = *reinterpret_cast<const double2*>(xchunk(pp, 2 * q + 1));
                    v[0] = static_cast<float>(t0.x); v[1] = static_cast<float>(t0.y);
                    v[2] = static_cast<float>(t1.x); v[3] = static_cast<float>(t1.y);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int d = 4 * q + u;
                    const float x = (p < np && d < n) ? v[u] : 0.f;
                    if constexpr (PPT == 2) {
                        if (i == 0) xp[d].x = x;
                        else xp[d].y = x;
                    } else {
                        if (d & 1) xp[d >> 1].y = x;
                        else xp[d >> 1].x = x;
                    }
                }
            }
        }
    };
    float2 nxl2, nxh2, nxr2;
    int mylab[PPT];
    {
        float lo[2] = {0.f, 0.f}, hi[2] = {0.f, 0.f};
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int p = tid + i * NT;
            if (p < np) {
                if constexpr (TC) {  // 16-byte chunks of the swizzled row (padding dims are 0)
                    const unsigned char* rowb = sm + L.xs + static_cast<size_t>(p) * 128;
                    for (int q = 0; q < (n + 3) / 4; ++q) {
                        const float4 v = *reinterpret_cast<const float4*>(rowb + static_cast<size_t>(q >> 3) * ASZ +
                                                                         (((q & 7) ^ (p & 7)) << 4));
                        lo[i] = __fmaf_rd(v.x, v.x, lo[i]);
                        hi[i] = __fmaf_ru(v.x, v.x, hi[i]);
                        lo[i] = __fmaf_rd(v.y, v.y, lo[i]);
                        hi[i] = __fmaf_ru(v.y, v.y, hi[i]);
                        lo[i] = __fmaf_rd(v.z, v.z, lo[i]);
                        hi[i] = __fmaf_ru(v.z, v.z, hi[i]);
                        lo[i] = __fmaf_rd(v.w, v.w, lo[i]);
                        hi[i] = __fmaf_ru(v.w, v.w, hi[i]);
                    }
                } else {
                    for (int d = 0; d < n; ++d) {
                        const float x = static_cast<float>(xat(p, d));
                        lo[i] = __fmaf_rd(x, x, lo[i]);
                        hi[i] = __fmaf_ru(x, x, hi[i]);
                    }
                }
            }
            mylab[i] = -1;
        }
        if (PPT == 1) {
            lo[1] = lo[0];
            hi[1] = hi[0];
        }
        // rows beyond the fp32 range guarantee of the bounds: (0, inf, inf)
        const bool ok0 = hi[0] <= 1.0e36f, ok1 = hi[1] <= 1.0e36f;
        nxl2 = make_float2(ok0 ? lo[0] : 0.f, ok1 ? lo[1] : 0.f);
        nxh2 = make_float2(ok0 ? hi[0] : finf, ok1 ? hi[1] : finf);
        nxr2 = make_float2(ok0 ? __fsqrt_ru(hi[0]) : finf, ok1 ? __fsqrt_ru(hi[1]) : finf);
    }
    if (tid == 0) {
        ctl.evals = 0;
        ctl.iterations = 0;
        ctl.stop = 0;
        ctl.state_error = 0;
    }

    const uint64_t ntiles = tiles_of(a.rows);
    bool part_valid = true;  // red mode: part[cta] holds this CTA's label partials of the last assignment
    for (unsigned long long r = 0;; ++r) {
        const int rr = r < 7 ? static_cast<int>(r) : 7;
        CDBG(rr, 0);
        const int slot = static_cast<int>(r & 1);                   // distance slot
        const int rslot = RED ? static_cast<int>(r % 3) : slot;     // round sums / changed flags
        // ---- centroids: C (global) -> compacted fp64 / fp32 rows + norms ----
        // (round 0: loaded while the rows were in flight)
        if (r > 0) load_centroids(rr, r);
        const int KA = act[kCKMax];
        // (tensor core: the round's MMAs were issued in the prologue / inside load_centroids)
        __syncthreads();
        if (KA == 0) {  // assign_nearest on all-degenerate centroids (core.cpp:115-118)
            if (tid == 0) ctl.state_error = 1;
            break;
        }

        CDBG(rr, 1);
        // ---- assign: certified screen, then the candidate masks ----
        unsigned cmask[PPT];
        if constexpr (TC) {
            // dot products of this thread's points with the 32 centroid slots
            // from TMEM (tile = point / 128; this warp's lane quarter); packed
            // bounds (two points, or two centroids); candidates j with L_j <= min U
            mbar_wait_parity(&s_mbar, mma_phase);
            mma_phase ^= 1u;
            tc_fence_after();
            // one point at a time: 32 dot products in registers, bounds of
            // centroid pairs (j, j+1), then the candidates j with L_j <= min U
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                const int p = tid + i * NT;
                float Lv[32];
                {  // the dot products with hi and with lo, added (fp32, round to nearest)
                    const unsigned ta = s_tmem + (static_cast<unsigned>(32 * (warp & 3)) << 16) + 64u * static_cast<unsigned>(p >> 7);
                    float Lw[32];
                    tmem_ld32(ta, Lv);
                    tmem_ld32(ta + 32u, Lw);
#pragma unroll
                    for (int j = 0; j < 32; ++j) Lv[j] = __fadd_rn(Lv[j], Lw[j]);
                }
#ifdef BM_CHUNK_MMA_DIAG
                if (a.dbg_mma && cta == 0 && p < np) {  // diagnostics: observed MMA error / (||x|| ||c||)
                    float worst = 0.f;
                    for (int j = 0; j < KA; ++j) {
                        double ex = 0.0;
                        for (int d = 0; d < n; ++d)
                            ex += static_cast<double>(xat(p, d)) * static_cast<double>(__double2float_rn(cd[j * cdld + d]));
                        const double den = sqrt(static_cast<double>(i ? nxh2.y : nxh2.x)) * sqrt(static_cast<double>(nch[j]));
                        if (den > 0) worst = fmaxf(worst, static_cast<float>(fabs(static_cast<double>(Lv[j]) - ex) / den));
                        if (a.dbg && !(fabs(static_cast<double>(Lv[j]) - ex) <= 1e-2 * den + 1e-30)) {
                            // theories: the row the MMA result belongs to
                            auto dotq = [&](int q) {
                                double e2 = 0.0;
                                for (int d = 0; d < n; ++d)
                                    e2 += static_cast<double>(xat(q, d)) * static_cast<double>(__double2float_rn(cd[j * cdld + d]));
                                return e2;
                            };
                            const int qa = (p & ~127) + (p & 31), qb = (p & ~127) + (p & 7);
                            const bool ma = fabs(dotq(qa) - Lv[j]) <= 1e-3 * (fabs(Lv[j]) + 1.0);
                            const bool mb = fabs(dotq(qb) - Lv[j]) <= 1e-3 * (fabs(Lv[j]) + 1.0);
                            atomicAdd(&a.dbg[(1 * 8 + 5) * 16 + (ma ? 1 : 0) + (mb ? 2 : 0)], 1ull);
                            if (r == 0) atomicAdd(&a.dbg[(0 * 8 + 5) * 16 + (p >> 7)], 1ull);
                            if (r == 0) atomicAdd(&a.dbg[(0 * 8 + 5) * 16 + 8 + (p & 7)], 1ull);
                            unsigned long long* slot = &a.dbg[((s_chunk & 3ull) * 8 + 6) * 16];
                            if (atomicCAS(slot, 0ull, 1ull) == 0ull) {
                                slot[1] = static_cast<unsigned long long>(p);
                                slot[2] = static_cast<unsigned long long>(j);
                                slot[3] = static_cast<unsigned long long>(r);
                                slot[4] = __double_as_longlong(static_cast<double>(Lv[j]));
                                slot[5] = __double_as_longlong(ex);
                                slot[6] = static_cast<unsigned long long>(KA);
                                slot[7] = static_cast<unsigned long long>(np);
                                // which row's dot product did the MMA return? (first match)
                                slot[8] = 0xFFFFFFFFull;
                                for (int q = 0; q < np; ++q) {
                                    double ex2 = 0.0;
                                    for (int d = 0; d < n; ++d)
                                        ex2 += static_cast<double>(xat(q, d)) * static_cast<double>(__double2float_rn(cd[j * cdld + d]));
                                    if (fabs(ex2 - static_cast<double>(Lv[j])) <= 1e-3 * (fabs(ex2) + 1.0)) {
                                        slot[8] = static_cast<unsigned long long>(q);
                                        break;
                                    }
                                }
                                // and with which centroid of the same row?
                                slot[9] = 0xFFFFFFFFull;
                                for (int jj = 0; jj < KA; ++jj) {
                                    double ex2 = 0.0;
                                    for (int d = 0; d < n; ++d)
                                        ex2 += static_cast<double>(xat(p, d)) * static_cast<double>(__double2float_rn(cd[jj * cdld + d]));
                                    if (fabs(ex2 - static_cast<double>(Lv[j])) <= 1e-3 * (fabs(ex2) + 1.0)) {
                                        slot[9] = static_cast<unsigned long long>(jj);
                                        break;
                                    }
                                }
                                slot[10] = static_cast<unsigned long long>(__float_as_uint(Lv[(j + 1) & 31]));
                                slot[11] = static_cast<unsigned long long>(__float_as_uint(Lv[(j + 2) & 31]));
                            }
                        }
                    }
                    if (a.dbg)
                        atomicMax(reinterpret_cast<unsigned*>(&a.dbg[((s_chunk & 3ull) * 8 + 7) * 16 + 14]),
                                  __float_as_uint(worst));
                }
#endif
                const float2 nl = make_float2(i ? nxl2.y : nxl2.x, i ? nxl2.y : nxl2.x);
                const float2 nh = make_float2(i ? nxh2.y : nxh2.x, i ? nxh2.y : nxh2.x);
                const float2 nr = make_float2(i ? nxr2.y : nxr2.x, i ? nxr2.y : nxr2.x);
                float mu = finf;
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    if (j >= KA) break;
                    const bool v1 = j + 1 < KA;
                    const int j1 = v1 ? j + 1 : j;
                    float2 Lb, Ub;
                    bounds2(make_float2(Lv[j], Lv[j + 1]), nl, nh, nr, make_float2(ncl[j], ncl[j1]),
                            make_float2(nch[j], nch[j1]), make_float2(ncr[j], ncr[j1]), cst, Lb, Ub);
                    Lv[j] = Lb.x;
                    Lv[j + 1] = Lb.y;
                    mu = fminf(mu, Ub.x);
                    if (v1) mu = fminf(mu, Ub.y);
                }
                unsigned m = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < KA) m |= (Lv[j] <= mu ? 1u : 0u) << j;
                cmask[i] = p < np ? m : 0u;
            }
            tc_fence_before();  // TMEM reads done before the next round's MMAs (behind CTA barriers)
            CDBG(rr, 2);
        } else {
        // certified fp32 screen (packed FFMA)
        // groups of JG centroids (8, then 4 / 2 / 1 for the rest: no padding
        // work); per point the running minimum of the upper bounds and the
        // running candidate mask {j : L_j <= running min at j} (a superset of
        // the final candidates, filtered against the final minimum below)
        float2 xp[NX];
        load_xp(xp);
        float2 minU2 = make_float2(finf, finf);
        unsigned rm[2] = {0u, 0u};
        auto group = [&](auto jg_tag, int j0) {
            constexpr int JG = decltype(jg_tag)::value;
            float2 acc[JG];
#pragma unroll
            for (int u = 0; u < JG; ++u) acc[u] = make_float2(0.f, 0.f);
#pragma unroll
            for (int d4 = 0; d4 < ND / 4; ++d4) {
#pragma unroll
                for (int u = 0; u < JG; ++u) {
                    const float4 c = *reinterpret_cast<const float4*>(cf + (j0 + u) * ND + 4 * d4);
                    if constexpr (PPT == 2) {
                        acc[u] = ffma2s(xp[4 * d4], c.x, acc[u]);
                        acc[u] = ffma2s(xp[4 * d4 + 1], c.y, acc[u]);
                        acc[u] = ffma2s(xp[4 * d4 + 2], c.z, acc[u]);
                        acc[u] = ffma2s(xp[4 * d4 + 3], c.w, acc[u]);
                    } else {
                        acc[u] = ffma2x(xp[2 * d4], make_float2(c.x, c.y), acc[u]);
                        acc[u] = ffma2x(xp[2 * d4 + 1], make_float2(c.z, c.w), acc[u]);
                    }
                }
            }
            if constexpr (PPT == 2) {  // bounds of (p0, p1) x centroid j
#pragma unroll
                for (int u = 0; u < JG; ++u) {
                    const int j = j0 + u;
                    float2 Lb, Ub;
                    bounds2(acc[u], nxl2, nxh2, nxr2, make_float2(ncl[j], ncl[j]), make_float2(nch[j], nch[j]),
                            make_float2(ncr[j], ncr[j]), cst, Lb, Ub);
                    Ls[j * B + tid] = Lb.x;
                    Ls[j * B + tid + NT] = Lb.y;
                    minU2 = make_float2(fminf(minU2.x, Ub.x), fminf(minU2.y, Ub.y));
                    rm[0] |= (Lb.x <= minU2.x ? 1u : 0u) << j;
                    rm[1] |= (Lb.y <= minU2.y ? 1u : 0u) << j;
                }
            } else {  // bounds of p x centroids (j, j+1)
#pragma unroll
                for (int u = 0; u < JG; u += 2) {
                    const int j = j0 + u;
                    const bool v1 = u + 1 < JG;
                    const float2 dot = v1 ? add2_rn(make_float2(acc[u].x, acc[v1 ? u + 1 : u].x),
                                                    make_float2(acc[u].y, acc[v1 ? u + 1 : u].y))
                                          : make_float2(__fadd_rn(acc[u].x, acc[u].y), 0.f);
                    const int j1 = v1 ? j + 1 : j;
                    float2 Lb, Ub;
                    bounds2(dot, nxl2, nxh2, nxr2, make_float2(ncl[j], ncl[j1]), make_float2(nch[j], nch[j1]),
                            make_float2(ncr[j], ncr[j1]), cst, Lb, Ub);
                    Ls[j * B + tid] = Lb.x;
                    minU2.x = fminf(minU2.x, Ub.x);
                    rm[0] |= (Lb.x <= minU2.x ? 1u : 0u) << j;
                    if (v1) {
                        Ls[j1 * B + tid] = Lb.y;
                        minU2.x = fminf(minU2.x, Ub.y);
                        rm[0] |= (Lb.y <= minU2.x ? 1u : 0u) << j1;
                    }
                }
            }
        };
        {
            int j0 = 0;
            for (; j0 + 8 <= KA; j0 += 8) group(std::integral_constant<int, 8>{}, j0);
            if (j0 + 4 <= KA) {
                group(std::integral_constant<int, 4>{}, j0);
                j0 += 4;
            }
            if (j0 + 2 <= KA) {
                group(std::integral_constant<int, 2>{}, j0);
                j0 += 2;
            }
            if (j0 < KA) group(std::integral_constant<int, 1>{}, j0);
        }
        const float minU[2] = {minU2.x, minU2.y};
        CDBG(rr, 2);
        // ---- exact fp64 recheck of the candidates: ascending j, strict < ----
        // final candidates: the running ones whose L_j <= the final minimum;
        // every thread rechecks its own points (lanes in lock step: one
        // candidate per point is the common case)
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int p = tid + i * NT;
            unsigned m = 0, r0 = p < np ? rm[i] : 0u;
            while (r0) {
                const int j = __ffs(r0) - 1;
                r0 &= r0 - 1;
                m |= (Ls[j * B + p] <= minU[i] ? 1u : 0u) << j;
            }
            cmask[i] = m;
        }
        }
        CDBG(rr, 9);
        unsigned chg = 0;  // labels this thread's points left or joined (r > 0)
        int oldlab[PPT];   // red mode: the label a moved point left (-1: not moved)
        double mysum = 0.0;
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int p = tid + i * NT;
            oldlab[i] = -1;
            if (p >= np) continue;
            double best = dinf;
            int bj = -1;
            {
                unsigned m = cmask[i];
                while (m) {
                    const int j = __ffs(m) - 1;
                    m &= m - 1;
                    const double v = exact(p, j);
                    if (v < best) {
                        best = v;
                        bj = j;
                    }
                }
            }
            if (bj < 0) {  // no candidate (non-finite bounds): full exact scan
                for (int j = 0; j < KA; ++j) {
                    const double v = exact(p, j);
                    if (v < best) {
                        best = v;
                        bj = j;
                    }
                }
                if (bj < 0) bj = 0;  // (NaN distances only; unreachable for finite data)
            }
            const int label = act[bj];
            if (r > 0 && label != mylab[i]) {
                chg |= (1u << label) | (1u << mylab[i]);
                if constexpr (RED) oldlab[i] = mylab[i];
            }
            mylab[i] = label;
            lab[p] = label;
            dist[p] = best;
            a.dists[static_cast<size_t>(slot) * a.rows + p0 + p] = best;
            mysum += best;
        }
        int nmoved = 0;
        if constexpr (RED) {
#pragma unroll
            for (int i = 0; i < PPT; ++i) nmoved += oldlab[i] >= 0 ? 1 : 0;
        }
        __syncthreads();  // red / wsum reuse below
        // CTA sum of the distances (unordered: certified interval below)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mysum += __shfl_down_sync(0xFFFFFFFFu, mysum, o);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) chg |= __shfl_xor_sync(0xFFFFFFFFu, chg, o);
        if (RED) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nmoved += __shfl_xor_sync(0xFFFFFFFFu, nmoved, o);
        }
        if (lane == 0) {
            red[warp] = mysum;
            reinterpret_cast<unsigned*>(red + 32)[warp] = chg;
            if constexpr (RED) reinterpret_cast<int*>(red + 32)[32 + warp] = nmoved;
        }
        __syncthreads();
        // labels whose membership changed in this tile (round 0: all of them);
        // only their update partials are refolded, only they are re-merged
        unsigned dirty = 0;
        for (int w = 0; w < NW; ++w) dirty |= reinterpret_cast<const unsigned*>(red + 32)[w];
        if (r == 0) dirty = k >= 32 ? 0xFFFFFFFFu : (1u << k) - 1u;
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += red[w];
            atomicAdd(a.rsum + rslot, s);
            if (r > 0 && dirty) atomicOr(a.rchg + rslot, static_cast<int>(dirty));
        }
        // red mode: the deltas of this assignment's label sums go to dsum[r % 3]
        // — refolded labels (new partial - old partial) while this CTA's
        // partials are current and many points moved, else per moved point
        double* dcur = a.dsum + static_cast<size_t>(r % 3) * kn;
        int* ccur = a.dcnt + (r % 3) * k;
        bool refold = true;
        if (RED && r > 0) {
            int mv = 0;
            for (int w = 0; w < NW; ++w) mv += reinterpret_cast<const int*>(red + 32)[32 + w];
            refold = part_valid && mv * 8 > np;
            if (!refold) part_valid = false;
        }

        CDBG(rr, 3);
        // ---- speculative update partials of the new labels (core.cpp:200-215) ----
        if (dirty && refold) {
            const int nc = (np + 31) / 32;
            unsigned char* up = sm + L.u;
            uint16_t* members = reinterpret_cast<uint16_t*>(up);
            unsigned char* rk = up + al16(static_cast<size_t>(B) * 2);
            int* cnt = reinterpret_cast<int*>(rk + al16(static_cast<size_t>(B)));
            int* ltot = cnt + al16(static_cast<size_t>(nc) * k * 4) / 4;
            int* loff = ltot + k + 1;
            for (int e = tid; e < nc * k; e += NT) cnt[e] = 0;
            __syncthreads();
            for (int c = warp; c < nc; c += NW) {
                const int p = 32 * c + lane;
                const int l = p < np ? lab[p] : -1;
                const unsigned peers = __match_any_sync(0xFFFFFFFFu, l);
                const int rnk = __popc(peers & ((1u << lane) - 1u));
                if (p < np) {
                    rk[p] = static_cast<unsigned char>(rnk);
                    if (rnk == 0) cnt[c * k + l] = __popc(peers);
                }
            }
            __syncthreads();
            for (int j = warp; j < k; j += NW) {  // chunk-wise exclusive offsets per label
                const int v = lane < nc ? cnt[lane * k + j] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane < nc) cnt[lane * k + j] = incl - v;
                if (lane == 31) ltot[j] = incl;
            }
            __syncthreads();
            if (warp == 0) {
                const int v = lane < k ? ltot[lane] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane < k) loff[lane + 1] = incl;
                if (lane == 0) loff[0] = 0;
            }
            __syncthreads();
            for (int p = tid; p < np; p += NT) {
                const int l = lab[p];
                members[loff[l] + cnt[(p >> 5) * k + l] + rk[p]] = static_cast<uint16_t>(p);
            }
            __syncthreads();
            CDBG(rr, 12);
            // this CTA's partial of (label j, dim d) / member count of label j: stored, and in
            // red mode its change added to the round's delta buffer
            auto emit_part = [&](int j, int d, double accv) {
                double* pp = a.part + static_cast<size_t>(cta) * k * n + static_cast<size_t>(j) * n + d;
                if (RED) {  // this thread wrote *pp in the earlier rounds
                    const double dl = r > 0 ? __dsub_rn(accv, __ldcg(pp)) : accv;
                    if (dl != 0.0) atomicAdd(dcur + j * n + d, dl);
                }
                *pp = accv;
            };
            auto emit_cnt = [&](int j, int members_j) {
                unsigned* pc = a.pcnt + static_cast<size_t>(cta) * k + j;
                if (RED) {
                    const int dc = members_j - (r > 0 ? static_cast<int>(__ldcg(pc)) : 0);
                    if (dc) atomicAdd(ccur + j, dc);
                }
                *pc = static_cast<unsigned>(members_j);
            };
            // lane groups of LG lanes, one label per group, DPL dims per lane:
            // row[d] += x[d] over the label's members in index order
            // (core.cpp:206-214), member rows fetched 8 ahead of the adds
            constexpr int LG = ND <= 64 ? 16 : 32;
            constexpr int DPL = (ND + LG - 1) / LG;
            const int NG = NT / LG, g = tid / LG, gl = tid - g * LG;
            // per dimension of this lane: byte offset within a member row, and
            // (tc) its 16-byte chunk index within the swizzle atom (lanes past n
            // read a valid dimension and are never stored)
            unsigned doff[DPL];
            int dq[DPL];
#pragma unroll
            for (int t = 0; t < DPL; ++t) {
                const int d = gl + LG * t < n ? gl + LG * t : 0;
                if constexpr (TC) {
                    doff[t] = static_cast<unsigned>(L.xs + static_cast<size_t>(d >> 5) * ASZ) + (d & 3) * 4;
                    dq[t] = (d >> 2) & 7;
                } else {
                    doff[t] = static_cast<unsigned>(L.xs) + d * static_cast<unsigned>(sizeof(T));
                    dq[t] = 0;
                }
            }
            const unsigned rstride = TC ? 128u : static_cast<unsigned>(xld * sizeof(T));
            for (int j = g; j < k; j += NG) {
                if (!((dirty >> j) & 1u)) continue;  // same members as last round: same partial
                const int b = loff[j], e = loff[j + 1];
                double acc[DPL];
#pragma unroll
                for (int t = 0; t < DPL; ++t) acc[t] = 0.0;
                for (int i = b; i < e; i += 8) {
                    const int cnt8 = min(8, e - i);
                    unsigned mrow[8];
                    int msw[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int m = members[min(i + r, e - 1)];
                        mrow[r] = static_cast<unsigned>(m) * rstride;
                        msw[r] = m & 7;
                    }
                    T xv[8][DPL];
#pragma unroll
                    for (int r = 0; r < 8; ++r)
#pragma unroll
                        for (int t = 0; t < DPL; ++t)
                            xv[r][t] = *reinterpret_cast<const T*>(sm + (doff[t] + mrow[r] +
                                                                          (TC ? static_cast<unsigned>((dq[t] ^ msw[r]) << 4) : 0u)));
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (r < cnt8)
#pragma unroll
                            for (int t = 0; t < DPL; ++t) acc[t] = __dadd_rn(acc[t], to_f64(xv[r][t]));
                }
#pragma unroll
                for (int t = 0; t < DPL; ++t) {
                    const int d = gl + LG * t;
                    if (d < n) emit_part(j, d, acc[t]);
                }
                if (gl == 0) emit_cnt(j, e - b);
            }
            CDBG(rr, 14);
        }
        if (RED && !refold) {  // per moved point: + its row to the new label's sums, - to the old one's
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                unsigned bal = __ballot_sync(0xFFFFFFFFu, oldlab[i] >= 0);
                while (bal) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    const int pm = __shfl_sync(0xFFFFFFFFu, tid + i * NT, src);
                    const int ln = __shfl_sync(0xFFFFFFFFu, mylab[i], src);
                    const int lo = __shfl_sync(0xFFFFFFFFu, oldlab[i], src);
                    for (int d = lane; d < n; d += 32) {
                        const double x = to_f64(xat(pm, d));
                        if (x != 0.0) {
                            atomicAdd(dcur + ln * n + d, x);
                            atomicAdd(dcur + lo * n + d, -x);
                        }
                    }
                    if (lane == 0) {
                        atomicAdd(ccur + ln, 1);
                        atomicAdd(ccur + lo, -1);
                    }
                }
            }
        }
        const int ppc = (kn + static_cast<int>(G) - 1) / static_cast<int>(G);
        const int q0 = static_cast<int>(cta) * ppc, q1 = min(kn, q0 + ppc);
        if (RED) {  // this CTA's share of the next round's delta buffer (last read a round ago)
            double* dnx = a.dsum + static_cast<size_t>((r + 1) % 3) * kn;
            for (int q = q0 + tid; q < q1; q += NT) dnx[q] = 0.0;
            if (cta == 0 && tid < k) a.dcnt[((r + 1) % 3) * k + tid] = 0;
        }
        CDBG(rr, 4);
        grid_sync(a.bar, G);  // ---------------- barrier A ----------------
        CDBG(rr, 5);
        // this CTA's merge pairs: their tile partials and counts staged now
        // (speculatively: discarded when the loop stops), overlapping the control
        double* stage = reinterpret_cast<double*>(sm + L.u);
        unsigned* cstage = reinterpret_cast<unsigned*>(sm + L.u + al16(static_cast<size_t>(ppc) * G * 8));
        const int mj0 = q0 / n;
        if (!RED && q0 < q1) {  // part[g][q] -> stage[q - q0][g], pcnt[g][j] -> cstage[j - mj0][g]
            const int nq = q1 - q0, nj = (q1 - 1) / n - mj0 + 1;
            batched_copy<4>(
                nq * static_cast<int>(G), tid, NT,
                [&](int e) {
                    const int g = e / nq;
                    return __ldcg(a.part + static_cast<size_t>(g) * kn + q0 + (e - g * nq));
                },
                [&](int e, double v) {
                    const int g = e / nq;
                    stage[static_cast<size_t>(e - g * nq) * G + g] = v;
                });
            batched_copy<2>(
                nj * static_cast<int>(G), tid, NT,
                [&](int e) {
                    const int g = e / nj;
                    return __ldcg(a.pcnt + static_cast<size_t>(g) * k + mj0 + (e - g * nj));
                },
                [&](int e, unsigned v) {
                    const int g = e / nj;
                    cstage[static_cast<size_t>(e - g * nj) * G + g] = v;
                });
        }

        // ---- Lloyd control (local_search.cpp:26-51), every CTA identically ----
        if (tid == 0) {
            const double s = __ldcg(a.rsum + rslot);
            const int chg_all = __ldcg(a.rchg + rslot);
            ctl.gdirty = r == 0 ? 0xFFFFFFFFu : static_cast<unsigned>(chg_all);
            double lo, hi;
            sum_interval(s, a.rows, G, &lo, &hi);
            ctl.s_last = s;
            ctl.lo_last = lo;
            ctl.hi_last = hi;
            ctl.evals += a.rows * static_cast<unsigned long long>(KA);
            ctl.undecided = 0;
            if (r == 0) {  // :26-28
                ctl.f = s;
                ctl.f_lo = lo;
                ctl.f_hi = hi;
                ctl.stop = 0;
            } else {
                ctl.iterations = r;  // :36
                bool stop = chg_all == 0;  // :39-44
                if (!stop) {
                    if (ctl.f <= 0.0) {  // :45-47 (nonnegative terms: exact f is 0 iff the sum is)
                        stop = true;
                    } else if (a.rel_tolerance > 0.0) {  // :48-50 on intervals
                        const double flo = fmax(ctl.f_lo, 0x1p-1074), fhi = ctl.f_hi;
                        bool decided = !a.force_exact && isfinite(fhi) && isfinite(hi);
                        if (decided) {
                            const double a_lo = __dsub_rn(flo, hi), a_hi = __dsub_rn(fhi, lo);
                            const double g0 = __ddiv_rn(a_lo, flo), g1 = __ddiv_rn(a_lo, fhi);
                            const double g2 = __ddiv_rn(a_hi, flo), g3 = __ddiv_rn(a_hi, fhi);
                            const double gmin = fmin(fmin(g0, g1), fmin(g2, g3));
                            const double gmax = fmax(fmax(g0, g1), fmax(g2, g3));
                            if (gmax < a.rel_tolerance) stop = true;
                            else if (!(gmin >= a.rel_tolerance)) decided = false;
                        }
                        if (!decided) ctl.undecided = 1;
                    }
                }
                ctl.stop = stop ? 1 : 0;
                if (!stop && !ctl.undecided) {  // :51
                    ctl.f = s;
                    ctl.f_lo = lo;
                    ctl.f_hi = hi;
                }
            }
        }
        __syncthreads();
        if (ctl.undecided) {  // exact block sums of both assignments (grid-uniform branch)
            for (uint64_t t = static_cast<uint64_t>(cta) * NT + tid; t < 2 * ntiles; t += static_cast<uint64_t>(G) * NT) {
                const int which = t < ntiles ? 0 : 1;  // 0: previous assignment, 1: this one
                const uint64_t tt = t - which * ntiles;
                const int sl = which ? slot : slot ^ 1;
                const uint64_t tb = tt * kTile;
                const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), a.rows - tb));
                a.tiles[t] = fold_global(a.dists + static_cast<size_t>(sl) * a.rows + tb, len);
            }
            grid_sync(a.bar, G);
            if (tid == 0) {
                double f = 0.0, fn = 0.0;
                for (uint64_t t = 0; t < ntiles; ++t) f = __dadd_rn(f, __ldcg(a.tiles + t));
                for (uint64_t t = 0; t < ntiles; ++t) fn = __dadd_rn(fn, __ldcg(a.tiles + ntiles + t));
                const bool stop = __ddiv_rn(__dsub_rn(f, fn), f) < a.rel_tolerance;
                ctl.stop = stop ? 1 : 0;
                if (!stop) {
                    const double s = __ldcg(a.rsum + rslot);
                    double lo, hi;
                    sum_interval(s, a.rows, G, &lo, &hi);
                    ctl.f = s;
                    ctl.f_lo = lo;
                    ctl.f_hi = hi;
                }
            }
            __syncthreads();
        }
        if (r >= 1 && r >= a.max_iterations) {  // :32 loop bound
            if (tid == 0) ctl.stop = 1;
            __syncthreads();
        }
        if (ctl.stop) break;
        // a round slot nobody reads again before it is next added to (two
        // barriers per round: the other one; red mode: the one before this)
        if (cta == 0 && tid == 0) {
            const int zs = RED ? static_cast<int>((r + 2) % 3) : slot ^ 1;
            a.rsum[zs] = 0.0;
            a.rchg[zs] = 0;
        }
        // (red mode: the next round forms its centroids from the label sums)
        if constexpr (!RED) {

        CDBG(rr, 6);
        // ---- merge (core.cpp:217-242): this CTA's (label, dim) pairs, tile order ----
        if (q0 < q1) {
            const unsigned gdirty = ctl.gdirty;
            for (int q = q0 + tid; q < q1; q += NT) {
                const int j = q / n, d = q - j * n;
                if (!((gdirty >> j) & 1u)) continue;  // no tile changed this label: C, mask unchanged
                const double* sv = stage + static_cast<size_t>(q - q0) * G;
                const unsigned* cv = cstage + static_cast<size_t>(j - mj0) * G;
                double tot = 0.0;
                unsigned c = 0;
                unsigned g = 0;
                for (; g + 8 <= G; g += 8) {
                    double v[8];
#pragma unroll
                    for (int r8 = 0; r8 < 8; ++r8) {
                        v[r8] = sv[g + r8];
                        c += cv[g + r8];
                    }
#pragma unroll
                    for (int r8 = 0; r8 < 8; ++r8) tot = __dadd_rn(tot, v[r8]);
                }
                for (; g < G; ++g) {
                    tot = __dadd_rn(tot, sv[g]);
                    c += cv[g];
                }
                double v = 0.0;
                if (c) v = __dmul_rn(tot, __ddiv_rn(1.0, static_cast<double>(c)));  // :237-239
                a.C[q] = v;
                if (d == 0) a.mask[j] = c == 0 ? 1 : 0;
            }
        }
        CDBG(rr, 7);
        grid_sync(a.bar, G);  // ---------------- barrier B ----------------
        CDBG(rr, 8);
        }
    }

    // (a dependent launch of the next chunk kernel may start its prologue on the SMs that free up)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // every control read of this CTA is done: CTA 0 resets the round slots
    // once all CTAs are here (bar[2])
    if (tid == 0 && cta != 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + 2) : "memory");
    if (RED) {  // nobody reads a delta buffer after the last barrier: dsum[0] / dcnt[0] zero for the next launch
        const int ppc = (kn + static_cast<int>(G) - 1) / static_cast<int>(G);
        const int q0 = static_cast<int>(cta) * ppc, q1 = min(kn, q0 + ppc);
        for (int q = q0 + tid; q < q1; q += NT) a.dsum[q] = 0.0;
        if (cta == 0 && tid < k) a.dcnt[tid] = 0;
    }
    if constexpr (TC) {  // the accumulators are no longer needed
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            const unsigned cols = umma::tmem_cols(static_cast<unsigned>(MP / 128) * 64);
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(cols) : "memory");
        }
    }
    // ---- after the stop: accept (big_means.cpp:89-94), record ----
    // f_opt is exact once every earlier chunk's deferred objective is folded
    // (their k_chunk_fix ran on the side stream during this chunk); the
    // decision fc < f_opt is taken on the certified interval of the final fast
    // sum, identically in every CTA; only an undecidable interval folds the
    // exact block_sum here.  Otherwise k_chunk_fix folds it after this kernel.
    CDBG(7, 9);
    const int fslot = static_cast<int>(ctl.iterations & 1);
    if (tid == 0) {
        if (a.fix_seq)
            while (ld_acquire64(a.fix_seq) < s_chunk) {
            }
        const double fo = __ldcg(&a.gs->fopt_exact);
        ctl.fo = fo;
        if (ctl.state_error) ctl.decision = 0;
        else if (!a.force_exact && ctl.hi_last < fo) ctl.decision = 1;
        else if (!a.force_exact && !(ctl.lo_last < fo)) ctl.decision = 0;
        else ctl.decision = -1;
    }
    __syncthreads();
    __shared__ double s_fc;
    if (ctl.decision < 0 || !a.fix_seq) {  // grid-uniform: the exact objective now
        // block_sum inner folds (core.cpp:167-173) of the final distances, one
        // thread per 1024-row tile from shared memory: ordered mode folds its
        // own tile (dist[]); exact-sum mode stages tile `cta` from global first
        if (a.ordered) {
            if (tid == 0) a.tiles[cta] = fold_smem(dist, np);
        } else if (cta < ntiles) {
            // (red mode: the rows are no longer needed, their region stages the tile)
            double* stage = reinterpret_cast<double*>(sm + (RED && L.cb - L.xs >= kTile * 8 ? L.xs : L.u));
            const uint64_t tb = static_cast<uint64_t>(cta) * kTile;
            const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), a.rows - tb));
            const double* src = a.dists + static_cast<size_t>(fslot) * a.rows + tb;
            batched_copy<8>(len, tid, NT, [&](int i) { return __ldcg(src + i); },
                            [&](int i, double v) { stage[i] = v; });
            __syncthreads();
            if (tid == 0) a.tiles[cta] = fold_smem(stage, len);
        }
        CDBG(7, 10);
        grid_sync(a.bar, G);
        CDBG(7, 11);
        if (cta != 0) return;
        double* tstage = reinterpret_cast<double*>(sm + L.u);
        batched_copy<4>(static_cast<int>(ntiles), tid, NT, [&](int t) { return __ldcg(a.tiles + t); },
                        [&](int t, double v) { tstage[t] = v; });
        __syncthreads();
        if (tid == 0) {
            const double fc = fold_smem(tstage, static_cast<int>(ntiles));  // block_sum outer fold
            s_fc = fc;
            ctl.decision = !ctl.state_error && fc < ctl.fo ? 1 : 0;  // :89 strict
        }
        __syncthreads();
    } else {
        if (cta != 0) return;
        if (tid == 0) s_fc = __longlong_as_double(0x7FF8000000000000LL);  // folded by k_chunk_fix
    }
    __shared__ int s_acc;
    __shared__ unsigned char s_mk[kCKMax];
    if (tid == 0) {
        const int accepted = ctl.decision;
        const bool exact = !(s_fc != s_fc);  // s_fc is not NaN
        s_acc = accepted;
        const unsigned long long chunk = s_chunk;
        Record* rec = a.rec_base + chunk;
        rec->chunk_index = chunk;
        rec->accepted = static_cast<unsigned long long>(accepted);
        rec->degenerate_repaired = static_cast<unsigned long long>(__ldcg(&a.gs->inc_degenerate));
        if (exact) {
            rec->candidate_objective = s_fc;
            rec->incumbent_objective = accepted ? s_fc : ctl.fo;
            if (accepted) {
                *a.f_opt = s_fc;
                a.gs->fopt_exact = s_fc;
            }
        }
        if (a.job) {
            FixJob* jb = a.job;
            jb->chunk = chunk;
            jb->fo = ctl.fo;
            jb->slot = fslot;
            jb->accepted = accepted;
            jb->have_exact = exact ? 1 : 0;
            jb->valid = 1;
        }
        *a.chunk_ctr = chunk + 1;
        while (ld_acquire(a.bar + 2) < G - 1) {  // every CTA has read the round slots
        }
        a.bar[2] = 0;
        for (int z = 0; z < 3; ++z) {
            a.rsum[z] = 0.0;
            a.rchg[z] = 0;
        }
    }
    __syncthreads();
    const int accepted = s_acc;
    // incumbent := trained (accepted); next start (:82) := incumbent
    // (red mode: the trained centroids are this CTA's label sums / counts — C
    // and mask in global memory still hold the start)
    const bool own = RED && ctl.iterations >= 1;
    const bool keep = RED && !accepted && start_is_inc;  // C, mask still hold the incumbent
    const int* fcnt = scnt + (ctl.iterations & 1) * kCKMax;  // the counts behind the trained centroids
    for (int j = tid; j < k; j += NT) {
        const uint8_t mv = !accepted ? __ldcg(a.maskinc + j) : own ? (fcnt[j] > 0 ? 0 : 1) : __ldcg(a.mask + j);
        s_mk[j] = mv;
        if (accepted) a.maskinc[j] = mv;
        if ((!accepted || own) && !keep) a.mask[j] = mv;
    }
    for (int e = tid; e < k * n && !keep; e += NT) {
        if (accepted) {
            double v;
            if (own) {
                const int j = e / n;
                v = fcnt[j] > 0 ? __dmul_rn(ssum[j * cdld + (e - j * n)], sinv[j]) : 0.0;  // core.cpp:231-242
                a.C[e] = v;
            } else {
                v = __ldcg(a.C + e);
            }
            a.Cinc[e] = v;
        } else {
            a.C[e] = __ldcg(a.Cinc + e);
        }
    }
    __syncthreads();
    if (tid == 0) {
        int dcount = 0;
        for (int j = 0; j < k; ++j) dcount += s_mk[j] ? 1 : 0;
        a.gs->inc_degenerate = dcount;
        a.gs->go = dcount == 0;
        a.gs->n_active = k - dcount;
        if (accepted) a.gs->n_active_inc = k - dcount;
        a.gs->pending_fix = -1;
        LloydStatus* st = a.st;
        st->f = ctl.f;
        st->objective = s_fc;
        st->evals = ctl.evals;
        st->iterations = ctl.iterations;
        st->parity = fslot;
        st->stop = 1;
        st->changed = 0;
        st->state_error = ctl.state_error;
        st->inc_degenerate = dcount;
        st->bad_label = 0;
        st->incomplete = 0;
        if (a.host_st) {
            volatile LloydStatus* h = a.host_st;
            h->objective = s_fc;
            h->evals = ctl.evals;
            h->iterations = ctl.iterations;
            h->stop = 1;
            h->state_error = ctl.state_error;
            h->inc_degenerate = dcount;
            h->bad_label = 0;
            h->incomplete = 0;
        }
        if (a.timing && s_chunk < a.timing_cap) a.timing[2 * s_chunk + 1] = gtimer();
        CDBG(7, 12);
    }
    (void)s_any;
}

// The deferred exact objective (block_sum core.cpp:165-175) of the chunk the
// preceding k_chunk accepted or rejected: CTA t folds tile t of its final
// distances in index order; the last CTA folds the tile partials in tile
// order and completes the record (big_means.cpp:94) and, for an accepted
// chunk, f_opt (:89-93); then publishes fix_seq = chunk + 1.
__global__ void __launch_bounds__(256) k_chunk_fix(const __grid_constant__ FixArgs f) {
    __shared__ __align__(16) double stage[kTile];
    __shared__ int last;
    FixJob jb;  // written by the previous kernel on the other stream: read through L2
    jb.valid = __ldcg(&f.job->valid);
    if (!jb.valid) return;
    jb.chunk = __ldcg(&f.job->chunk);
    jb.fo = __ldcg(&f.job->fo);
    jb.slot = __ldcg(&f.job->slot);
    jb.accepted = __ldcg(&f.job->accepted);
    jb.have_exact = __ldcg(&f.job->have_exact);  // its chunk kernel found go == 0 (relaunched after the repair)
    const int tid = threadIdx.x;
    const uint64_t t = blockIdx.x, ntiles = gridDim.x;
    if (!jb.have_exact) {
        const uint64_t tb = t * kTile;
        const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), f.rows - tb));
        const double* src = f.dists + static_cast<size_t>(jb.slot) * f.rows + tb;
        batched_copy<4>(len, tid, blockDim.x, [&](int i) { return __ldcg(src + i); },
                        [&](int i, double v) { stage[i] = v; });
        __syncthreads();
        if (tid == 0) f.tiles[t] = fold_smem(stage, len);
    }
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(f.counter, 1u) == ntiles - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (!jb.have_exact) {
        batched_copy<4>(static_cast<int>(ntiles), tid, blockDim.x, [&](int i) { return __ldcg(f.tiles + i); },
                        [&](int i, double v) { stage[i] = v; });
        __syncthreads();
    }
    if (tid == 0) {
        *f.counter = 0u;
        if (!jb.have_exact) {
            const double fc = fold_smem(stage, static_cast<int>(ntiles));
            Record* rec = f.rec_base + jb.chunk;
            rec->candidate_objective = fc;
            rec->incumbent_objective = jb.accepted ? fc : jb.fo;
            if (jb.accepted) {
                *f.f_opt = fc;
                f.gs->fopt_exact = fc;
            }
        }
        f.job->valid = 0;
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f.fix_seq), "l"(jb.chunk + 1) : "memory");
    }
}

}  // namespace dev

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
namespace {

float f_ru32(double x) {
    float f = static_cast<float>(x);
    if (static_cast<double>(f) < x) f = std::nextafter(f, INFINITY);
    return f;
}
float f_rd32(double x) {
    float f = static_cast<float>(x);
    if (static_cast<double>(f) > x) f = std::nextafter(f, -INFINITY);
    return f;
}

template <typename T, int ND, int PPT, bool TC, bool RED>
void* kernel_ptr() {
    return reinterpret_cast<void*>(&dev::k_chunk<T, ND, PPT, TC, RED>);
}

// (ND, PPT) instances: ND = padded width (multiple of 8); fp32 with the
// tensor-core screen (tc) or the packed-FFMA screen, fp64 with the latter.
struct Inst {
    int nd, ppt;
    void* f32tc[2];  // [red]
    void* f32[2];
    void* f64[2];
};

#define BM_CHUNK_INST(ND, PPT)                                                                      \
    {ND, PPT,                                                                                       \
     {kernel_ptr<float, ND, PPT, true, false>(), kernel_ptr<float, ND, PPT, true, true>()},        \
     {kernel_ptr<float, ND, PPT, false, false>(), kernel_ptr<float, ND, PPT, false, true>()},      \
     {kernel_ptr<double, ND, PPT, false, false>(), kernel_ptr<double, ND, PPT, false, true>()}}
const std::vector<Inst>& instances() {
    static const std::vector<Inst> v = {
        BM_CHUNK_INST(8, 2),  BM_CHUNK_INST(16, 2), BM_CHUNK_INST(24, 2), BM_CHUNK_INST(32, 2),
        BM_CHUNK_INST(40, 1), BM_CHUNK_INST(56, 1), BM_CHUNK_INST(72, 1), BM_CHUNK_INST(88, 1),
    };
    return v;
}
#undef BM_CHUNK_INST

std::mutex g_attr_mu;

}  // namespace

dev::ScreenConsts chunk_screen_consts(int n, bool tc, bool rows_tf32_exact) {
    // |computed dot - x^.c^| <= gb ||x^|| ||c^||  (x^, c^: the fp32 rows / centroids):
    //  * packed-FFMA screen: two interleaved fp32 FMA chains added at the end,
    //    gamma_{ceil(n/2)+1}, taken as gamma_{n+2};
    //  * tensor core (tcgen05 kind::tf32, fp32 accumulate): c^ = hi + lo with
    //    hi = tf32(c^), lo exact; the MMA reads lo (and x^, unless every row
    //    value is exactly a tf32) truncated to tf32 (< 2^-10 relative), products
    //    are exact, and each of the <= 2n accumulations loses < 2^-23 of the
    //    running magnitude (<= sum |x^_d c^_d|): gb = e_x + 2^-21 + 2n 2^-23,
    //    doubled as a safety margin.
    // The rest as in engine.cu's screen_consts.
    const double u = std::ldexp(1.0, -24);
    auto gam = [&](double m) { return m * u / (1.0 - m * u); };
    // (tensor core: + 2^-24 for the fp32 sum of the hi and lo dot products, read from separate columns)
    const double gb = tc ? 2.0 * ((rows_tf32_exact ? 0.0 : std::ldexp(1.0, -10)) + std::ldexp(1.0, -21) +
                                  2.0 * n * std::ldexp(1.0, -23) + std::ldexp(1.0, -24))
                         : gam(n + 2);
    const double up = u * (1.0 + 4 * u) / (1.0 - u);
    const double K = gb / 2.0 + 2.0 * up + up * up;
    const double u64 = std::ldexp(1.0, -53);
    const double g64 = (n + 3) * u64 / (1.0 - (n + 3) * u64);
    dev::ScreenConsts c;
    c.K = f_ru32(K * (1.0 + 1e-6));
    c.dabs = std::ldexp(1.0f, -40);
    c.lo64 = f_rd32((1.0 - g64) * (1.0 - 4 * u64));
    c.hi64 = f_ru32((1.0 + g64) * (1.0 + 4 * u64));
    return c;
}

namespace {
ChunkPlan chunk_plan_spare(int device, uint64_t s, int n, int k, bm_dtype storage, bool exact_sums, bool tc, bool red,
                           int spare);
}

// Exact-sum chunks spread over the SMs: a few SMs are left to the side kernels
// (the coming chunks' draws, resolution and gather, the deferred objective) —
// on c2 131 CTAs x 384 rows instead of 143 x 352 is 5% faster per step (the
// chunk kernel's rounds wait for its slowest CTA, and a CTA that shares its SM
// with a prep kernel is slow); without a fitting plan, every SM.
// BM_CHUNK_SPARE=n overrides the number (A/B).
ChunkPlan chunk_plan(int device, uint64_t s, int n, int k, bm_dtype storage, bool exact_sums, bool tc, bool red) {
    static const int spare_env = std::getenv("BM_CHUNK_SPARE") ? std::atoi(std::getenv("BM_CHUNK_SPARE")) : -1;
    const int spare = spare_env >= 0 ? spare_env : 8;
    ChunkPlan p = chunk_plan_spare(device, s, n, k, storage, exact_sums, tc, red, exact_sums ? spare : 0);
    if (!p.ok && exact_sums && spare > 0) p = chunk_plan_spare(device, s, n, k, storage, exact_sums, tc, red, 0);
    return p;
}

namespace {
ChunkPlan chunk_plan_spare(int device, uint64_t s, int n, int k, bm_dtype storage, bool exact_sums, bool tc, bool red,
                           int spare) {
    tc = tc && storage == BM_F32;
    ChunkPlan p;
    if (k < 1 || k > dev::kCKMax || n < 1 || s < 1 || s > (1ull << 31)) return p;
    const Inst* in = nullptr;
    for (const Inst& i : instances())
        if (n <= i.nd) {
            in = &i;
            break;
        }
    if (!in) return p;
    int sms = 148, smem_optin = 227 * 1024;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const int es = storage == BM_F64 ? 8 : 4;
    // shared-memory row: whole 16-byte units, an odd number of them (conflict-free row reads)
    int units = (n * es + 15) / 16;
    if ((units & 1) == 0) ++units;
    const int xld = units * 16 / es;
    int B, threads;
    if (!exact_sums) {  // ordered: one reduction tile per CTA
        if (in->ppt != 2) return p;
        B = kTile;
        threads = kTile / 2;
    } else {  // exact sums: spread over the SMs but `spare`
        const int use = std::max(1, sms - std::max(0, spare));
        const uint64_t per = (s + use - 1) / use;
        threads = static_cast<int>(std::min<uint64_t>(dev::kCMaxT, ((per + in->ppt - 1) / in->ppt + 31) / 32 * 32));
        threads = std::max(threads, 32);
        // tensor-core screen with two points per thread: thread t's second point
        // (t + threads) must sit in the same TMEM lane quarter as its first
        if (tc && in->ppt == 2) threads = (threads + 127) / 128 * 128;
        B = threads * in->ppt;
    }
    const unsigned grid = static_cast<unsigned>((s + B - 1) / B);
    if (grid > static_cast<unsigned>(sms)) return p;  // one CTA per SM, all co-resident
    red = red && exact_sums;
    const dev::CLayout L = dev::chunk_layout(B, xld, es, k, in->nd, n, grid, tc, red);
    if (L.total + 2048 > static_cast<size_t>(smem_optin)) return p;
    // the previous chunk's k_chunk_fix must find room next to this kernel's
    // CTAs (the accept waits for it): a free SM, or room on every SM
    if (grid >= static_cast<unsigned>(sms) && (threads > 384 || L.total > 216 * 1024)) return p;
    p.ok = true;
    p.tc = tc;
    p.B = B;
    p.threads = threads;
    p.ppt = in->ppt;
    p.nd = in->nd;
    p.xld = xld;
    p.ordered = exact_sums ? 0 : 1;
    p.red = red ? 1 : 0;
    p.grid = grid;
    p.smem = L.total;
    return p;
}
}  // namespace

CUtensorMap chunk_rows_map(const ChunkPlan& p, bm_dtype storage, const void* X, uint64_t rows, int n, uint64_t ld) {
    CUtensorMap m{};
    auto enc = tmap_encoder();
    if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
    const size_t es = storage == BM_F64 ? 8 : 4;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
    const cuuint32_t box[2] = {p.tc ? 32u : (cuuint32_t)p.xld, p.tc ? 128u : (cuuint32_t)dev::chunk_box_rows(p.B)};
    const cuuint32_t estr[2] = {1, 1};
    const auto dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const auto sw = p.tc ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (enc(&m, dt, 2, const_cast<void*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(chunk rows) failed");
    return m;
}

void chunk_fix_prefer_max_smem() {
    BM_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(dev::k_chunk_fix),
                                 cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
}

void launch_chunk_fix(cudaStream_t st, const dev::FixArgs& f) {
    const unsigned tiles = static_cast<unsigned>(tiles_of(f.rows));
    dev::k_chunk_fix<<<tiles, 256, 0, st>>>(f);
    BM_CUDA(cudaGetLastError());
}

void launch_chunk(cudaStream_t st, const ChunkPlan& p, bm_dtype storage, const dev::ChunkArgs& a0) {
    void* fn = nullptr;
    for (const Inst& i : instances())
        if (i.nd == p.nd && i.ppt == p.ppt)
            fn = storage == BM_F64 ? i.f64[p.red ? 1 : 0] : p.tc ? i.f32tc[p.red ? 1 : 0] : i.f32[p.red ? 1 : 0];
    if (!fn) throw CudaError("chunk kernel: no instance");
    {
        // the attribute is a per-device maximum: raise it, never lower it
        static std::map<std::pair<int, void*>, size_t> cur;
        int dev = 0;
        BM_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_attr_mu);
        size_t& c = cur[std::make_pair(dev, fn)];
        if (p.smem > c) {
            BM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)));
            c = p.smem;
        }
    }
    dev::ChunkArgs a = a0;
    a.B = p.B;
    a.xld = p.xld;
    a.ordered = p.ordered;
    a.red = p.red;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    static const bool own_sm = std::getenv("BM_CHUNK_OWN_SM") && std::string(std::getenv("BM_CHUNK_OWN_SM")) == "1";
    a.threads = p.threads;
    cfg.blockDim = dim3(own_sm ? dev::kCMaxT : p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    // BM_CHUNK_PDL=1: plain launch with programmatic stream serialization (the next
    // chunk kernel's prologue overlaps this one's accept); BM_CHUNK_COOP=0: plain launch
    static const bool pdl = std::getenv("BM_CHUNK_PDL") && std::string(std::getenv("BM_CHUNK_PDL")) == "1";
    static const bool coop = !pdl && !(std::getenv("BM_CHUNK_COOP") && std::string(std::getenv("BM_CHUNK_COOP")) == "0");
    if (pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.numAttrs = coop || pdl ? 1 : 0;
    void* args[] = {&a};
    BM_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace bm
