// kernels_assign.cuh — nearest-centroid assignment: exact, certified-screen (TMA ring) and the streaming final pass; exact-sum label sums.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

// ===========================================================================
// 3. Exact nearest-centroid assignment (assign_nearest core.cpp:106-161).
//
// CTA = 128 points x all active centroids.  Thread (pg, cg) owns points
// {pg + 32 t : t < 4} and compacted centroids {4 cg + u : u < 4}: 16
// independent fp64 chains, each a strict left fold over d (P1).  Points and
// centroids are staged through shared memory in 16-dim slabs, transposed so
// that the point loads are conflict-free and the centroid loads broadcast.
// Centroids are the COMPACTED active rows in ascending original index, so an
// ascending strict-< scan over them is the reference's masked j-loop (P2).
// ===========================================================================
constexpr int kAP = 4;            // points per thread
constexpr int kAK = 4;            // centroids per thread
constexpr int kAPG = 32;          // point groups (= lanes) per CTA
constexpr int kABP = kAP * kAPG;  // 128 points per CTA
constexpr int kADC = 16;          // dims per shared-memory slab
constexpr int kAMaxCG = 8;        // centroid groups per CTA (<= 32 centroids per pass)
constexpr int kAXS = kABP + 1;    // padded slab stride

template <typename T>
__global__ void __launch_bounds__(kAPG * kAMaxCG)
k_assign(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
         const double* __restrict__ Cact, int ldc, const int* __restrict__ act_idx,
         const int* __restrict__ n_active_ptr,
         int32_t* __restrict__ labels_pair, uint64_t pair_stride, const int* __restrict__ parity_ptr,
         double* __restrict__ dists_out, int* __restrict__ changed_flag,
         const int* __restrict__ stop_ptr) {
    __shared__ double xs[kADC * kAXS];
    __shared__ double cs[kADC * kAMaxCG * kAK];
    __shared__ double red_d[kAMaxCG][kABP];
    __shared__ int red_j[kAMaxCG][kABP];
    __shared__ double best_d[kABP];
    __shared__ int best_j[kABP];

    if (stop_ptr && *stop_ptr) return;  // Lloyd loop already finished
    const int KA = *n_active_ptr;
    // Lloyd mode: write labels[1-parity], compare with labels[parity] (:34,:39).
    int32_t* labels_out = labels_pair;
    const int32_t* labels_old = nullptr;
    if (parity_ptr) {
        const int par = *parity_ptr;
        labels_out = labels_pair + (1 - par) * pair_stride;
        labels_old = labels_pair + par * pair_stride;
    }
    const int KG = blockDim.x / kAPG;
    const int KB = KG * kAK;  // centroids per pass
    const int tid = threadIdx.x, pg = tid % kAPG, cg = tid / kAPG;
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * kABP;

    for (int p = tid; p < kABP; p += blockDim.x) {
        best_d[p] = __longlong_as_double(0x7FF0000000000000LL);  // +inf
        best_j[p] = -1;
    }
    for (int kb = 0; kb < KA; kb += KB) {
        double acc[kAP][kAK];
#pragma unroll
        for (int t = 0; t < kAP; ++t)
#pragma unroll
            for (int u = 0; u < kAK; ++u) acc[t][u] = 0.0;

        for (int d0 = 0; d0 < n; d0 += kADC) {
            const int dl = min(kADC, n - d0);
            __syncthreads();
            for (int e = tid; e < kABP * kADC; e += blockDim.x) {
                const int p = e / kADC, d = e % kADC;
                const uint64_t gp = p0 + p;
                double v = 0.0;
                if (gp < rows && d < dl) v = to_f64(X[gp * ld + d0 + d]);
                xs[d * kAXS + p] = v;
            }
            for (int e = tid; e < KB * kADC; e += blockDim.x) {
                const int j = e / kADC, d = e % kADC;
                double v = 0.0;
                if (kb + j < KA && d < dl) v = Cact[static_cast<uint64_t>(kb + j) * ldc + d0 + d];
                cs[d * KB + j] = v;
            }
            __syncthreads();
            for (int d = 0; d < dl; ++d) {
                double xv[kAP], cv[kAK];
#pragma unroll
                for (int t = 0; t < kAP; ++t) xv[t] = xs[d * kAXS + pg + kAPG * t];
#pragma unroll
                for (int u = 0; u < kAK; ++u) cv[u] = cs[d * KB + cg * kAK + u];
#pragma unroll
                for (int t = 0; t < kAP; ++t)
#pragma unroll
                    for (int u = 0; u < kAK; ++u) acc[t][u] = dist_step(acc[t][u], xv[t], cv[u]);
            }
        }
        // Ascending strict-< within the thread's 4 centroids ...
#pragma unroll
        for (int t = 0; t < kAP; ++t) {
            double b = __longlong_as_double(0x7FF0000000000000LL);
            int bj = -1;
#pragma unroll
            for (int u = 0; u < kAK; ++u) {
                const int j = kb + cg * kAK + u;
                if (j < KA && acc[t][u] < b) {
                    b = acc[t][u];
                    bj = j;
                }
            }
            red_d[cg][pg + kAPG * t] = b;
            red_j[cg][pg + kAPG * t] = bj;
        }
        __syncthreads();
        // ... then across centroid groups in ascending order (first minimum wins).
        for (int p = tid; p < kABP; p += blockDim.x) {
            double b = best_d[p];
            int bj = best_j[p];
            for (int g = 0; g < KG; ++g) {
                if (red_j[g][p] >= 0 && red_d[g][p] < b) {
                    b = red_d[g][p];
                    bj = red_j[g][p];
                }
            }
            best_d[p] = b;
            best_j[p] = bj;
        }
        __syncthreads();
    }
    for (int p = tid; p < kABP; p += blockDim.x) {
        const uint64_t gp = p0 + p;
        if (gp < rows) {
            const int bj = best_j[p];
            const int label = bj >= 0 ? act_idx[bj] : -1;
            labels_out[gp] = label;
            if (dists_out) dists_out[gp] = best_d[p];
            if (labels_old && labels_old[gp] != label) *changed_flag = 1;
        }
    }
}

// ===========================================================================
// 3b. Screened exact assignment (same results as k_assign, bit for bit).
//
// Screen (fp32, norm form).  With x^ = fl32(x), c^ = fl32(c), the dot product
// s = sum_d x^_d c^_d is accumulated with packed FFMA2 in 16-dim blocks that
// are then added up (error <= g_b ||x^|| ||c^||, g_b = g_16 + g_S(1+g_16)),
// and ||x^||^2, ||c^||^2 are accumulated with rounding down and up.  Writing
// S = ||x^||+||c^|| (upper bound), the reference's fp64 value d_ref
// (core.cpp:142-146) is certified to lie in [L, U]:
//   r^2 in [ nx_lo + nc_lo - 2s - K S^2 , nx_hi + nc_hi - 2s + K S^2 ]
//   K = g_b/2 + 2u' + u'^2,  u' = u(1+4u)/(1-u)   (input rounding to fp32,
//       via (r^ +- w)^2 with w <= u' S and r^ <= S)
//   d_ref in [ r^2 (1-g64), r^2 (1+g64) ],  g64 = gamma_{n+3} (fp64 rounding)
// evaluated with directed-rounding fp32 ops.  Every centroid whose L exceeds
// the point's smallest U can be neither the reference's minimum nor tie it;
// the remaining candidates are recomputed exactly in fp64 (direct form,
// ascending j, strict <), which reproduces assign_nearest exactly.  Inputs or
// intermediates beyond fp32 range force L = 0, U = inf (exact fallback).
//
// Fused per-1024-point tile sums (block_sum inner loop core.cpp:167-173): the
// last CTA to finish a tile folds the tile's distances in index order.
// ===========================================================================
constexpr int kFailMax = 24;      // Lloyd-round bound failures handled per point
constexpr int kSThreads = 256;    // 8 warps: warp w < KG owns centroids 4w..4w+3
constexpr int kSXS = kABP + 4;    // fp32 slab stride (16-byte aligned rows)
constexpr int kItemCap = 4 * kABP;  // (point, candidate) items per CTA (2 per thread)



// ---------------------------------------------------------------------------
// 3c. Screened exact assignment, TMA pipeline (v5).  Same mathematics and
// results as the direct screen (3b); only the data movement differs:
//  * one thread issues 2-D TMA tile loads (128 points x 16 dims, hardware
//    swizzle) of the points and of the fp32 transposed centroids (CT32[d][j])
//    into a 2-stage ring, completion on one mbarrier per stage;
//  * all threads convert the landed raw slab once (f64 -> fp32, round to
//    nearest) into a double-buffered [d][p] fp32 slab, ONE CTA barrier per
//    slab, after which the stage is refilled with slab+2 while the screen of
//    the current slab runs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_el(void* smem, const void* gmem, int bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <typename T, int NS = 2>
struct TmaSmem {
    static constexpr int kRawBytes = kABP * kADC * sizeof(T);  // 16 KB (f64) / 8 KB (f32)
    alignas(1024) unsigned char raw[NS][kRawBytes];            // swizzled point tiles (NS-stage ring)
    alignas(1024) float craw[NS][kADC][kSMaxK];                // centroid tiles [d][j]
    alignas(16) float xs[2][kADC][kABP];                       // fp32 point slabs [d][p]
    alignas(16) float cs[2][kADC][kSMaxK];
    float red_u[8][kABP];                                      // per-warp min upper bound
    float nx_lo[kABP], nx_hi[kABP], nxr[kABP];
    float nc_lo[kSMaxK], nc_hi[kSMaxK], ncr[kSMaxK];
    unsigned cand[kABP];                                       // candidate bitmask per point
    int icount[kABP];
    int lab_rank[kABP];                                        // chosen compacted centroid per point
    int lab_new[kABP], lab_old[kABP];                          // exact-sum mode: this launch's label change per point
    int rank_of[kSMaxK];                                       // label -> compacted index
    float delta[kSMaxK];                                       // centroid movement per label (rounded up)
    alignas(16) float lbs[sizeof(T) == 4 ? kABP : 1][kSMaxK];  // fp32 round fast path: the bound rows (16-byte chunks swizzled)
    uint64_t bar[NS];
    uint32_t n_items;
    int is_last;
};

// ---------------------------------------------------------------------------
// 5b. Exact-sum mode.  When every stored value is an integer multiple of 2^e
// and m * max|x| < 2^53 * 2^e (checked once per dataset, bm_dataset_create),
// every partial sum of any subset of the values of one dimension is exactly
// representable in fp64: the reference's ordered sums (per-tile folds in index
// order, tile merge in order, core.cpp:206-229) then equal the exact sums,
// whatever the order.  The label sums are kept as integers (x * 2^-e) per
// chunk buffer: a begin adds every point, a Lloyd round moves only the points
// whose label changed, and k_centroids turns them into the next centroids
// (sum * (1.0/count), core.cpp:237-239) — no ordered update pass at all.
// ---------------------------------------------------------------------------
constexpr int kSumCopies = 8;  // CTA b adds into copy b % 8 (spreads same-address atomics)
#ifndef BM_SUM_GROUP
#define BM_SUM_GROUP 8
#endif
constexpr int kSumGroup = BM_SUM_GROUP;  // a begin's CTAs whose partial sums one of them merges
static_assert(kSumGroup >= 1 && kSumGroup <= 32, "BM_SUM_GROUP must be in [1, 32]");

__device__ __forceinline__ long long sum_units(double x, double scale) {
    return __double2ll_rn(__dmul_rn(x, scale));  // exact: x * 2^-e is an integer below 2^53
}

template <typename T, int NS>
__device__ __noinline__ void label_sums(TmaSmem<T, NS>& S, const LloydCtl& ctl, const T* __restrict__ X, uint64_t ld,
                                        int n, uint64_t p0, int np, bool full, int kfull, unsigned char* scratch,
                                        size_t scratch_bytes, unsigned blk, const float* pre) {
    __syncthreads();  // every point's (new, old) label recorded; the scratch area is free
    const int tid = threadIdx.x;
    const int which = ctl.sum_which >= 0 ? ctl.sum_which : ctl.st->sum_sel;
    // this CTA's copy: [kSumCopies][kSMaxK][n] sums, then [kSumCopies][kSMaxK] counts
    // (a begin spreads its atomics over the copies, which its control CTA then
    // folds into copy 0; a round's few moves go to copy 0 directly)
    const int cp = full ? static_cast<int>(blk % kSumCopies) : 0;
    long long* half = ctl.sums + static_cast<uint64_t>(which) * ctl.sum_half;
    long long* sg = half + static_cast<uint64_t>(cp) * kSMaxK * n;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n +
                                                                    cp * kSMaxK);
    // Per label, the points that join it (+x) and the points that leave it (-x)
    // (a begin: every point joins its label), bucketed by a counting sort; then
    // one thread per (label, dim) sums its members' coordinates.  The partial
    // sums are exact in fp64 (§5b: multiples of 2^e below 2^52 * 2^e), so the
    // order is free.
    // (the lists live in red_u, free until the control tail; the moved rows are
    // staged in the scratch area when they fit)
    int* pc = reinterpret_cast<int*>(&S.red_u[0][0]);  // [kSMaxK + 1] join offsets
    int* mc = pc + (kSMaxK + 1);                 // [kSMaxK + 1] leave offsets
    int* pcur = mc + (kSMaxK + 1);               // [kSMaxK] cursors
    int* mcur = pcur + kSMaxK;                   // [kSMaxK]
    short* plist = reinterpret_cast<short*>(mcur + kSMaxK);  // [kABP]
    short* mlist = plist + kABP;                             // [kABP]
    int* flag = reinterpret_cast<int*>(mlist + kABP);        // [2]: any move, group leader
    if (tid < kSMaxK) {
        pcur[tid] = 0;
        mcur[tid] = 0;
    }
    if (tid == 0) flag[0] = 0;
    __syncthreads();
    int a = -1, b = -1;
    int* rslot = flag + 2;  // [kABP] staged row of each moved point
    if (tid == 0) flag[1] = 0;
    __syncthreads();
    if (tid < np) {
        a = full ? -1 : S.lab_old[tid];
        b = S.lab_new[tid];
        if (a == b) a = b = -1;
        if (b >= 0) atomicAdd(&pcur[b], 1);
        if (a >= 0) atomicAdd(&mcur[a], 1);
        if (b >= 0 || a >= 0) rslot[tid] = atomicAdd(&flag[1], 1);
    }
    __syncthreads();
    const int nm = flag[1];
    if (nm == 0) return;  // nothing moved in this CTA
    // stage the moved rows (whole 16-byte vectors) with cp.async
    constexpr int kV = 16 / sizeof(T);
    const int vpr = static_cast<int>((n + kV - 1) / kV);
    // pre: every row of the block already in shared memory (the full screen's
    // staged fp32 rows, [p][ld]); else the moved rows are staged here
    const bool staged = !pre && (ld % kV) == 0 && static_cast<size_t>(nm) * vpr * 16 <= scratch_bytes;
    T* xs = reinterpret_cast<T*>(scratch);
    if (staged) {
        for (int e = tid; e < np * vpr; e += blockDim.x) {
            const int p = e / vpr, v = e - p * vpr;
            const int la = full ? -1 : S.lab_old[p], lb = S.lab_new[p];
            if (la != lb && (la >= 0 || lb >= 0))
                cp_async_16(xs + static_cast<size_t>(rslot[p]) * vpr * kV + v * kV, X + (p0 + p) * ld + v * kV);
        }
        cp_async_commit();
    }
    if (tid < 32) {  // exclusive scans of the join / leave counts (k <= 32)
        const int lane = tid;
        const int vp = pcur[lane], vm = mcur[lane];
        int ip = vp, im = vm;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yp = __shfl_up_sync(0xFFFFFFFFu, ip, o), ym = __shfl_up_sync(0xFFFFFFFFu, im, o);
            if (lane >= o) {
                ip += yp;
                im += ym;
            }
        }
        pc[lane] = ip - vp;
        mc[lane] = im - vm;
        if (lane == 31) {
            pc[32] = ip;
            mc[32] = im;
        }
        pcur[lane] = ip - vp;
        mcur[lane] = im - vm;
    }
    __syncthreads();
    if (b >= 0) plist[atomicAdd(&pcur[b], 1)] = static_cast<short>(staged ? rslot[tid] : tid);
    if (a >= 0) mlist[atomicAdd(&mcur[a], 1)] = static_cast<short>(staged ? rslot[tid] : tid);
    if (staged) cp_async_wait<0>();
    __syncthreads();
    const double sc = ctl.sum_scale;
    const bool grouped = full && ctl.parts;
    const uint64_t slot_len = static_cast<uint64_t>(kSMaxK) * n + kSMaxK;
    long long* slot = grouped ? ctl.parts + blk * slot_len : nullptr;
    const T* Xb = pre ? reinterpret_cast<const T*>(pre) : staged ? xs : X + p0 * ld;
    const uint64_t rs = staged ? static_cast<uint64_t>(vpr) * kV : ld;  // row stride of Xb
    for (int e = tid; e < kfull * n; e += blockDim.x) {
        const int j = e / n, d = e - j * n;
        double s = 0.0;
        int q = pc[j];
        const int q1 = pc[j + 1];
        for (; q + 4 <= q1; q += 4) {
            const double x0 = to_f64(Xb[plist[q] * rs + d]), x1 = to_f64(Xb[plist[q + 1] * rs + d]);
            const double x2 = to_f64(Xb[plist[q + 2] * rs + d]), x3 = to_f64(Xb[plist[q + 3] * rs + d]);
            s = __dadd_rn(__dadd_rn(s, x0), __dadd_rn(__dadd_rn(x1, x2), x3));
        }
        for (; q < q1; ++q) s = __dadd_rn(s, to_f64(Xb[plist[q] * rs + d]));
        for (int r = mc[j]; r < mc[j + 1]; ++r) s = __dsub_rn(s, to_f64(Xb[mlist[r] * rs + d]));
        const long long v = sum_units(s, sc);
        if (grouped) slot[e] = v;
        else if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&sg[e]), static_cast<unsigned long long>(v));
    }
    if (!grouped) {
        if (tid < kfull) {
            const long long c = (pc[tid + 1] - pc[tid]) - (mc[tid + 1] - mc[tid]);
            if (c != 0) atomicAdd(&cnt[tid], static_cast<unsigned long long>(c));
        }
        __threadfence();  // this CTA's atomics before its arrival
        return;
    }
    // A begin: the partials of kSumGroup CTAs are merged by the last of them (fewer
    // global atomics, which are the bottleneck at this volume).
    if (tid < kfull) slot[static_cast<uint64_t>(kSMaxK) * n + tid] = pc[tid + 1] - pc[tid];
    __threadfence();
    __syncthreads();
    const int g = static_cast<int>(blk / kSumGroup);
    const int pts_ctas = static_cast<int>((ctl.pts_rows + kABP - 1) / kABP);
    const int members = min(kSumGroup, pts_ctas - kSumGroup * g);
    if (tid == 0) flag[1] = atomicAdd(&ctl.grp_ctr[g], 1u) == static_cast<unsigned>(members) - 1;
    __syncthreads();
    if (!flag[1]) return;
    __threadfence();
    long long* gsg = half + static_cast<uint64_t>(g % kSumCopies) * kSMaxK * n;
    unsigned long long* gcnt = reinterpret_cast<unsigned long long*>(
        half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n + (g % kSumCopies) * kSMaxK);
    const long long* gbase = ctl.parts + static_cast<uint64_t>(kSumGroup) * g * slot_len;
    const int kn = kfull * n;
    for (int e = tid; e < kn + kfull; e += blockDim.x) {
        const bool is_cnt = e >= kn;
        const uint64_t off = is_cnt ? static_cast<uint64_t>(kSMaxK) * n + (e - kn) : static_cast<uint64_t>(e);
        long long v = 0;
#pragma unroll
        for (int m = 0; m < kSumGroup; ++m)
            if (m < members) v += __ldcg(gbase + m * slot_len + off);
        if (v != 0) {
            if (is_cnt) atomicAdd(&gcnt[e - kn], static_cast<unsigned long long>(v));
            else atomicAdd(reinterpret_cast<unsigned long long*>(&gsg[off]), static_cast<unsigned long long>(v));
        }
    }
    if (tid == 0) ctl.grp_ctr[g] = 0u;
    __threadfence();  // this CTA's atomics before its arrival (the control CTA folds the copies)
}

// Exact-sum mode update (update_centroids core.cpp:183-244 via §5b): the
// label sums kept by the assignments give sum * (1.0/count) per (label, dim)
// (:237-239), count 0 a degenerate row of 0.0; plus everything k_update's
// merge writes (mask, active list, Cact, CT32, per-label movement).  CTA-wide
// (any whole number of warps), a warp per label; tot / rank: shared scratch.
__device__ __noinline__ void centroids_from_sums(const long long* __restrict__ half, int k, int n, double unscale,
                                                 double* __restrict__ C, uint8_t* __restrict__ mask,
                                                 double* __restrict__ Cact, int ldc, int* __restrict__ act_idx,
                                                 int* __restrict__ n_active, float* __restrict__ CT32,
                                                 float* __restrict__ delta, long long* tot, int* rank) {
    const long long* cnts = half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        long long c = 0;
        if (lane < k) c = __ldcg(cnts + lane);  // copy 0 (the begin's control CTA folded the others into it)
        const unsigned live = __ballot_sync(0xFFFFFFFFu, c > 0);
        if (lane < k) {
            tot[lane] = c;
            const int r = __popc(live & ((1u << lane) - 1u));
            rank[lane] = c > 0 ? r : -1;
            mask[lane] = c > 0 ? 0 : 1;
            if (c > 0) act_idx[r] = lane;
        }
        if (lane == 0) *n_active = __popc(live);
    }
    __syncthreads();
    for (int j = warp; j < k; j += blockDim.x / 32) {
        const long long c = tot[j];
        const uint64_t row = static_cast<uint64_t>(j) * n;
        if (c <= 0) {
            for (int d = lane; d < n; d += 32) C[row + d] = 0.0;
            continue;
        }
        const double inv = __ddiv_rn(1.0, static_cast<double>(c));
        const int rk = rank[j];
        double sq = 0.0;
        for (int d = lane; d < n; d += 32) {
            const long long s = __ldcg(half + row + d);  // copy 0
            const double sum = __dmul_rn(static_cast<double>(s), unscale);  // exact (§5b)
            const double v = __dmul_rn(sum, inv);
            const double dv = __dsub_rn(v, C[row + d]);
            sq = __dadd_rn(sq, __dmul_rn(dv, dv));  // order-free: only bounds use it
            C[row + d] = v;
            Cact[static_cast<uint64_t>(rk) * ldc + d] = v;
            if (CT32) CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
        if (lane == 0) delta[j] = __double2float_ru(__dsqrt_ru(sq * (1.0 + 1e-12)) * (1.0 + 1e-12) + 1e-300);
    }
}

// The same for one label j per CTA (many CTAs in parallel: the begin that
// finds the speculative one current): every CTA ranks the labels from the
// counts; CTA 0 also writes the mask, the active list and their count.
__device__ __noinline__ void centroid_of_label(const long long* __restrict__ half, int k, int n, double unscale,
                                               double* __restrict__ C, uint8_t* __restrict__ mask,
                                               double* __restrict__ Cact, int ldc, int* __restrict__ act_idx,
                                               int* __restrict__ n_active, float* __restrict__ CT32,
                                               float* __restrict__ delta, int j, double* red) {
    const long long* cnts = half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ long long cj;
    __shared__ int rj;
    if (warp == 0) {
        const long long c = lane < k ? __ldcg(cnts + lane) : 0;
        const unsigned live = __ballot_sync(0xFFFFFFFFu, c > 0);
        const int r = __popc(live & ((1u << lane) - 1u));
        if (lane == j) {
            cj = c;
            rj = c > 0 ? r : -1;
        }
        if (blockIdx.x == 0 && lane < k) {
            mask[lane] = c > 0 ? 0 : 1;
            if (c > 0) act_idx[r] = lane;
            if (lane == 0) *n_active = __popc(live);
        }
    }
    __syncthreads();
    const long long c = cj;
    const uint64_t row = static_cast<uint64_t>(j) * n;
    if (c <= 0) {
        for (int d = tid; d < n; d += blockDim.x) C[row + d] = 0.0;
        return;
    }
    const double inv = __ddiv_rn(1.0, static_cast<double>(c));
    const int rk = rj;
    double sq = 0.0;
    for (int d = tid; d < n; d += blockDim.x) {
        const long long sv = __ldcg(half + row + d);  // copy 0
        const double sum = __dmul_rn(static_cast<double>(sv), unscale);  // exact (§5b)
        const double v = __dmul_rn(sum, inv);
        const double dv = __dsub_rn(v, C[row + d]);
        sq = __dadd_rn(sq, __dmul_rn(dv, dv));  // order-free: only bounds use it
        C[row + d] = v;
        Cact[static_cast<uint64_t>(rk) * ldc + d] = v;
        if (CT32) CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        delta[j] = __double2float_ru(__dsqrt_ru(t * (1.0 + 1e-12)) * (1.0 + 1e-12) + 1e-300);
    }
}

// A begin's control CTA: copies 1..7 of the half folded into copy 0 and zeroed
// (CTA-wide; exact integer adds), so later readers touch one copy.
__device__ __noinline__ void fold_sum_copies(long long* half, int k, int n) {
    const uint64_t span = static_cast<uint64_t>(kSMaxK) * n;
    long long* cnts = half + static_cast<uint64_t>(kSumCopies) * span;
    const int kn = k * n;
    for (int e = threadIdx.x; e < kn + k; e += blockDim.x) {
        const bool is_cnt = e >= kn;
        long long* base = is_cnt ? cnts + (e - kn) : half + e;
        const uint64_t stride = is_cnt ? static_cast<uint64_t>(kSMaxK) : span;
        long long v = __ldcg(base);
#pragma unroll
        for (int q = 1; q < kSumCopies; ++q) v += __ldcg(base + q * stride);
        *base = v;
#pragma unroll
        for (int q = 1; q < kSumCopies; ++q) base[q * stride] = 0;
    }
    __threadfence();
    __syncthreads();
}

// The same, element-parallel (the control CTA of a round that goes on): every
// thread's sums and old centroids loaded up front, the squared movements
// through shared memory (dsq: k * n doubles), then a warp per label.
__device__ __noinline__ void centroids_from_sums_ilp(const long long* __restrict__ half, int k, int n, double unscale,
                                                     double* __restrict__ C, uint8_t* __restrict__ mask,
                                                     double* __restrict__ Cact, int ldc, int* __restrict__ act_idx,
                                                     int* __restrict__ n_active, float* __restrict__ CT32,
                                                     float* __restrict__ delta, long long* tot, int* rank,
                                                     double* dsq) {
    const long long* cnts = half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n;
    __shared__ double inv_s[kSMaxK];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nth = blockDim.x;
    if (warp == 0) {
        long long c = 0;
        if (lane < k) c = __ldcg(cnts + lane);  // copy 0
        const unsigned live = __ballot_sync(0xFFFFFFFFu, c > 0);
        if (lane < k) {
            tot[lane] = c;
            const int r = __popc(live & ((1u << lane) - 1u));
            rank[lane] = c > 0 ? r : -1;
            mask[lane] = c > 0 ? 0 : 1;
            if (c > 0) act_idx[r] = lane;
            inv_s[lane] = c > 0 ? __ddiv_rn(1.0, static_cast<double>(c)) : 0.0;
        }
        if (lane == 0) *n_active = __popc(live);
    }
    __syncthreads();
    const int kn = k * n;
    constexpr int kU = 4;
    for (int e0 = tid; e0 < kn; e0 += kU * nth) {
        long long sv[kU];
        double cv[kU];
#pragma unroll
        for (int r = 0; r < kU; ++r) {
            const int e = e0 + r * nth;
            if (e < kn) {
                sv[r] = __ldcg(half + e);
                cv[r] = C[e];
            }
        }
#pragma unroll
        for (int r = 0; r < kU; ++r) {
            const int e = e0 + r * nth;
            if (e >= kn) continue;
            const int j = e / n, d = e - j * n;
            if (tot[j] <= 0) {
                C[e] = 0.0;
                dsq[e] = 0.0;
                continue;
            }
            const double v = __dmul_rn(__dmul_rn(static_cast<double>(sv[r]), unscale), inv_s[j]);  // exact sum (§5b)
            const double dv = __dsub_rn(v, cv[r]);
            dsq[e] = __dmul_rn(dv, dv);
            C[e] = v;
            const int rk = rank[j];
            Cact[static_cast<uint64_t>(rk) * ldc + d] = v;
            if (CT32) CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v);
        }
    }
    __syncthreads();
    for (int j = warp; j < k; j += nth / 32) {
        if (tot[j] <= 0) continue;
        double sq = 0.0;
        for (int d = lane; d < n; d += 32) sq = __dadd_rn(sq, dsq[j * n + d]);  // order-free: only bounds use it
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
        if (lane == 0) delta[j] = __double2float_ru(__dsqrt_ru(sq * (1.0 + 1e-12)) * (1.0 + 1e-12) + 1e-300);
    }
}

// The fused form (LloydCtl::sum_fuse): the live half of this chunk buffer's sums.
__device__ __forceinline__ void centroids_fused(const LloydCtl& c, int sum_sel, int k, int n, long long* tot,
                                                int* rank) {
    centroids_from_sums(c.sums + static_cast<uint64_t>(sum_sel) * c.sum_half, k, n, c.sum_unscale, c.cC, c.cmask,
                        c.cCact, c.cldc, c.cact, c.cn_active, c.cCT32, c.cdelta, tot, rank);
}

template <typename T>
__device__ __forceinline__ T raw_at(const unsigned char* raw, int p, int d) {
    if constexpr (sizeof(T) == 8) {  // 128-byte rows, SWIZZLE_128B: chunk ^= p & 7
        const int off = p * 128 + ((((d >> 1) ^ p) & 7) << 4) + ((d & 1) << 3);
        return *reinterpret_cast<const double*>(raw + off);
    } else {  // 64-byte rows, SWIZZLE_64B: chunk ^= (p >> 1) & 3
        const int off = p * 64 + ((((d >> 2) ^ (p >> 1)) & 3) << 4) + ((d & 3) << 2);
        return *reinterpret_cast<const float*>(raw + off);
    }
}

// One thread's share of a slab conversion: point p, dims 8h..8h+7 of the
// swizzled TMA slab (f32: 64-byte rows, SWIZZLE_64B; f64: 128-byte rows,
// SWIZZLE_128B) as 16-byte vector loads, into the fp32 [d][p] slab.
template <typename T>
__device__ __forceinline__ void convert_slab_part(const unsigned char* raw, float (*xs)[kABP], int p, int h) {
    if constexpr (sizeof(T) == 4) {
        const int sw = (p >> 1) & 3;
        const float4 a = *reinterpret_cast<const float4*>(raw + p * 64 + (((2 * h) ^ sw) << 4));
        const float4 b = *reinterpret_cast<const float4*>(raw + p * 64 + (((2 * h + 1) ^ sw) << 4));
        float* o = &xs[8 * h][p];
        o[0 * kABP] = a.x; o[1 * kABP] = a.y; o[2 * kABP] = a.z; o[3 * kABP] = a.w;
        o[4 * kABP] = b.x; o[5 * kABP] = b.y; o[6 * kABP] = b.z; o[7 * kABP] = b.w;
    } else {
        const int sw = p & 7;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double2 v = *reinterpret_cast<const double2*>(raw + p * 128 + (((4 * h + c) ^ sw) << 4));
            xs[8 * h + 2 * c][p] = static_cast<float>(v.x);
            xs[8 * h + 2 * c + 1][p] = static_cast<float>(v.y);
        }
    }
}

// Exact fp64 distance of one stored row to one centroid row: the reference's
// sequential chain (core.cpp:142-146) with vector loads (rows are 16-byte aligned
// whenever the TMA path runs: TMA strides are multiples of 16 bytes).
template <typename T>
__device__ __forceinline__ double exact_row_dist(const T* __restrict__ x, const double* __restrict__ c, int n) {
    double a = 0.0;
    int d = 0;
    if constexpr (sizeof(T) == 4) {
#pragma unroll 4
        for (; d + 4 <= n; d += 4) {
            const float4 xv = __ldg(reinterpret_cast<const float4*>(x + d));
            const double2 c0 = __ldg(reinterpret_cast<const double2*>(c + d));
            const double2 c1 = __ldg(reinterpret_cast<const double2*>(c + d + 2));
            a = dist_step(a, xv.x, c0.x);
            a = dist_step(a, xv.y, c0.y);
            a = dist_step(a, xv.z, c1.x);
            a = dist_step(a, xv.w, c1.y);
        }
    } else {
#pragma unroll 4
        for (; d + 2 <= n; d += 2) {
            const double2 xv = __ldg(reinterpret_cast<const double2*>(x + d));
            const double2 cv = __ldg(reinterpret_cast<const double2*>(c + d));
            a = dist_step(a, xv.x, cv.x);
            a = dist_step(a, xv.y, cv.y);
        }
    }
    for (; d < n; ++d) a = dist_step(a, to_f64(x[d]), c[d]);
    return a;
}

// Exact fp64 distance (core.cpp:142-146) of a point row staged in shared memory
// (fp32 storage, 16-byte aligned) to a centroid row read from L1/L2.
__device__ __forceinline__ double chain_smem_row(const float* x, const double* __restrict__ c, int n) {
    double a = 0.0;
    int d = 0;
#pragma unroll 4
    for (; d + 4 <= n; d += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(x + d);
        const double2 c0 = __ldg(reinterpret_cast<const double2*>(c + d));
        const double2 c1 = __ldg(reinterpret_cast<const double2*>(c + d + 2));
        a = dist_step(a, xv.x, c0.x);
        a = dist_step(a, xv.y, c0.y);
        a = dist_step(a, xv.z, c1.x);
        a = dist_step(a, xv.w, c1.y);
    }
    for (; d < n; ++d) a = dist_step(a, x[d], c[d]);
    return a;
}

// Exact fp64 distances (core.cpp:142-146) of `ni` (point, compacted centroid)
// items (ni <= 2 * kSThreads, up to 2 per thread), each chain carried in a
// register in dimension order.  The CTA's 128-row point block streams through
// the raw TMA ring again (one 16-dim slab per stage; slab i is TMA sequence
// number qb + i of this CTA), the matching centroid slabs through cp.async.
template <typename T, int NS>
__device__ __forceinline__ void tma_chains(TmaSmem<T, NS>& S, const CUtensorMap* tmx, uint64_t p0, int n, int nslab,
                                           int qb, const double* __restrict__ Cact, int ldc, int KA, uint32_t ni,
                                           const short* item_p, const signed char* item_j, double* item_d) {
    constexpr int kCS = 18;  // centroid slab row stride (doubles): 16-byte rows, spread banks
    // slabs in flight: the 6-stage ring (wide rows) keeps 4 ahead, its centroid
    // pieces in 5 buffers over the (now free) screen staging from craw on;
    // the 2-stage ring keeps 2 ahead in 2 buffers over xs
    constexpr int DEPTH = NS >= 6 ? 4 : 2;
    constexpr int NCB = DEPTH + 1 > 2 ? DEPTH + 1 : 2;
    using SmemT = TmaSmem<T, NS>;
    static_assert(NS < 6 || offsetof(SmemT, craw) + NCB * kSMaxK * kCS * sizeof(double) <=
                                offsetof(SmemT, red_u) - kItemCap * (sizeof(double) + 3),
                  "tma_chains centroid ring overlaps the item list");
    const int tid = threadIdx.x;
    double(*c64)[kSMaxK][kCS] = reinterpret_cast<double(*)[kSMaxK][kCS]>(
        NS >= 6 ? reinterpret_cast<void*>(&S.craw[0][0][0]) : reinterpret_cast<void*>(&S.xs[0][0][0]));
    __syncthreads();  // item list complete; the ring and the staging area are free
    double acc[2] = {0.0, 0.0};
    int ip[2] = {-1, -1}, ij[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const uint32_t i = tid + r * kSThreads;
        if (i < ni) {
            ip[r] = item_p[i];
            ij[r] = item_j[i];
        }
    }
    auto issue = [&](int sl) {
        const int st = (qb + sl) % NS, cb = sl % NCB;
        if (tid == 0) {
            mbar_expect_tx(&S.bar[st], TmaSmem<T, NS>::kRawBytes);
            tma_load_2d(S.raw[st], tmx, &S.bar[st], sl * kADC, static_cast<int>(p0));
        }
        if (tid < KA * (kADC / 2)) {
            const int j = tid >> 3, h = tid & 7, d = sl * kADC + 2 * h;
            if (d < n) cp_async_16(&c64[cb][j][2 * h], Cact + static_cast<uint64_t>(j) * ldc + d);
        }
        cp_async_commit();
    };
    for (int i = 0; i < DEPTH; ++i) {
        if (i < nslab) issue(i);
        else cp_async_commit();  // (empty groups keep the wait count uniform)
    }
    for (int sl = 0; sl < nslab; ++sl) {
        const int q = qb + sl, st = q % NS, cb = sl % NCB;
        cp_async_wait<DEPTH - 1>();  // slab sl's centroid pieces (DEPTH groups are in flight)
        mbar_wait(&S.bar[st], (q / NS) & 1);
        if (qb == 0 && sl < 5) ktrace(16 + 2 * sl, 2);
        __syncthreads();  // everyone's centroid pieces landed
        const int dl = min(kADC, n - sl * kADC);
        const unsigned char* raw = S.raw[st];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (ip[r] < 0) continue;
            const int p = ip[r];
            const double* cr = c64[cb][ij[r]];
            double a = acc[r];
            if (dl == kADC) {
                if constexpr (sizeof(T) == 4) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 xv = *reinterpret_cast<const float4*>(raw + p * 64 + (((c ^ (p >> 1)) & 3) << 4));
                        a = dist_step(a, xv.x, cr[4 * c]);
                        a = dist_step(a, xv.y, cr[4 * c + 1]);
                        a = dist_step(a, xv.z, cr[4 * c + 2]);
                        a = dist_step(a, xv.w, cr[4 * c + 3]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const double2 xv = *reinterpret_cast<const double2*>(raw + p * 128 + (((c ^ p) & 7) << 4));
                        a = dist_step(a, xv.x, cr[2 * c]);
                        a = dist_step(a, xv.y, cr[2 * c + 1]);
                    }
                }
            } else {
                for (int d = 0; d < dl; ++d) a = dist_step(a, to_f64(raw_at<T>(raw, p, d)), cr[d]);
            }
            acc[r] = a;
        }
        __syncthreads();  // stage st consumed
        if (qb == 0 && sl < 5) ktrace(17 + 2 * sl, 2);
        if (sl + DEPTH < nslab) issue(sl + DEPTH);
        else cp_async_commit();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int r = 0; r < 2; ++r)
        if (ip[r] >= 0) item_d[tid + r * kSThreads] = acc[r];
    __syncthreads();
}

// hmode: 0 = screen; 1 = screen and record the certified lower bound of every
// (point, active label) distance (lbk, distance units); 2 = Lloyd round: the
// exact distance to the previous label, then the bounds decayed by each
// label's centroid movement decide which labels need an exact recheck
// (Elkan-style; the reference's argmin is certified), else the full screen.
template <typename T, int NS>
__global__ void __launch_bounds__(kSThreads, NS <= 2 ? 3 : 2)
k_assign_tma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmc,
             const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
             const double* __restrict__ Cact, int ldc, const int* __restrict__ act_idx,
             const int* __restrict__ n_active_ptr,
             int32_t* __restrict__ labels_pair, uint64_t pair_stride,
             const int* __restrict__ parity_ptr, double* __restrict__ dists_out,
             int* __restrict__ changed_flag, const int* __restrict__ stop_ptr,
             double* __restrict__ tile_out, unsigned* __restrict__ tile_counter,
             unsigned long long* __restrict__ cand_counter, ScreenConsts cst, const __grid_constant__ LloydCtl ctl,
             int hmode, float* __restrict__ lbk, const float* __restrict__ delta, int kfull,
             uint64_t dstride, const PreDots pdots) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // pdots.best: wide rows pre-screened and rechecked by k_wide_screen /
    // k_wide_recheck (wide.cu) — each point's exact minimum comes precomputed;
    // no slab screen and no recheck here (hmode is 0)
    const bool pm = pdots.best != nullptr;
    // TMA destinations with 128-byte swizzle need 1024-byte alignment
    unsigned char* smem_al = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    TmaSmem<T, NS>& S = *reinterpret_cast<TmaSmem<T, NS>*>(smem_al);
    constexpr unsigned kStageBytes = TmaSmem<T, NS>::kRawBytes + kADC * kSMaxK * sizeof(float);

    klog_start(10 + hmode);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {  // independent of the previous kernel: overlaps its tail under PDL
        tma_prefetch_map(&tmx);
        tma_prefetch_map(&tmc);
        for (int i = 0; i < NS; ++i) mbar_init(&S.bar[i], 1);
        fence_mbar_init();
    }
    pdl_wait();
    if (stop_ptr && *stop_ptr) {  // a finished loop: close the WHILE node if this launch drives one
        if (ctl.use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(ctl.cond, 0u);
        klog_exit(10 + hmode);
        return;
    }
    if (ctl.go && !*ctl.go) {
        klog_exit(10 + hmode);
        return;
    }
    if (ctl.begin_kind == 2 && ctl.st->begin_version ==
                                   static_cast<long long>(*reinterpret_cast<const volatile long long*>(&ctl.gs->inc_version))) {
        // the speculative begin of this chunk is current; with the fused exact-sum
        // update CTA 0 turns its sums into round 1's centroids
        if (ctl.sum_fuse) {  // a label per CTA (round 1's centroids)
            const long long* half = ctl.sums + static_cast<uint64_t>(ctl.st->sum_sel) * ctl.sum_half;
            for (int j = static_cast<int>(blockIdx.x); j < kfull; j += static_cast<int>(gridDim.x)) {
                centroid_of_label(half, kfull, n, ctl.sum_unscale, ctl.cC, ctl.cmask, ctl.cCact, ctl.cldc, ctl.cact,
                                  ctl.cn_active, ctl.cCT32, ctl.cdelta, j, reinterpret_cast<double*>(&S.red_u[0][0]));
                __syncthreads();
            }
        }
        klog_exit(10 + hmode);
        return;
    }
    if (ctl.begin_kind == 1) {  // speculative begin: the incumbent version before any of its reads
        if (threadIdx.x == 0) {
            const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(&ctl.gs->inc_version));
            atomicMin(reinterpret_cast<unsigned long long*>(&ctl.st->bv_min), v);
            __threadfence();
        }
        __syncthreads();
    }
    const int KA = *n_active_ptr;
    int32_t* labels_out = labels_pair;
    const int32_t* labels_old = nullptr;
    if (parity_ptr) {  // rounds: read slot par (0, 1, or 2 after a graph-mode begin), write the other of 0/1
        const int par = *parity_ptr, out = par == 0 ? 1 : 0;
        labels_out = labels_pair + out * pair_stride;
        labels_old = labels_pair + par * pair_stride;
        if (dists_out) dists_out += out * dstride;  // dstride 0: one distance buffer
    }
    const int KG = (KA + kAK - 1) / kAK;
    const bool comp = warp < KG;
    const bool normw = warp == 7;
    const float finf = __int_as_float(0x7F800000);
    const int nslab = (n + kADC - 1) / kADC;
    // reusable block (pass-1 buffers) for the staged exact chains; item list at its end
    unsigned char* reuse = &S.raw[0][0];
    const size_t reuse_bytes = static_cast<size_t>(reinterpret_cast<unsigned char*>(&S.red_u[0][0]) - reuse);
    double* item_d = reinterpret_cast<double*>(reuse + reuse_bytes - kItemCap * (sizeof(double) + 3));
    short* item_p = reinterpret_cast<short*>(item_d + kItemCap);
    signed char* item_j = reinterpret_cast<signed char*>(item_p + kItemCap);
    using SmemT = TmaSmem<T, NS>;
    static_assert(offsetof(SmemT, red_u) - kItemCap * (sizeof(double) + 3) >=
                      offsetof(SmemT, xs) + 2 * kSMaxK * 18 * sizeof(double),
                  "centroid staging of tma_chains overlaps the item list");
    ktrace(0, hmode);
    int qb = 0;  // TMA slabs this CTA has consumed (ring position)
    // one 128-point block per CTA, or (ctl.nblk: a speculative begin capped in
    // CTAs so that it leaves SM slots to the engine stream) a loop over blocks
    const unsigned nblk = ctl.nblk ? ctl.nblk : gridDim.x;
    for (unsigned blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const uint64_t p0 = static_cast<uint64_t>(blk) * kABP;
    const int np = p0 < rows ? static_cast<int>(min(static_cast<uint64_t>(kABP), rows - p0)) : 0;
    const float* pre_rows = nullptr;  // the full screen's staged fp32 rows ([128][ld]), for the label sums
    if (np == 0) {  // fixup CTA of a round-1 launch: one tile of the pending chunk's final distances
        const GState* gst = ctl.gs;
        const int pend = gst->pending_fix;
        if (ctl.fix_tiles && pend >= 0) {
            const uint64_t t = (p0 - rows) / kABP;  // fixup CTAs follow the point blocks
            const uint64_t R = ctl.fix_rows, tb = t * kTile;
            if (tb < R) {
                const double* dv = ctl.dists_all + (3 * static_cast<uint64_t>(pend % kStateBufs) + gst->fix_par) * R + tb;
                const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), R - tb));
                double* fbuf = reinterpret_cast<double*>(&S.raw[0][0]);
                for (int i = tid; i < len; i += kSThreads) fbuf[i] = __ldcg(dv + i);
                __syncthreads();
                if (tid == 0) ctl.fix_tiles[t] = seq_fold_smem(fbuf, len);
            }
        }
        goto fold;
    }  // TMA slabs this CTA has consumed (ring position)

    // ------- Lloyd-round fast path, fp32 storage (exact, certified) -------
    // As the generic path below, but the CTA's point rows and bound rows are
    // fetched once with cp.async at the start (overlapping the setup), and
    // every exact chain reads its point from shared memory.
    if constexpr (sizeof(T) == 4) {
        const int ldr = static_cast<int>(ld);  // floats per row, a multiple of 4
        const size_t rows_cap = static_cast<size_t>(reinterpret_cast<unsigned char*>(item_d) - reuse);
        if (hmode == 2 && labels_old && lbk && delta && static_cast<size_t>(kABP) * ldr * 4 <= rows_cap) {
            float* xr = reinterpret_cast<float*>(reuse);  // [128][ldr]
            const int vpr = ldr / 4;
            for (int e = tid; e < np * vpr; e += kSThreads) {
                const int p = e / vpr, v = e - p * vpr;
                cp_async_16(xr + p * ldr + 4 * v, X + (p0 + p) * ld + 4 * v);
            }
            for (int e = tid; e < np * (kSMaxK / 4); e += kSThreads) {
                const int p = e >> 3, c = e & 7;
                cp_async_16(&S.lbs[p][4 * ((c ^ p) & 7)], lbk + (p0 + p) * kSMaxK + 4 * c);
            }
            cp_async_commit();
            if (tid < kSMaxK) {
                S.rank_of[tid] = -1;
                S.delta[tid] = 0.f;
            }
            __syncthreads();
            if (tid < KA) {
                const int j = act_idx[tid];
                S.rank_of[j] = tid;
                S.delta[j] = delta[j];  // movement of label j in the last update (rounded up)
            }
            int a = -1, ra = -1;
            if (tid < np) a = labels_old[p0 + tid];
            cp_async_wait<0>();
            __syncthreads();  // rows, bounds, ranks and movements in place
            if (tid < np) ra = (a >= 0 && a < kfull) ? S.rank_of[a] : -1;
            ktrace(13, hmode);
            // the exact distance to the previous label; decayed bounds of the others
            unsigned fails = 0;
            double dn = 0.0;
            if (tid < np) {
                if (ra >= 0) dn = chain_smem_row(xr + tid * ldr, Cact + static_cast<uint64_t>(ra) * ldc, n);
#pragma unroll
                for (int c4 = 0; c4 < kSMaxK / 4; ++c4) {
                    float* vv = &S.lbs[tid][4 * ((c4 ^ tid) & 7)];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = 4 * c4 + e;
                        if (S.rank_of[j] < 0 || j == a) continue;
                        const float lbn = fmaxf(__fsub_rd(vv[e], S.delta[j]), 0.f);
                        vv[e] = lbn;
                        const float L = __fmul_rd(__fmul_rd(lbn, lbn), cst.lo64);
                        if (ra < 0 || !(dn < static_cast<double>(L))) fails |= 1u << j;
                    }
                }
            }
            if (tid < kABP) S.cand[tid] = fails;
            __syncthreads();
            if (tid < 32) {  // exclusive scan of the per-point recheck counts -> item offsets
                int v[4], run = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    v[q] = __popc(S.cand[4 * tid + q]);
                    run += v[q];
                }
                int incl = run;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (tid >= o) incl += y;
                }
                int ex = incl - run;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    S.icount[4 * tid + q] = ex;
                    ex += v[q];
                }
                if (tid == 31) S.n_items = static_cast<uint32_t>(incl);
            }
            __syncthreads();
            const uint32_t NI = S.n_items;
            if (tid == 0 && cand_counter) {
                atomicAdd(cand_counter, static_cast<unsigned long long>(np + NI));
                atomicAdd(cand_counter + 1, static_cast<unsigned long long>(np));
            }
            if (NI <= static_cast<uint32_t>(kItemCap)) {
                if (tid < np) {
                    uint32_t it = S.icount[tid];
                    unsigned bits = fails;
                    while (bits) {  // ascending label = ascending compacted rank
                        const int j = __ffs(bits) - 1;
                        bits &= bits - 1;
                        item_p[it] = static_cast<short>(tid);
                        item_j[it] = static_cast<signed char>(S.rank_of[j]);
                        ++it;
                    }
                }
                __syncthreads();
                for (uint32_t i = tid; i < NI; i += kSThreads)
                    item_d[i] = chain_smem_row(xr + item_p[i] * ldr, Cact + static_cast<uint64_t>(item_j[i]) * ldc, n);
                __syncthreads();
                if (tid < np) {
                    const uint64_t gp = p0 + tid;
                    // (value, label) minimum over the previous label and the rechecked ones:
                    // every other label is certified strictly farther (core.cpp:147)
                    const double inf = __longlong_as_double(0x7FF0000000000000LL);
                    double best = ra >= 0 ? dn : inf;
                    int bl = ra >= 0 ? a : -1;
                    const uint32_t i0 = S.icount[tid], i1 = i0 + __popc(fails);
                    const double hi = static_cast<double>(cst.hi64);
                    auto lbound = [&](double d) {  // true distance >= fl64 distance / (1+g64)
                        const double q = __dsub_rd(__ddiv_rd(d, hi), 1e-300);
                        return q > 0.0 ? (q < 3.0e38 ? __fsqrt_rd(__double2float_rd(q)) : 1.0e19f) : 0.f;
                    };
                    for (uint32_t i = i0; i < i1; ++i) {
                        const double d = item_d[i];
                        const int l = act_idx[item_j[i]];
                        S.lbs[tid][4 * (((l >> 2) ^ tid) & 7) + (l & 3)] = lbound(d);
                        if (d < best || (d == best && l < bl)) {
                            best = d;
                            bl = l;
                        }
                    }
                    if (ra >= 0) S.lbs[tid][4 * (((a >> 2) ^ tid) & 7) + (a & 3)] = lbound(dn);
                    labels_out[gp] = bl;
                    if (dists_out) dists_out[gp] = best;
                    if (bl != a) *changed_flag = 1;
                    S.lab_new[tid] = bl;
                    S.lab_old[tid] = a;
                }
                __syncthreads();
                for (int e = tid; e < np * (kSMaxK / 4); e += kSThreads) {  // bound rows back, coalesced
                    const int p = e >> 3, c = e & 7;
                    reinterpret_cast<float4*>(lbk + (p0 + p) * kSMaxK)[c] =
                        *reinterpret_cast<const float4*>(&S.lbs[p][4 * ((c ^ p) & 7)]);
                }
                ktrace(15, hmode);
                pre_rows = xr;  // the label sums read the moved rows from here
                goto fold;
            }
            // many rechecks: the full screen below rewrites everything; its TMA
            // writes (async proxy) follow our generic writes to the same bytes
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
        }
    }

    // ---------------- Lloyd-round fast path (exact, certified) ----------------
    // Per (point, label) lower bounds in distance units (lbk, written by the
    // previous assignment) minus the label's centroid movement stay lower
    // bounds.  A label whose decayed bound squared (x (1-g64)) exceeds the
    // exact distance to the previous label cannot win or tie the reference's
    // scan; the others are rechecked exactly.  Too many rechecks: full screen.
    if (hmode == 2 && labels_old && lbk && delta &&
        !(sizeof(T) == 4 && static_cast<size_t>(kABP) * ld * 4 <=
                                static_cast<size_t>(reinterpret_cast<unsigned char*>(item_d) - reuse))) {
        if (tid < kSMaxK) {
            S.rank_of[tid] = -1;
            S.delta[tid] = 0.f;
        }
        __syncthreads();
        if (tid < KA) S.rank_of[act_idx[tid]] = tid;
        if (tid < KA) {  // per-label movement of the last update (k_update's last merger)
            const int j = act_idx[tid];
            S.delta[j] = delta[j];
        }
        __syncthreads();
        ktrace(13, hmode);
        int a = -1, ra = -1;
        if (tid < np) {
            a = labels_old[p0 + tid];
            ra = (a >= 0 && a < kfull) ? S.rank_of[a] : -1;
            item_p[tid] = static_cast<short>(tid);
            item_j[tid] = static_cast<signed char>(ra < 0 ? 0 : ra);
        }
        ktrace(26, hmode);
        tma_chains<T>(S, &tmx, p0, n, nslab, qb, Cact, ldc, KA, static_cast<uint32_t>(np), item_p, item_j, item_d);
        qb += nslab;
        // decay the bounds, test every other active label
        unsigned fails = 0;
        double dn = 0.0;
        if (tid < np) {
            dn = item_d[tid];
            float4* row = reinterpret_cast<float4*>(lbk + (p0 + tid) * kSMaxK);
#pragma unroll
            for (int c4 = 0; c4 < kSMaxK / 4; ++c4) {
                float4 v = __ldcg(row + c4);
                float* vv = reinterpret_cast<float*>(&v);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = 4 * c4 + e;
                    if (S.rank_of[j] < 0 || j == a) continue;
                    const float lbn = fmaxf(__fsub_rd(vv[e], S.delta[j]), 0.f);
                    vv[e] = lbn;
                    const float L = __fmul_rd(__fmul_rd(lbn, lbn), cst.lo64);
                    if (ra < 0 || !(dn < static_cast<double>(L))) fails |= 1u << j;
                }
                row[c4] = v;
            }
        }
        if (tid < kABP) S.cand[tid] = fails;
        __syncthreads();
        if (tid < 32) {  // exclusive scan of the per-point recheck counts -> item offsets
            int v[4], run = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                v[q] = __popc(S.cand[4 * tid + q]);
                run += v[q];
            }
            int incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (tid >= o) incl += y;
            }
            int ex = incl - run;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                S.icount[4 * tid + q] = ex;
                ex += v[q];
            }
            if (tid == 31) S.n_items = static_cast<uint32_t>(incl);
        }
        __syncthreads();
        const uint32_t NI = S.n_items;
        if (tid == 0 && cand_counter) {
            atomicAdd(cand_counter, static_cast<unsigned long long>(np + NI));
            atomicAdd(cand_counter + 1, static_cast<unsigned long long>(np));
        }
#ifdef BM_KTRACE
        if (tid == 0) {  // fast-path statistics: [199990] CTAs, [199991] fallbacks, [199992] rechecked pairs
            atomicAdd(&g_ktrace[199990], 1ull);
            if (NI > static_cast<uint32_t>(kItemCap)) atomicAdd(&g_ktrace[199991], 1ull);
            atomicAdd(&g_ktrace[199992], static_cast<unsigned long long>(NI));
            unsigned pts = 0;
            for (int q = 0; q < kABP; ++q) pts += S.cand[q] != 0;
            atomicAdd(&g_ktrace[199993], static_cast<unsigned long long>(pts));
        }
#endif
        if (NI <= static_cast<uint32_t>(kItemCap)) {
            // own-label distances stay in registers; the item list is rebuilt for the rechecks
            if (tid < np) {
                uint32_t it = S.icount[tid];
                unsigned bits = fails;
                while (bits) {  // ascending label = ascending compacted rank
                    const int j = __ffs(bits) - 1;
                    bits &= bits - 1;
                    item_p[it] = static_cast<short>(tid);
                    item_j[it] = static_cast<signed char>(S.rank_of[j]);
                    ++it;
                }
            }
            if (NI > static_cast<uint32_t>(kSThreads) || (NI > 0 && n > 256)) {  // (wide rows: streamed)
                tma_chains<T>(S, &tmx, p0, n, nslab, qb, Cact, ldc, KA, NI, item_p, item_j, item_d);
                qb += nslab;
            } else if (NI > 0) {  // few rechecks: one thread per item, rows straight from L2
                __syncthreads();
                if (tid < static_cast<int>(NI))
                    item_d[tid] = exact_row_dist(X + (p0 + item_p[tid]) * ld,
                                                 Cact + static_cast<uint64_t>(item_j[tid]) * ldc, n);
                __syncthreads();
            }
            if (tid < np) {
                const uint64_t gp = p0 + tid;
                // (value, label) minimum over the previous label and the rechecked ones:
                // every other label is certified strictly farther (core.cpp:147)
                const double inf = __longlong_as_double(0x7FF0000000000000LL);
                double best = ra >= 0 ? dn : inf;
                int bl = ra >= 0 ? a : -1;
                const uint32_t i0 = S.icount[tid], i1 = i0 + __popc(fails);
                float* row = lbk + gp * kSMaxK;
                const double hi = static_cast<double>(cst.hi64);
                auto lbound = [&](double d) {  // true distance >= fl64 distance / (1+g64)
                    const double q = __dsub_rd(__ddiv_rd(d, hi), 1e-300);
                    return q > 0.0 ? (q < 3.0e38 ? __fsqrt_rd(__double2float_rd(q)) : 1.0e19f) : 0.f;
                };
                for (uint32_t i = i0; i < i1; ++i) {
                    const double d = item_d[i];
                    const int l = act_idx[item_j[i]];
                    row[l] = lbound(d);
                    if (d < best || (d == best && l < bl)) {
                        best = d;
                        bl = l;
                    }
                }
                if (ra >= 0) row[a] = lbound(dn);
                labels_out[gp] = bl;
                if (dists_out) dists_out[gp] = best;
                if (bl != a) *changed_flag = 1;
                    S.lab_new[tid] = bl;
                    S.lab_old[tid] = a;
            }
            ktrace(15, hmode);
            goto fold;
        }
        // many rechecks: full screen of the block (rewrites labels, distances, bounds)
        __syncthreads();
    }
    {
    __syncthreads();
    auto issue = [&](int sl) {
        const int st = (qb + sl) % NS;
        mbar_expect_tx(&S.bar[st], kStageBytes);
        tma_load_2d(S.raw[st], &tmx, &S.bar[st], sl * kADC, static_cast<int>(p0));
        tma_load_2d(&S.craw[st][0][0], &tmc, &S.bar[st], 0, sl * kADC);
    };
    if (tid == 0 && !pm)
        for (int i = 0; i < NS && i < nslab; ++i) issue(i);

    float2 tot[2][kAK];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < kAK; ++u) tot[h][u] = make_float2(0.f, 0.f);
    float nxl[4] = {0.f, 0.f, 0.f, 0.f}, nxh[4] = {0.f, 0.f, 0.f, 0.f};
    float ncl = 0.f, nch = 0.f;
    const int cp_ = tid & (kABP - 1), chalf = tid >> 7;  // conversion: point, 8-dim half

    for (int sl = 0; sl < (pm ? 0 : nslab); ++sl) {
        const int q = qb + sl, st = q % NS, xb = q & 1, dl = min(kADC, n - sl * kADC);
        mbar_wait(&S.bar[st], (q / NS) & 1);
        if (sl < 6) ktrace(1 + sl, hmode);
        // raw (swizzled [p][d], storage type) -> fp32 [d][p], once per element
        convert_slab_part<T>(S.raw[st], S.xs[xb], cp_, chalf);
        if (tid < kADC * kSMaxK / 4) {
            const float4 v = reinterpret_cast<const float4*>(&S.craw[st][0][0])[tid];
            reinterpret_cast<float4*>(&S.cs[xb][0][0])[tid] = v;
        }
        __syncthreads();  // slab ready; every thread has left slab sl-1 and stage st is free
        if (tid == 0 && sl + NS < nslab) issue(sl + NS);
        if (comp) {
            float2 part[2][kAK];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < kAK; ++u) part[h][u] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int d = 0; d < dl; ++d) {
                const float4 xv = *reinterpret_cast<const float4*>(&S.xs[xb][d][4 * lane]);
                const float4 cv = *reinterpret_cast<const float4*>(&S.cs[xb][d][4 * warp]);
                const float2 xa = make_float2(xv.x, xv.y), xb = make_float2(xv.z, xv.w);
                part[0][0] = ffma2(xa, cv.x, part[0][0]);
                part[0][1] = ffma2(xa, cv.y, part[0][1]);
                part[0][2] = ffma2(xa, cv.z, part[0][2]);
                part[0][3] = ffma2(xa, cv.w, part[0][3]);
                part[1][0] = ffma2(xb, cv.x, part[1][0]);
                part[1][1] = ffma2(xb, cv.y, part[1][1]);
                part[1][2] = ffma2(xb, cv.z, part[1][2]);
                part[1][3] = ffma2(xb, cv.w, part[1][3]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < kAK; ++u) tot[h][u] = fadd2(tot[h][u], part[h][u]);
        }
        if (normw) {
            for (int d = 0; d < dl; ++d) {
                const float4 xv = *reinterpret_cast<const float4*>(&S.xs[xb][d][4 * lane]);
                nxl[0] = __fmaf_rd(xv.x, xv.x, nxl[0]); nxh[0] = __fmaf_ru(xv.x, xv.x, nxh[0]);
                nxl[1] = __fmaf_rd(xv.y, xv.y, nxl[1]); nxh[1] = __fmaf_ru(xv.y, xv.y, nxh[1]);
                nxl[2] = __fmaf_rd(xv.z, xv.z, nxl[2]); nxh[2] = __fmaf_ru(xv.z, xv.z, nxh[2]);
                nxl[3] = __fmaf_rd(xv.w, xv.w, nxl[3]); nxh[3] = __fmaf_ru(xv.w, xv.w, nxh[3]);
                const float c = S.cs[xb][d][lane];
                ncl = __fmaf_rd(c, c, ncl);
                nch = __fmaf_ru(c, c, nch);
            }
        }
    }
    if (!pm) qb += nslab;  // (the screen's slabs; a streamed recheck takes them again below)
    if (normw && !pm) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            S.nx_lo[4 * lane + q] = nxl[q];
            S.nx_hi[4 * lane + q] = nxh[q];
            S.nxr[4 * lane + q] = __fsqrt_ru(nxh[q]);
        }
        S.nc_lo[lane] = ncl;
        S.nc_hi[lane] = nch;
        S.ncr[lane] = __fsqrt_ru(nch);
    }
    __syncthreads();
    ktrace(7, hmode);
    // fp32 rows that fit the freed slab buffers: fetched now with cp.async,
    // landing while the bounds are computed; the exact rechecks and the label
    // sums then read them from shared memory
    float* const xrow = reinterpret_cast<float*>(reuse);
    const int ldr = static_cast<int>(ld);
    const bool pre = sizeof(T) == 4 && static_cast<size_t>(kABP) * ld * 4 <=
                                           static_cast<size_t>(reinterpret_cast<unsigned char*>(item_d) - reuse);
    if (pre) {
        pre_rows = xrow;
        const int vpr = ldr / 4;
        for (int e = tid; e < np * vpr; e += kSThreads) {
            const int p = e / vpr, v = e - p * vpr;
            cp_async_16(xrow + p * ldr + 4 * v, X + (p0 + p) * ld + 4 * v);
        }
        cp_async_commit();
    }
    // certified bounds: upper bounds first, then each warp tests its lower
    // bounds against the point's minimum U and sets candidate bits.
    float Lk[4][kAK];
    if (tid < kABP) S.cand[tid] = 0u;
    if (comp && !pm) {
        float un[4] = {finf, finf, finf, finf};
#pragma unroll
        for (int u = 0; u < kAK; ++u) {
            const int j = kAK * warp + u;
            const float cl = j < KA ? S.nc_lo[j] : 0.f, ch = j < KA ? S.nc_hi[j] : 0.f;
            const float crr = j < KA ? S.ncr[j] : 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int p = 4 * lane + q;
                const float sdot = q & 1 ? tot[q >> 1][u].y : tot[q >> 1][u].x;
                const float t2 = 2.f * sdot;
                const float Sn = __fadd_ru(S.nxr[p], crr);
                const float Al = __fadd_rd(S.nx_lo[p], cl), Ah = __fadd_ru(S.nx_hi[p], ch);
                float L = 0.f, U = finf;
                if (fabsf(t2) <= 1.0e37f && Sn <= 1.0e18f && Ah <= 1.0e37f) {
                    const float D = __fadd_ru(__fmul_ru(__fmul_ru(cst.K, Sn), Sn), cst.dabs);
                    L = fmaxf(__fsub_rd(__fsub_rd(Al, t2), D), 0.f);
                    L = __fmul_rd(L, cst.lo64);
                    U = __fmul_ru(__fadd_ru(__fsub_ru(Ah, t2), D), cst.hi64);
                }
                Lk[q][u] = j < KA ? L : finf;
                if (j < KA) un[q] = fminf(un[q], U);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) S.red_u[warp][4 * lane + q] = un[q];
    }
    __syncthreads();
    if (comp && !pm) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int p = 4 * lane + q;
            float m = finf;
            for (int g = 0; g < KG; ++g) m = fminf(m, S.red_u[g][p]);
            unsigned bits = 0;
#pragma unroll
            for (int u = 0; u < kAK; ++u)
                if (kAK * warp + u < KA && Lk[q][u] <= m) bits |= 1u << (kAK * warp + u);
            if (bits && p < np) atomicOr(&S.cand[p], bits);
        }
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the candidate counts -> item offsets
        int v[4], run = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = __popc(S.cand[4 * tid + q]);
            run += v[q];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= o) incl += y;
        }
        int ex = incl - run;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            S.icount[4 * tid + q] = ex;
            ex += v[q];
        }
        if (tid == 31) {
            S.n_items = static_cast<uint32_t>(incl);
            if (cand_counter) {
                atomicAdd(cand_counter, static_cast<unsigned long long>(incl));
                atomicAdd(cand_counter + 1, static_cast<unsigned long long>(np));
            }
        }
    }
    __syncthreads();
    const uint32_t NI = S.n_items;
    const bool overflow = NI > static_cast<uint32_t>(kItemCap);
    ktrace(8, hmode);
    // ---- pass 2: exact fp64 recheck of the candidates ----
    if (!overflow) {
        if (tid < np) {
            const int p = tid;
            uint32_t it = S.icount[p];
            unsigned bits = S.cand[p];
            while (bits) {  // ascending j
                const int j = __ffs(bits) - 1;
                bits &= bits - 1;
                item_p[it] = static_cast<short>(p);
                item_j[it] = static_cast<signed char>(j);
                ++it;
            }
        }
        if (pre) {  // the rows from shared memory (up to 2 items per thread)
            cp_async_wait<0>();
            __syncthreads();
            for (uint32_t i = tid; i < NI; i += kSThreads)
                item_d[i] = chain_smem_row(xrow + item_p[i] * ldr, Cact + static_cast<uint64_t>(item_j[i]) * ldc, n);
            __syncthreads();
        } else if (NI > 0 && (NI > static_cast<uint32_t>(kSThreads) || n > 256)) {
            // streamed through the TMA ring (wide rows: a chain straight from L2
            // would wait one L2 round trip per 16 dims)
            tma_chains<T>(S, &tmx, p0, n, nslab, qb, Cact, ldc, KA, NI, item_p, item_j, item_d);
            qb += nslab;
        } else {  // one item per thread, rows straight from L2
            __syncthreads();
            if (tid < static_cast<int>(NI))
                item_d[tid] = exact_row_dist(X + (p0 + item_p[tid]) * ld,
                                             Cact + static_cast<uint64_t>(item_j[tid]) * ldc, n);
            __syncthreads();
        }
    }
    if (pre && overflow) {  // (the rows are still read by the label sums)
        cp_async_wait<0>();
        __syncthreads();
    }
    ktrace(9, hmode);
    if (tid < np) {
        const int p = tid;
        const uint64_t gp = p0 + p;
        double best = __longlong_as_double(0x7FF0000000000000LL);
        int bj = -1;
        if (pm) {  // k_wide_recheck's minimum
            best = pdots.best[gp];
            bj = pdots.bj[gp];
        } else if (!overflow) {  // ascending j, strict < (core.cpp:147)
            const uint32_t b1 = p + 1 < np ? static_cast<uint32_t>(S.icount[p + 1]) : NI;
            for (uint32_t i = S.icount[p]; i < b1; ++i) {
                if (item_d[i] < best) {
                    best = item_d[i];
                    bj = item_j[i];
                }
            }
        } else {  // candidate sets too large for the item buffer: full exact scan
            const T* x = X + gp * ld;
            for (int j = 0; j < KA; ++j) {
                const double* c = Cact + static_cast<uint64_t>(j) * ldc;
                double sm = 0.0;
                for (int d = 0; d < n; ++d) sm = dist_step(sm, to_f64(x[d]), c[d]);
                if (sm < best) {
                    best = sm;
                    bj = j;
                }
            }
        }
        const int label = bj >= 0 ? act_idx[bj] : -1;
        labels_out[gp] = label;
        if (dists_out) dists_out[gp] = best;
        const int lold = labels_old ? labels_old[gp] : -1;
        if (labels_old && lold != label) *changed_flag = 1;
        S.lab_rank[p] = bj;
        S.lab_new[p] = label;
        S.lab_old[p] = lold;
    }
    if (hmode >= 1 && lbk) {  // per (point, label) lower bounds in distance units, staged for coalesced rows
        __syncthreads();
        // [128][32], column j ^ (p & 31); the staged rows keep the slab buffers
        float* lbt = pre ? reinterpret_cast<float*>(&S.lbs[0][0]) : reinterpret_cast<float*>(&S.raw[0][0]);
        if (comp) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int p = 4 * lane + q;
#pragma unroll
                for (int u = 0; u < kAK; ++u) {
                    const int c = kAK * warp + u;
                    if (c < KA) lbt[p * kSMaxK + (act_idx[c] ^ (p & 31))] = __fsqrt_rd(Lk[q][u]);
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < np * (kSMaxK / 4); e += kSThreads) {
            const int p = e >> 3, c4 = (e & 7) * 4;
            float4 v;
            v.x = lbt[p * kSMaxK + ((c4 + 0) ^ (p & 31))];
            v.y = lbt[p * kSMaxK + ((c4 + 1) ^ (p & 31))];
            v.z = lbt[p * kSMaxK + ((c4 + 2) ^ (p & 31))];
            v.w = lbt[p * kSMaxK + ((c4 + 3) ^ (p & 31))];
            reinterpret_cast<float4*>(lbk + (p0 + p) * kSMaxK)[e & 7] = v;
        }
        ktrace(27, hmode);
    }
    }
fold:
    ktrace(10, hmode);
    if (ctl.sums && np > 0) label_sums<T>(S, ctl, X, ld, n, p0, np, labels_old == nullptr, kfull, reuse,
                                          static_cast<size_t>(reinterpret_cast<unsigned char*>(item_d) - reuse), blk,
                                          pre_rows);
    ktrace(31, hmode);
    if (ctl.fast) {  // unordered CTA sum -> st->fsum; the last CTA runs the control
        __syncthreads();  // distances of this CTA written (some by other threads)
        double v = tid < np ? dists_out[p0 + tid] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
        double* wsum = reinterpret_cast<double*>(&S.red_u[0][0]);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double c = 0.0;
            for (int w = 0; w < kSThreads / 32; ++w) c += wsum[w];
            atomicAdd(&ctl.st->fsum, c);
        }
        if (blk + gridDim.x < nblk) {  // the next block's TMA loads land in buffers written generically
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
        }
        continue;
    }
    if (!tile_out) return;
    __syncthreads();
    const uint64_t tile = p0 / kTile;
    if (tid == 0) {
        __threadfence();
        const uint64_t tb = tile * kTile;
        const unsigned ctas = static_cast<unsigned>((min(rows, tb + kTile) - tb + kABP - 1) / kABP);
        const unsigned old = atomicAdd(&tile_counter[tile], 1u);
        S.is_last = old == ctas - 1;
    }
    __syncthreads();
    ktrace(11, hmode);
    if (!S.is_last) return;
    __threadfence();
    const uint64_t tb = tile * kTile;
    const int len = static_cast<int>(min(rows, tb + kTile) - tb);
    double* fold = reinterpret_cast<double*>(&S.raw[0][0]);
    for (int i = tid; i < len; i += kSThreads) fold[i] = __ldcg(dists_out + tb + i);
    __syncthreads();
    if (tid == 0) {
        double a = 0.0;
        int i = 0;
        for (; i + 8 <= len; i += 8) {
            const double2 v0 = *reinterpret_cast<const double2*>(fold + i);
            const double2 v1 = *reinterpret_cast<const double2*>(fold + i + 2);
            const double2 v2 = *reinterpret_cast<const double2*>(fold + i + 4);
            const double2 v3 = *reinterpret_cast<const double2*>(fold + i + 6);
            a = __dadd_rn(a, v0.x); a = __dadd_rn(a, v0.y);
            a = __dadd_rn(a, v1.x); a = __dadd_rn(a, v1.y);
            a = __dadd_rn(a, v2.x); a = __dadd_rn(a, v2.y);
            a = __dadd_rn(a, v3.x); a = __dadd_rn(a, v3.y);
        }
        for (; i < len; ++i) a = __dadd_rn(a, fold[i]);
        tile_out[tile] = a;
        ktrace(12, hmode);
        tile_counter[tile] = 0u;
        tile_done_control(ctl, tile_out, rows);
    }
    }  // point blocks
    if (!ctl.fast) return;
    {
        if (tid == 0) {  // this CTA's arrival (its blocks' sums are in st->fsum)
            __threadfence();
            const unsigned done = atomicAdd(&ctl.st->ctas_done, 1u);
            S.is_last = done == gridDim.x - 1;
        }
        __syncthreads();
        if (!S.is_last) return;
        __threadfence();
        ktrace(28, hmode);
        // Everything the control and the accept read, in one round trip: the
        // status, the chain state, the chunk counter, both masks, the fixup
        // tile partials and the incumbent's centroids (the usual next start),
        // staged in shared memory (the pass-1 buffers are free now).
        LloydStatus* sst = reinterpret_cast<LloydStatus*>(&S.red_u[0][0]);
        constexpr int kW = sizeof(LloydStatus) / 8;
        for (int i = tid; i < kW; i += kSThreads)
            reinterpret_cast<unsigned long long*>(sst)[i] = __ldcg(reinterpret_cast<const unsigned long long*>(ctl.st) + i);
        const bool tail_acc = ctl.has_acc && ctl.mode == 2;
        TailIn* tin = reinterpret_cast<TailIn*>(reuse);
        double* stage = nullptr;  // k x n doubles for the accept's copies
        bool cinc_staged = false;
        if (tail_acc) {
            constexpr int kG = sizeof(GState) / 8;
            if (tid < kG)
                reinterpret_cast<unsigned long long*>(&tin->gs)[tid] =
                    __ldcg(reinterpret_cast<const unsigned long long*>(ctl.gs) + tid);
            if (tid == 32) tin->chunk = __ldcg(ctl.acc.chunk_ctr);
            if (tid >= 64 && tid < 64 + kfull) {
                tin->mk_inc[tid - 64] = ctl.acc.maskinc[tid - 64];
                tin->mk_cand[tid - 64] = ctl.acc.mask[tid - 64];
            }
            const int kn = kfull * n;
            if (ctl.accept_run && 16384 + static_cast<size_t>(kn) * 8 <= reuse_bytes) {
                stage = reinterpret_cast<double*>(reuse + 16384);
                for (int e = tid; e < kn; e += kSThreads) stage[e] = __ldcg(ctl.acc.Cinc + e);
                cinc_staged = true;
            }
        }
        const double* fix_tiles = ctl.fix_tiles;  // the fixup tile partials, staged for the control's fold
        if (fix_tiles) {
            double* ft = reinterpret_cast<double*>(&S.raw[0][0]) + 1024;
            const int nt = static_cast<int>(tiles_of(ctl.fix_rows));
            if (nt <= 1024) {
                for (int i = tid; i < nt; i += kSThreads) ft[i] = __ldcg(ctl.fix_tiles + i);
                fix_tiles = ft;
            }
        }
        __syncthreads();
        ktrace(1, hmode);
        if (tid == 0)
            S.n_items = static_cast<uint32_t>(
                lloyd_fast_control(ctl, sst, rows, nblk, KA, tail_acc ? &tin->gs : ctl.gs, fix_tiles));
        ktrace(2, hmode);
        __syncthreads();
        ktrace(29, hmode);
        const int decision = static_cast<int>(S.n_items);
        if (decision >= 0) accept_fast(sst, ctl.acc, decision, tin, stage, cinc_staged);
        ktrace(3, hmode);
        __syncthreads();
        ktrace(4, hmode);
        for (int i = tid; i < kW; i += kSThreads)
            reinterpret_cast<unsigned long long*>(ctl.st)[i] = reinterpret_cast<const unsigned long long*>(sst)[i];
        ktrace(5, hmode);
        if (ctl.host_st && (decision >= 0 || sst->incomplete)) status_to_host(sst, ctl.host_st);
        ktrace(30, hmode);
        // a begin's sums: its copies folded into copy 0 (off the critical path for a speculative begin)
        if (ctl.sums && ctl.mode == 1)
            fold_sum_copies(ctl.sums + static_cast<uint64_t>(sst->sum_sel) * ctl.sum_half, kfull, n);
        // fused exact-sum update: the next round's centroids when the loop goes on
        if (ctl.sum_fuse && !sst->stop && !sst->state_error) {
            __syncthreads();  // (the accept's staging area is free: the loop goes on)
            if (16384 + static_cast<size_t>(kfull) * n * 8 <= reuse_bytes)
                centroids_from_sums_ilp(ctl.sums + static_cast<uint64_t>(sst->sum_sel) * ctl.sum_half, kfull, n,
                                        ctl.sum_unscale, ctl.cC, ctl.cmask, ctl.cCact, ctl.cldc, ctl.cact,
                                        ctl.cn_active, ctl.cCT32, ctl.cdelta, reinterpret_cast<long long*>(&S.cand[0]),
                                        &S.icount[0], reinterpret_cast<double*>(reuse + 16384));
            else
                centroids_fused(ctl, sst->sum_sel, kfull, n, reinterpret_cast<long long*>(&S.cand[0]), &S.icount[0]);
        }
        if (tid == 0) klog_end(10 + hmode);
        return;
    }
}

// ---------------------------------------------------------------------------
// 3d. Final full-data pass (big_means.cpp:102-107: assign_nearest over all m
// rows), throughput form.  Same certified screen and exact recheck as
// k_assign_tma (identical labels and distances, bit for bit), organised for
// HBM streaming instead of latency: persistent CTAs (2 per SM) walk their
// 128-point blocks through ONE continuous TMA ring of 16-dim slabs (kFS
// stages), so the next block's slabs are in flight while the current block
// does its bounds, candidates and exact rechecks; the fp32 centroids and their
// norms are staged once per CTA.  Rows up to kFMaxD dims; the tile partials of
// block_sum come from k_tile_sums afterwards.
// ---------------------------------------------------------------------------
constexpr int kFMaxD = 80;  // dims of the streaming final pass (5 slabs; c1-c3)
template <typename T>
struct FinalSmem {
    static constexpr int kNS = sizeof(T) == 4 ? 4 : 3;           // ring stages
    static constexpr int kRawBytes = kABP * kADC * sizeof(T);   // one swizzled slab
    alignas(1024) unsigned char raw[kNS][kRawBytes];
    // fp32 points [d][p]: the whole block (exact copies of fp32 storage, so the
    // exact recheck reads its rows from here; fp64 storage rechecks from L2)
    alignas(16) float xs[kFMaxD][kABP];
    alignas(16) float ct[kFMaxD][kSMaxK];                       // fp32 centroids [d][j]
    float red_u[8][kABP];
    float nx_lo[kABP], nx_hi[kABP], nxr[kABP];
    float nc_lo[kSMaxK], nc_hi[kSMaxK], ncr[kSMaxK];
    unsigned cand[kABP];
    int icount[kABP];
    double item_d[kItemCap];
    short item_p[kItemCap];
    signed char item_j[kItemCap];
    uint64_t bar[kNS];
    uint32_t n_items;
};

template <typename T>
constexpr size_t final_smem_bytes() { return sizeof(FinalSmem<T>) + 1024; }

template <typename T>
__global__ void __launch_bounds__(kSThreads, 2)
k_final(const __grid_constant__ CUtensorMap tmx, const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
        const double* __restrict__ Cact, int ldc, const int* __restrict__ act_idx, const int* __restrict__ n_active_ptr,
        const float* __restrict__ CT32, int32_t* __restrict__ labels_out, double* __restrict__ dists_out,
        unsigned long long* __restrict__ cand_counter, ScreenConsts cst) {
    extern __shared__ __align__(16) unsigned char fsm_raw[];
    unsigned char* fsm_al = fsm_raw + ((1024u - (smem_u32(fsm_raw) & 1023u)) & 1023u);
    FinalSmem<T>& S = *reinterpret_cast<FinalSmem<T>*>(fsm_al);
    constexpr int NS = FinalSmem<T>::kNS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KA = *n_active_ptr;
    const int KG = (KA + kAK - 1) / kAK;
    const bool comp = warp < KG;
    const bool normw = warp == 7;
    const float finf = __int_as_float(0x7F800000);
    const int nslab = (n + kADC - 1) / kADC;
    const uint64_t nblk_all = (rows + kABP - 1) / kABP;
    const uint64_t my_blocks = blockIdx.x < nblk_all ? (nblk_all - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t total_q = my_blocks * nslab;  // slabs this CTA streams, in order
    auto issue = [&](uint64_t q) {               // thread 0: slab q of this CTA's sequence
        const int st = static_cast<int>(q % NS);
        const uint64_t b = blockIdx.x + (q / nslab) * gridDim.x;
        const int sl = static_cast<int>(q % nslab);
        mbar_expect_tx(&S.bar[st], FinalSmem<T>::kRawBytes);
        tma_load_2d(S.raw[st], &tmx, &S.bar[st], sl * kADC, static_cast<int>(b * kABP));
    };
    if (tid == 0) {
        tma_prefetch_map(&tmx);
        for (int i = 0; i < NS; ++i) mbar_init(&S.bar[i], 1);
        fence_mbar_init();
        for (uint64_t q = 0; q < static_cast<uint64_t>(NS) && q < total_q; ++q) issue(q);
    }
    // the fp32 centroids [d][j] and their norms (rounded down / up), once
    for (int e = tid; e < n * kSMaxK; e += kSThreads) S.ct[e / kSMaxK][e % kSMaxK] = CT32[e];
    __syncthreads();
    if (tid < kSMaxK) {
        float ncl = 0.f, nch = 0.f;
        for (int d = 0; d < n; ++d) {
            const float c = S.ct[d][tid];
            ncl = __fmaf_rd(c, c, ncl);
            nch = __fmaf_ru(c, c, nch);
        }
        S.nc_lo[tid] = ncl;
        S.nc_hi[tid] = nch;
        S.ncr[tid] = __fsqrt_ru(nch);
    }
    __syncthreads();
    uint64_t q = 0;
    const int cp_ = tid & (kABP - 1), chalf = tid >> 7;  // conversion: point, 8-dim half
    for (uint64_t bi = 0; bi < my_blocks; ++bi) {
        __syncthreads();  // the previous block's rows in xs are no longer read
        const uint64_t p0 = (blockIdx.x + bi * gridDim.x) * kABP;
        const int np = static_cast<int>(min(static_cast<uint64_t>(kABP), rows - p0));
        float2 tot[2][kAK];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < kAK; ++u) tot[h][u] = make_float2(0.f, 0.f);
        float nxl[4] = {0.f, 0.f, 0.f, 0.f}, nxh[4] = {0.f, 0.f, 0.f, 0.f};
        for (int sl = 0; sl < nslab; ++sl, ++q) {
            const int st = static_cast<int>(q % NS);
            const int d0 = sl * kADC;
            const int dl = min(kADC, n - d0);
            mbar_wait(&S.bar[st], static_cast<unsigned>((q / NS) & 1));
            float(*xsl)[kABP] = &S.xs[d0];
            convert_slab_part<T>(S.raw[st], xsl, cp_, chalf);
            __syncthreads();  // slab converted; stage st is free
            if (tid == 0 && q + NS < total_q) issue(q + NS);
            if (comp) {
                float2 part[2][kAK];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int u = 0; u < kAK; ++u) part[h][u] = make_float2(0.f, 0.f);
                auto step = [&](int d) {
                    const float4 xv = *reinterpret_cast<const float4*>(&xsl[d][4 * lane]);
                    const float4 cv = *reinterpret_cast<const float4*>(&S.ct[d0 + d][4 * warp]);
                    const float2 xa = make_float2(xv.x, xv.y), xb2 = make_float2(xv.z, xv.w);
                    part[0][0] = ffma2(xa, cv.x, part[0][0]);
                    part[0][1] = ffma2(xa, cv.y, part[0][1]);
                    part[0][2] = ffma2(xa, cv.z, part[0][2]);
                    part[0][3] = ffma2(xa, cv.w, part[0][3]);
                    part[1][0] = ffma2(xb2, cv.x, part[1][0]);
                    part[1][1] = ffma2(xb2, cv.y, part[1][1]);
                    part[1][2] = ffma2(xb2, cv.z, part[1][2]);
                    part[1][3] = ffma2(xb2, cv.w, part[1][3]);
                };
                if (dl == kADC) {
#pragma unroll
                    for (int d = 0; d < kADC; ++d) step(d);
                } else {
                    for (int d = 0; d < dl; ++d) step(d);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int u = 0; u < kAK; ++u) tot[h][u] = fadd2(tot[h][u], part[h][u]);
            }
            if (normw) {
                for (int d = 0; d < dl; ++d) {
                    const float4 xv = *reinterpret_cast<const float4*>(&xsl[d][4 * lane]);
                    nxl[0] = __fmaf_rd(xv.x, xv.x, nxl[0]); nxh[0] = __fmaf_ru(xv.x, xv.x, nxh[0]);
                    nxl[1] = __fmaf_rd(xv.y, xv.y, nxl[1]); nxh[1] = __fmaf_ru(xv.y, xv.y, nxh[1]);
                    nxl[2] = __fmaf_rd(xv.z, xv.z, nxl[2]); nxh[2] = __fmaf_ru(xv.z, xv.z, nxh[2]);
                    nxl[3] = __fmaf_rd(xv.w, xv.w, nxl[3]); nxh[3] = __fmaf_ru(xv.w, xv.w, nxh[3]);
                }
            }
        }
        if (normw) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                S.nx_lo[4 * lane + qq] = nxl[qq];
                S.nx_hi[4 * lane + qq] = nxh[qq];
                S.nxr[4 * lane + qq] = __fsqrt_ru(nxh[qq]);
            }
        }
        if (tid < kABP) S.cand[tid] = 0u;
        __syncthreads();
        // certified bounds (as k_assign_tma): upper bounds first, then each warp
        // tests its lower bounds against the point's minimum U
        float Lk[4][kAK];
        if (comp) {
            float un[4] = {finf, finf, finf, finf};
#pragma unroll
            for (int u = 0; u < kAK; ++u) {
                const int j = kAK * warp + u;
                const float cl = j < KA ? S.nc_lo[j] : 0.f, ch = j < KA ? S.nc_hi[j] : 0.f;
                const float crr = j < KA ? S.ncr[j] : 0.f;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const int p = 4 * lane + qq;
                    const float sdot = qq & 1 ? tot[qq >> 1][u].y : tot[qq >> 1][u].x;
                    const float t2 = 2.f * sdot;
                    const float Sn = __fadd_ru(S.nxr[p], crr);
                    const float Al = __fadd_rd(S.nx_lo[p], cl), Ah = __fadd_ru(S.nx_hi[p], ch);
                    float L = 0.f, U = finf;
                    if (fabsf(t2) <= 1.0e37f && Sn <= 1.0e18f && Ah <= 1.0e37f) {
                        const float D = __fadd_ru(__fmul_ru(__fmul_ru(cst.K, Sn), Sn), cst.dabs);
                        L = fmaxf(__fsub_rd(__fsub_rd(Al, t2), D), 0.f);
                        L = __fmul_rd(L, cst.lo64);
                        U = __fmul_ru(__fadd_ru(__fsub_ru(Ah, t2), D), cst.hi64);
                    }
                    Lk[qq][u] = j < KA ? L : finf;
                    if (j < KA) un[qq] = fminf(un[qq], U);
                }
            }
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) S.red_u[warp][4 * lane + qq] = un[qq];
        }
        __syncthreads();
        if (comp) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int p = 4 * lane + qq;
                float m = finf;
                for (int g = 0; g < KG; ++g) m = fminf(m, S.red_u[g][p]);
                unsigned bits = 0;
#pragma unroll
                for (int u = 0; u < kAK; ++u)
                    if (kAK * warp + u < KA && Lk[qq][u] <= m) bits |= 1u << (kAK * warp + u);
                if (bits && p < np) atomicOr(&S.cand[p], bits);
            }
        }
        __syncthreads();
        if (tid < 32) {  // exclusive scan of the candidate counts -> item offsets
            int v[4], run = 0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                v[qq] = __popc(S.cand[4 * tid + qq]);
                run += v[qq];
            }
            int incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (tid >= o) incl += y;
            }
            int ex = incl - run;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                S.icount[4 * tid + qq] = ex;
                ex += v[qq];
            }
            if (tid == 31) {
                S.n_items = static_cast<uint32_t>(incl);
                if (cand_counter) {
                    atomicAdd(cand_counter, static_cast<unsigned long long>(incl));
                    atomicAdd(cand_counter + 1, static_cast<unsigned long long>(np));
                }
            }
        }
        __syncthreads();
        const uint32_t NI = S.n_items;
        const bool overflow = NI > static_cast<uint32_t>(kItemCap);
        // exact fp64 recheck of the candidates (core.cpp:142-146), rows from L2
        if (!overflow) {
            if (tid < np) {
                uint32_t it = S.icount[tid];
                unsigned bits = S.cand[tid];
                while (bits) {  // ascending j
                    const int j = __ffs(bits) - 1;
                    bits &= bits - 1;
                    S.item_p[it] = static_cast<short>(tid);
                    S.item_j[it] = static_cast<signed char>(j);
                    ++it;
                }
            }
            __syncthreads();
            for (uint32_t i = tid; i < NI; i += kSThreads) {
                const int p = S.item_p[i];
                const double* c = Cact + static_cast<uint64_t>(S.item_j[i]) * ldc;
                if constexpr (sizeof(T) == 4) {  // the row from shared memory (exact fp32 copies)
                    double a = 0.0;
                    int d = 0;
#pragma unroll 4
                    for (; d + 2 <= n; d += 2) {
                        const double2 cv = __ldg(reinterpret_cast<const double2*>(c + d));
                        a = dist_step(a, S.xs[d][p], cv.x);
                        a = dist_step(a, S.xs[d + 1][p], cv.y);
                    }
                    for (; d < n; ++d) a = dist_step(a, S.xs[d][p], c[d]);
                    S.item_d[i] = a;
                } else {
                    S.item_d[i] = exact_row_dist(X + (p0 + p) * ld, c, n);
                }
            }
            __syncthreads();
        }
        if (tid < np) {
            const int p = tid;
            const uint64_t gp = p0 + p;
            double best = __longlong_as_double(0x7FF0000000000000LL);
            int bj = -1;
            if (!overflow) {  // ascending j, strict < (core.cpp:147)
                const uint32_t b1 = p + 1 < np ? static_cast<uint32_t>(S.icount[p + 1]) : NI;
                for (uint32_t i = S.icount[p]; i < b1; ++i) {
                    if (S.item_d[i] < best) {
                        best = S.item_d[i];
                        bj = S.item_j[i];
                    }
                }
            } else {  // candidate sets too large for the item buffer: full exact scan
                const T* x = X + gp * ld;
                for (int j = 0; j < KA; ++j) {
                    const double* c = Cact + static_cast<uint64_t>(j) * ldc;
                    double sm = 0.0;
                    for (int d = 0; d < n; ++d) sm = dist_step(sm, to_f64(x[d]), c[d]);
                    if (sm < best) {
                        best = sm;
                        bj = j;
                    }
                }
            }
            labels_out[gp] = bj >= 0 ? act_idx[bj] : -1;
            dists_out[gp] = best;
        }
        __syncthreads();  // cand / icount / items of this block consumed
    }
}

template <typename T, int NS = 2>
constexpr size_t tma_smem_bytes() { return sizeof(TmaSmem<T, NS>) + 1024; }

}  // namespace dev
}  // namespace bm
