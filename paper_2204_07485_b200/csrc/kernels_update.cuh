// kernels_update.cuh — per-tile sums, the ordered centroid update and the accept / chain-state kernels.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

// ===========================================================================
// 4. Per-tile sequential sums (block_sum inner loop core.cpp:167-173).
//    One warp per (array, tile); lanes stage 32 values, all lanes fold them in
//    index order (redundantly), lane 0 writes.
// ===========================================================================
__global__ void k_tile_sums(const double* __restrict__ v, uint64_t count, uint64_t stride,
                            int narrays, double* __restrict__ tiles, const int* __restrict__ stop_ptr) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    // one CTA per (array, tile): coalesced staging, then a single-thread fold
    __shared__ __align__(16) double sm[kTile];
    if (stop_ptr && *stop_ptr) return;
    const uint64_t ntiles = (count + kTile - 1) / kTile;
    const uint64_t a = blockIdx.x / ntiles, t = blockIdx.x % ntiles;
    const double* src = v + a * stride + t * kTile;
    const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), count - t * kTile));
    for (int i = threadIdx.x; i < len; i += blockDim.x) sm[i] = src[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    double acc = 0.0;
    int i = 0;
    for (; i + 8 <= len; i += 8) {
        const double2 v0 = *reinterpret_cast<const double2*>(sm + i);
        const double2 v1 = *reinterpret_cast<const double2*>(sm + i + 2);
        const double2 v2 = *reinterpret_cast<const double2*>(sm + i + 4);
        const double2 v3 = *reinterpret_cast<const double2*>(sm + i + 6);
        acc = __dadd_rn(acc, v0.x); acc = __dadd_rn(acc, v0.y);
        acc = __dadd_rn(acc, v1.x); acc = __dadd_rn(acc, v1.y);
        acc = __dadd_rn(acc, v2.x); acc = __dadd_rn(acc, v2.y);
        acc = __dadd_rn(acc, v3.x); acc = __dadd_rn(acc, v3.y);
    }
    for (; i < len; ++i) acc = __dadd_rn(acc, sm[i]);
    tiles[a * ntiles + t] = acc;
}


// ===========================================================================
// 5. Centroid update (update_centroids core.cpp:183-244), bit-exact order,
//    one kernel, grid (tile, d-slab).
//
// Per CTA: stable bucketing of the tile's points by label (warp-synchronous,
// index order preserved); the tile's coordinate slab staged in shared memory
// with coalesced loads; one thread per (label, dim) folds its members'
// coordinates in index order from 0.0 — the reference's per-block partial
// row[d] += x[d] (:206-214) — into psum (+0.0 when the label is absent).
// The CTA that completes a slab (arrival counter) merges it: one thread per
// (label, dim) folds the tile partials in tile order (:217-229; absent labels
// add +0.0 to a sum that is never -0.0, the identity), then sum * (1.0/count)
// (:237-239); count 0 -> degenerate row of 0.0 (:231 all_degenerate).  The
// merge also writes the compacted centroids (Cact, CT32), the active list and
// the squared movement per label of this slab (bounds of the next assignment).
// ===========================================================================
constexpr int kUThreads = 256;
constexpr int kUWarps = kUThreads / 32;
constexpr int kUChunks = kTile / 32;  // 32-point chunks per tile

struct UpdateArgs {
    double* psum;            // [n][k][tstride]: tile partials, contiguous per (dim, label)
    uint64_t tstride;        // tiles rounded up to even
    uint64_t shm_bytes;      // dynamic shared memory of the launch (the merge streams partials through it)
    unsigned* slab_ctr;      // [slabs] arrival counters (reset by the last merger)
    unsigned* slab_done;     // [slabs] mergers finished
    int mergers;             // G: CTAs merging each slab
    const int* go;           // when set and *go == 0 the launch does nothing (skipped chunk)
    unsigned* all_done;      // mergers finished (all slabs)
    float* delta;            // [k] movement per label of this update (rounded up)
    unsigned* slab_tot;      // [slabs][k] label totals (reset by the merging CTA)
    double* C;               // [k][n]
    uint8_t* mask;
    double* Cact;
    int ldc;
    int* act_idx;
    int* n_active;
    float* CT32;
    double* drift_part;      // [slabs][k] squared movement of this slab's dims
    int* bad_label;
    const int* stop;
};

template <typename T>
__global__ void __launch_bounds__(kUThreads)
k_update(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
         const int32_t* __restrict__ labels_pair, uint64_t pair_stride,
         const int* __restrict__ parity_ptr, int k, int dslab, UpdateArgs u) {
    klog_start(2);
    pdl_wait();
    if (u.stop && *u.stop) return;
    if (u.go && !*u.go) return;
    extern __shared__ __align__(16) unsigned char ush_raw[];
    ktrace_u(0);
    int* ush = reinterpret_cast<int*>(ush_raw);
    short* order = reinterpret_cast<short*>(ush);      // [kTile]
    int* cnt = ush + kTile / 2;                         // [k] tile totals
    int* off = cnt + k;                                 // [k] label offsets in `order`
    int* wcount = off + k;                              // [warps][k] per-warp counts -> bases
    T* xs = reinterpret_cast<T*>(ush_raw + ((static_cast<size_t>(kTile / 2 + (2 + kUWarps) * k) * 4 + 15) & ~size_t(15)));

    const int32_t* labels = labels_pair + (parity_ptr ? (*parity_ptr) * pair_stride : 0);
    const uint64_t tile = blockIdx.x, ntiles = gridDim.x;
    const uint64_t b = tile * kTile;
    const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), rows - b));
    const int slab = blockIdx.y;
    const int d0 = slab * dslab;
    const int dl = min(n, d0 + dslab) - d0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // stage the coordinate slab with 16-byte cp.async (independent of the
    // bucketing; dslab, d0 and ld are multiples of 16 bytes / sizeof(T))
    constexpr int kV = 16 / sizeof(T);
    const int dv = (dl + kV - 1) / kV, dlp = dv * kV;  // padded row of the staged slab
    {
        const T* Xt = X + b * ld + d0;
        for (int e = threadIdx.x; e < len * dv; e += blockDim.x) {
            const int p = e / dv, v = e - p * dv;
            cp_async_16(xs + p * dlp + v * kV, Xt + static_cast<uint64_t>(p) * ld + v * kV);
        }
        cp_async_commit();
    }
    for (int e = threadIdx.x; e < kUWarps * k; e += blockDim.x) wcount[e] = 0;
    __syncthreads();
    ktrace_u(1);
    // Stable bucketing.  Warp w owns the contiguous points [128 w, 128 w + 128)
    // as 4 chunks of 32 in index order; per chunk __match_any_sync gives each
    // point its rank among equal labels, and the label's running count in the
    // warp (kept by the group leader) gives the chunk's base.
    constexpr int kQ = kUChunks / kUWarps;
    int lab_r[kQ], pos_r[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const int i = (warp * kQ + q) * 32 + lane;
        int l = -1 - lane;
        if (i < len) {
            l = labels[b + i];
            if (l < 0 || l >= k) {  // update_centroids label range check (core.cpp:189-193)
                *u.bad_label = 1;
                l = 0;
            }
        }
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, l);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (i < len && lane == leader) {
            base = wcount[warp * k + l];
            wcount[warp * k + l] = base + __popc(peers);
        }
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        lab_r[q] = l;
        pos_r[q] = base + __popc(peers & ((1u << lane) - 1u));
        __syncwarp();
    }
    __syncthreads();
    ktrace_u(2);
    // exclusive prefix over the warps per label; tile totals
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        int r = 0;
#pragma unroll
        for (int w = 0; w < kUWarps; ++w) {
            const int v = wcount[w * k + j];
            wcount[w * k + j] = r;
            r += v;
        }
        cnt[j] = r;
        if (r) atomicAdd(&u.slab_tot[slab * k + j], static_cast<unsigned>(r));
    }
    __syncthreads();
    if (warp == 0) {  // label offsets: exclusive scan of the totals
        int carry = 0;
        for (int j0 = 0; j0 < k; j0 += 32) {
            const int j = j0 + lane;
            const int v = j < k ? cnt[j] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            if (j < k) off[j] = carry + incl - v;
            carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
    }
    __syncthreads();
    ktrace_u(3);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const int i = (warp * kQ + q) * 32 + lane;
        if (i < len) order[off[lab_r[q]] + wcount[warp * k + lab_r[q]] + pos_r[q]] = static_cast<short>(i);
    }
    cp_async_wait<0>();
    __syncthreads();
    ktrace_u(4);
    for (int e = threadIdx.x; e < k * dl; e += blockDim.x) {
        const int j = e / dl, dd = e - j * dl;
        const int c = cnt[j];
        const short* ord = order + off[j];
        double acc = 0.0;
        int q = 0;
        for (; q + 8 <= c; q += 8) {
            double v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = to_f64(xs[ord[q + r] * dlp + dd]);
#pragma unroll
            for (int r = 0; r < 8; ++r) acc = __dadd_rn(acc, v[r]);
        }
        for (; q < c; ++q) acc = __dadd_rn(acc, to_f64(xs[ord[q] * dlp + dd]));
        u.psum[(static_cast<uint64_t>(d0 + dd) * k + j) * u.tstride + tile] = acc;
    }

    // ---- the last G CTAs of this slab merge it, pairs g, g + G, ... each ----
    // (they wait for the slab's other CTAs: those hold no resources the
    // waiting ones need, so they always complete)
    __shared__ int mg;
    __threadfence();
    __syncthreads();
    ktrace_u(5);
    const int G = u.mergers;
    if (threadIdx.x == 0) {
        const int a = static_cast<int>(atomicAdd(&u.slab_ctr[slab], 1u));
        mg = a - (static_cast<int>(ntiles) - G);
        if (mg >= 0)
            while (__ldcg(&u.slab_ctr[slab]) < ntiles) __nanosleep(64);
    }
    __syncthreads();
    if (mg < 0) return;
    __threadfence();
    ktrace_u(6);
    // reuse the shared memory: totals, ranks, squared movements, staged partials
    int* tot = ush;                                          // [k]
    int* rank = tot + k;                                     // [k]
    const size_t o_sq = (static_cast<size_t>(2 * k) * 4 + 15) & ~size_t(15);
    double* sq = reinterpret_cast<double*>(ush_raw + o_sq);  // [k] this merger's movement per label
    const size_t o_m = (o_sq + static_cast<size_t>(k) * 8 + 15) & ~size_t(15);
    double* mbuf = reinterpret_cast<double*>(ush_raw + o_m);
    const int mstride = static_cast<int>(u.tstride) + 1;     // odd: conflict-free folds
    const int cap = static_cast<int>((u.shm_bytes - o_m) / (static_cast<size_t>(mstride) * 8));
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        tot[j] = static_cast<int>(__ldcg(&u.slab_tot[slab * k + j]));
        sq[j] = 0.0;
    }
    __syncthreads();
    ktrace_u(7);
    if (threadIdx.x == 0) {
        int r = 0;
        for (int j = 0; j < k; ++j) {
            rank[j] = tot[j] ? r : -1;
            if (slab == 0 && mg == 0) {
                u.mask[j] = tot[j] ? 0 : 1;
                if (tot[j]) u.act_idx[r] = j;
            }
            r += tot[j] != 0;
        }
        if (slab == 0 && mg == 0) *u.n_active = r;
    }
    // This merger's pairs (dim, label) = q G + mg; each pair's tile partials are
    // contiguous in psum: staged through shared memory with cp.async (a warp per
    // pair), then one thread per pair folds them in tile order.
    const int npairs = k * dl;
    const int mine = npairs > mg ? (npairs - mg + G - 1) / G : 0;
    const double* src = u.psum + static_cast<uint64_t>(d0) * k * u.tstride;
    for (int q0 = 0; q0 < mine; q0 += cap) {
        const int nq = min(cap, mine - q0);
        for (int pl = warp; pl < nq; pl += kUWarps) {
            const double* sp = src + static_cast<uint64_t>((q0 + pl) * G + mg) * u.tstride;
            for (int t = lane; t < static_cast<int>(ntiles); t += 32) cp_async_el(mbuf + pl * mstride + t, sp + t, 8);
        }
        cp_async_commit_wait_all();
        __syncthreads();
        if (q0 == 0) ktrace_u(9);
        for (int e = threadIdx.x; e < nq; e += blockDim.x) {
            const int pair = (q0 + e) * G + mg;
            const int j = pair % k, d = d0 + pair / k;
            const uint64_t ce = static_cast<uint64_t>(j) * n + d;
            if (tot[j] == 0) {
                u.C[ce] = 0.0;
                continue;
            }
            const double* mp = mbuf + static_cast<uint64_t>(e) * mstride;
            double acc = 0.0;
            for (int t = 0; t < static_cast<int>(ntiles); ++t) acc = __dadd_rn(acc, mp[t]);
            const double inv = __ddiv_rn(1.0, static_cast<double>(tot[j]));
            const double v = __dmul_rn(acc, inv);
            const double dv = __dsub_rn(v, u.C[ce]);
            atomicAdd(&sq[j], __dmul_rn(dv, dv));  // order-free: only bounds use it
            u.C[ce] = v;
            const int rk = rank[j];
            u.Cact[static_cast<uint64_t>(rk) * u.ldc + d] = v;
            if (u.CT32 && rk < kSMaxK) u.CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v);
        }
        __syncthreads();
        if (q0 == 0) ktrace_u(10);
    }
    ktrace_u(8);
    if (u.drift_part)
        for (int j = threadIdx.x; j < k; j += blockDim.x) u.drift_part[(slab * G + mg) * k + j] = sq[j];
    // the last merger to finish resets the slab's counters for the next launch
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&u.slab_done[slab], 1u) == static_cast<unsigned>(G) - 1) {
        for (int j = 0; j < k; ++j) u.slab_tot[slab * k + j] = 0u;
        u.slab_done[slab] = 0u;
        __threadfence();
        u.slab_ctr[slab] = 0u;
    }
    // the very last merger turns the parts into each label's movement (distance
    // units, rounded up with margin: only bounds use it)
    __shared__ int lastm;
    if (threadIdx.x == 0) lastm = atomicAdd(u.all_done, 1u) == static_cast<unsigned>(G) * gridDim.y - 1;
    __syncthreads();
    if (!lastm) return;
    __threadfence();
    const int parts = G * static_cast<int>(gridDim.y);
    // all parts staged in one round trip (not one per label), when they fit
    double* dp = reinterpret_cast<double*>(ush_raw + o_m);
    const bool staged = static_cast<size_t>(parts) * k * 8 <= u.shm_bytes - o_m;
    if (staged) {
        for (int i = threadIdx.x; i < parts * k; i += blockDim.x) dp[i] = __ldcg(u.drift_part + i);
        __syncthreads();
    }
    for (int j = warp; j < k; j += kUWarps) {  // a warp per label, lanes over the parts (any order)
        double sj = 0.0;
        for (int q = lane; q < parts; q += 32) sj += staged ? dp[q * k + j] : __ldcg(&u.drift_part[q * k + j]);
#pragma unroll
        for (int o = 16; o; o >>= 1) sj += __shfl_xor_sync(0xFFFFFFFFu, sj, o);
        if (lane == 0) u.delta[j] = __double2float_ru(__dsqrt_ru(sj * (1.0 + 1e-12)) * (1.0 + 1e-12) + 1e-300);
    }
    if (threadIdx.x == 0) {
        *u.all_done = 0u;
        klog_end(2);
    }
}

// Compact the active rows of (C, mask) for the assignment (single CTA).
__global__ void k_compact(const double* __restrict__ C, const uint8_t* __restrict__ mask, int k, int n,
                          double* __restrict__ Cact, int ldc, int* __restrict__ act_idx, int* __restrict__ n_active,
                          float* __restrict__ CT32) {
    extern __shared__ int csh[];
    for (int j = threadIdx.x; j < k; j += blockDim.x) csh[j] = mask[j];  // staged: the rank loop is serial
    __syncthreads();
    if (threadIdx.x == 0) {
        int r = 0;
        for (int j = 0; j < k; ++j) {
            const bool deg = csh[j] != 0;
            csh[j] = deg ? -1 : r;
            if (!deg) act_idx[r++] = j;
        }
        *n_active = r;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * n; e += blockDim.x) {
        const int j = e / n;
        if (csh[j] >= 0) {
            Cact[static_cast<uint64_t>(csh[j]) * ldc + (e % n)] = C[e];
            if (CT32 && csh[j] < kSMaxK) CT32[static_cast<uint64_t>(e % n) * kSMaxK + csh[j]] = __double2float_rn(C[e]);
        }
    }
}

// Exact-sum mode update as its own launch (the unfused form, BM_SUMS_FUSE=0).
__global__ void __launch_bounds__(1024)
k_centroids(const LloydStatus* __restrict__ st, const int* __restrict__ stop, const int* __restrict__ go,
            const long long* __restrict__ sums, uint64_t sum_half, double unscale, int k, int n,
            double* __restrict__ C, uint8_t* __restrict__ mask, double* __restrict__ Cact, int ldc,
            int* __restrict__ act_idx, int* __restrict__ n_active, float* __restrict__ CT32, float* __restrict__ delta) {
    klog_start(1);
    pdl_wait();
    if (stop && *stop) return;
    if (go && !*go) return;
    __shared__ long long tot[kSMaxK];
    __shared__ int rank[kSMaxK];
    centroids_from_sums(sums + static_cast<uint64_t>(st->sum_sel) * sum_half, k, n, unscale, C, mask, Cact, ldc,
                        act_idx, n_active, CT32, delta, tot, rank);
    if (threadIdx.x == 0) klog_end(1);
}

// ===========================================================================
// 7. Accept (big_means.cpp:89-94) on the device.
// ===========================================================================
// rec_base[*chunk_ctr] receives the record; the chunk counter and the
// incumbent's degenerate count (the next chunk's `repaired`, :83) live on the
// device so the chunk can run inside a CUDA graph.  The incumbent is also
// written in compacted form (Cact/act/n_active/CT32): it is the next chunk's
// start (:82) when no repair is needed.
__global__ void k_accept(LloydStatus* st, AcceptArgs A, LloydStatus* host_st) {
    extern __shared__ int asm_[];  // [2k]
    __shared__ int accepted;
    klog_start(3);
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) accepted = st->objective < *A.f_opt;  // strict (:89)
    __syncthreads();
    accept_body(st, A, accepted, host_st, asm_);
    if (threadIdx.x == 0) klog_end(3);
}

// Head of a chunk's Lloyd graph: the chunk runs only when the previous accept
// left no degenerate incumbent rows, or the host has repaired them (st->go).
__global__ void k_guard(const GState* gs, cudaGraphConditionalHandle h) {
    klog_start(0);
    cudaGraphSetConditional(h, gs->go != 0 ? 1u : 0u);
    klog_end(0);
}

// The last chunk's record: its exact objective (graph mode, after the loop).
__global__ void k_fix_final(GState* gs, AcceptArgs A, const double* __restrict__ dists_all, uint64_t R,
                            double* __restrict__ tiles, unsigned* __restrict__ counter) {
    __shared__ __align__(16) double fbuf[kTile];
    __shared__ int last;
    const int pend = gs->pending_fix;
    if (pend < 0) return;
    const uint64_t tb = static_cast<uint64_t>(blockIdx.x) * kTile;
    const double* dv = dists_all + (3 * static_cast<uint64_t>(pend % kStateBufs) + gs->fix_par) * R + tb;
    const int len = static_cast<int>(min(static_cast<uint64_t>(kTile), R - tb));
    for (int i = threadIdx.x; i < len; i += blockDim.x) fbuf[i] = __ldcg(dv + i);
    __syncthreads();
    if (threadIdx.x == 0) {
        tiles[blockIdx.x] = seq_fold_smem(fbuf, len);
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
        if (last) {
            __threadfence();
            *counter = 0u;
            FixOut fx;
            if (fix_compute(gs, tiles, gridDim.x, &fx)) fix_commit(gs, A, fx);
        }
    }
}

__global__ void k_bump_version(GState* gs) { gs->inc_version += 1; }

// Reset of the per-run device state (incumbent all degenerate, f_opt = +inf).
__global__ void k_run_init(LloydStatus* st, int nst, GState* gs, double* f_opt, double* Cinc, uint8_t* maskinc,
                           double* C, uint8_t* mask, int k, int n, unsigned long long* chunk_ctr) {
    for (int e = threadIdx.x; e < k * n; e += blockDim.x) Cinc[e] = C[e] = 0.0;
    for (int j = threadIdx.x; j < k; j += blockDim.x) maskinc[j] = mask[j] = 1;
    if (threadIdx.x == 0) {
        *f_opt = __longlong_as_double(0x7FF0000000000000LL);
        for (int b = 0; b < nst; ++b) {
            st[b].inc_degenerate = k;
            st[b].stop = 1;  // a skipped chunk's rounds see a finished loop
            st[b].incomplete = 0;
            st[b].begin_version = -1;
        }
        gs->fopt_exact = __longlong_as_double(0x7FF0000000000000LL);
        gs->inc_version = 0;
        gs->n_active_inc = 0;
        gs->inc_degenerate = k;
        gs->go = 0;
        gs->pending_fix = -1;
        gs->fix_par = 0;
        *chunk_ctr = 0;
    }
}

}  // namespace dev
}  // namespace bm
