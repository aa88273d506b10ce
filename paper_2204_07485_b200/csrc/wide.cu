// wide.cu — tensor-core pre-screen of wide rows (the assignment screen of
// assign_nearest core.cpp:129-155 for rows too wide for the persistent chunk
// kernel: n > 88, fp32 storage, every value exact in tf32 — c5's integer rows).
//
// Why: the multi-launch assignment (k_assign_tma) walks a 128-point block's
// n dims in 16-dim slabs on ONE CTA; with s = 4000 rows (c5) that is 32 CTAs
// on 148 SMs, 313 serial slabs each.  Here the dot products x.c of a 128-point
// tile are split over KS CTAs along K (the dims) and computed on the tensor
// core: tcgen05.mma kind::tf32, M = 128 points, N = NP centroid slots, K = 8
// dims per step, one TMEM accumulator block per 32-dim atom (the blocked sum
// keeps the certified error bound tight).  Each CTA writes its split's partial
// dot products and partial squared norms; k_assign_tma (pre-screened mode)
// adds the KS partials in split order, forms the certified bounds, and runs
// its exact fp64 recheck as before — assign_nearest's result bit for bit.
//
// Error model (wide_screen_consts): with x exact in tf32 and fl32(c) = hi + lo
// (hi = tf32(c), lo exact; the MMA reads lo truncated to tf32, |error| <=
// 2^-21 |c|), products are exact except that truncation; each of the 2 x 32
// accumulations of an atom block loses < 2^-23 of the running magnitude; the
// atom blocks and then the splits are added in fp32 (round to nearest):
//   |dot - x^.c^| <= (2^-21 + 64 2^-23 + gamma_na + gamma_KS) sum_d |x^_d c^_d|,
// doubled as a safety margin (the same treatment as the chunk kernel's
// tensor-core screen).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"
#include "wide.h"

namespace bm {
namespace dev {

namespace {
constexpr unsigned kWAtomBytes = 16384; // 128 rows x 128 B
}  // namespace

// Shared memory: a ring of stages [A: 128 rows x 128 B][B: hi NP rows x 128 B][lo NP rows x 128 B], 1024-aligned.
__host__ __device__ constexpr int wide_stages(int np_) { return np_ == 16 ? 10 : 8; }
__host__ __device__ inline size_t wide_stage_bytes(int np_) { return kWAtomBytes + 2 * static_cast<size_t>(np_) * 128; }
__host__ __device__ inline size_t wide_smem_bytes(int np_) {
    return 1024 + static_cast<size_t>(wide_stages(np_)) * wide_stage_bytes(np_);
}

// k_wide_prep: the B operands of every 32-dim atom once per pass — rows = the
// compacted active centroids (0 past KA), K-major, 128-byte swizzle, fl32(c) =
// hi + lo (hi = tf32(c) rounded to nearest, lo exact) — and each atom's partial
// squared norms of fl32(c) (rounded down / up).  Grid: one CTA per atom.
template <int NP>
__global__ void __launch_bounds__(128) k_wide_prep(const __grid_constant__ WideArgs a) {
    pdl_wait();
    if ((a.stop && *a.stop) || (a.go && !*a.go)) return;
    const int tid = threadIdx.x, at = static_cast<int>(blockIdx.x);
    const int KA = *a.n_active;
    unsigned char* B = reinterpret_cast<unsigned char*>(a.bops) + static_cast<size_t>(at) * 2 * NP * 128;
    __shared__ float slo[NP][33], shi[NP][33];
    for (int e = tid; e < NP * 32; e += 128) {  // e = (row, dim)
        const int rk = e >> 5, dd = e & 31, d = at * 32 + dd;
        const double v = rk < KA && d < a.n ? __ldcg(a.Cact + static_cast<size_t>(rk) * a.ldc + d) : 0.0;
        const float f = __double2float_rn(v), hi = umma::tf32_rna(f);
        const size_t off = static_cast<size_t>(rk) * 128 + ((((dd >> 2) & 7) ^ (rk & 7)) << 4) + (dd & 3) * 4;
        *reinterpret_cast<float*>(B + off) = hi;
        *reinterpret_cast<float*>(B + off + NP * 128) = f - hi;
        slo[rk][dd] = f;
    }
    __syncthreads();
    if (tid < NP) {
        float lo = 0.f, hi = 0.f;
        for (int dd = 0; dd < 32; ++dd) {
            const float f = slo[tid][dd];
            lo = __fmaf_rd(f, f, lo);
            hi = __fmaf_ru(f, f, hi);
        }
        a.nc[(static_cast<size_t>(at) * NP + tid) * 2] = lo;
        a.nc[(static_cast<size_t>(at) * NP + tid) * 2 + 1] = hi;
    }
    (void)shi;
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     umma::smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(umma::smem_addr(bar))
                 : "memory");
}

// 160 threads: warps 0-3 consume the atoms (row tid's squared norm; thread 0
// issues the MMAs and commits them), warp 4's lane 0 produces them (the A box by
// TMA, the atom's B operands by a bulk copy).  A stage is free again once its
// 128 readers have arrived and its MMAs retired (empty barrier: 128 + 1 commit).
template <int NP>
__global__ void __launch_bounds__(160, 1) k_wide_screen(const __grid_constant__ WideArgs a) {
    extern __shared__ __align__(16) unsigned char wsm_raw[];
    constexpr int NS = wide_stages(NP);
    constexpr unsigned kB = 2 * NP * 128;                 // B bytes per atom (hi + lo)
    constexpr unsigned kStage = kWAtomBytes + kB;
    __shared__ __align__(8) unsigned long long s_full[NS], s_empty[NS];
    __shared__ unsigned s_tmem;
    pdl_wait();
    if ((a.stop && *a.stop) || (a.go && !*a.go)) return;  // a finished loop / a chunk that needs a repair
    const int tid = threadIdx.x, warp = tid >> 5;
    const unsigned tile = blockIdx.x, ks = blockIdx.y;
    const uint64_t p0 = static_cast<uint64_t>(tile) * 128;
    const int np = static_cast<int>(min(static_cast<uint64_t>(128), a.rows - p0));
    const int A0 = static_cast<int>(ks) * a.na;
    const int nA = min(a.na, a.natoms - A0);  // >= 1 (plan)
    unsigned char* stg = wsm_raw + ((1024u - (umma::smem_addr(wsm_raw) & 1023u)) & 1023u);
    constexpr unsigned kIdesc = umma::idesc_tf32<NP>();
    const int nblk = (nA + a.bpa - 1) / a.bpa;  // accumulator blocks
    const unsigned cols = umma::tmem_cols(static_cast<unsigned>(nblk) * NP);
    const bool producer = tid == 128;

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(reinterpret_cast<uint64_t*>(&s_full[i]), 1);
            mbar_init(reinterpret_cast<uint64_t*>(&s_empty[i]), 129);
        }
        fence_mbar_init();
    }
    __syncthreads();
#ifdef BM_WIDE_DBG
    auto stamp = [&](int slot, int t) {
        if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && t < 64) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            a.dbg[slot * 64 + t] = g;
        }
    };
#else
    auto stamp = [](int, int) {};
#endif
    auto load_atom = [&](int t) {
        stamp(0, t);
        const int s_ = t % NS;
        unsigned char* st = stg + static_cast<size_t>(s_) * kStage;
        uint64_t* bar = reinterpret_cast<uint64_t*>(&s_full[s_]);
        mbar_expect_tx(bar, kStage);
        tma_load_2d(st, &a.xmap, bar, (A0 + t) * 32, static_cast<int>(p0));
        bulk_g2s(st + kWAtomBytes, reinterpret_cast<const unsigned char*>(a.bops) + static_cast<size_t>(A0 + t) * kB, kB,
                 &s_full[s_]);
    };
    if (producer) {
        tma_prefetch_map(&a.xmap);
        for (int t = 0; t < NS && t < nA; ++t) load_atom(t);
    }
    if (warp == 0) umma::tmem_alloc(&s_tmem, cols);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const unsigned tbase = s_tmem;
    if (producer) {  // refill each stage as soon as its previous atom is consumed
        for (int t = NS; t < nA; ++t) {
            const int s_ = t % NS;
            umma::mbar_wait_parity(&s_empty[s_], ((t / NS) - 1) & 1);
            stamp(3, t - NS);  // atom t - NS consumed and its MMAs retired
            load_atom(t);
        }
    }
    if (tid < 128) {
        const unsigned us = umma::smem_addr(stg) >> 4;
        float nxl = 0.f, nxh = 0.f;  // this thread's row (point tid), this split's dims
        for (int t = 0; t < nA; ++t) {
            const int s_ = t % NS;
            mbar_wait(reinterpret_cast<uint64_t*>(&s_full[s_]), (t / NS) & 1);
            if (tid == 0) stamp(1, t);
            if (tid == 0) {  // the atom's MMAs: 8 dims (32 B) per step inside the swizzle atom
                umma::fence_after();
                const unsigned sa = us + static_cast<unsigned>(s_) * (kStage >> 4);
                const unsigned sbh = sa + (kWAtomBytes >> 4), sbl = sbh + (NP * 128 >> 4);
                const unsigned d_t = tbase + static_cast<unsigned>(t / a.bpa) * NP;  // this atom's accumulator block
                const bool first = t % a.bpa == 0;
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const unsigned long long da = umma::desc_sw128(sa + 2 * k4);
                    umma::mma_tf32(d_t, da, umma::desc_sw128(sbh + 2 * k4), kIdesc, !(first && k4 == 0));
                    umma::mma_tf32(d_t, da, umma::desc_sw128(sbl + 2 * k4), kIdesc, 1);
                }
                umma::commit(&s_empty[s_]);
                stamp(2, t);
            }
            {  // squared norm of row tid over the atom (swizzled 16-byte chunks; dims >= n are 0)
                const unsigned char* row = stg + static_cast<size_t>(s_) * kStage + static_cast<size_t>(tid) * 128;
                float4 v[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = *reinterpret_cast<const float4*>(row + ((c ^ (tid & 7)) << 4));
                mbar_arrive(&s_empty[s_]);  // this thread's reads of the stage are done
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    nxl = __fmaf_rd(v[c].x, v[c].x, nxl); nxh = __fmaf_ru(v[c].x, v[c].x, nxh);
                    nxl = __fmaf_rd(v[c].y, v[c].y, nxl); nxh = __fmaf_ru(v[c].y, v[c].y, nxh);
                    nxl = __fmaf_rd(v[c].z, v[c].z, nxl); nxh = __fmaf_ru(v[c].z, v[c].z, nxh);
                    nxl = __fmaf_rd(v[c].w, v[c].w, nxl); nxh = __fmaf_ru(v[c].w, v[c].w, nxh);
                }
            }
        }
        // the last atom's barrier phase completes after its (and so every) MMA retired
        umma::mbar_wait_parity(&s_empty[(nA - 1) % NS], ((nA - 1) / NS) & 1);
        umma::fence_after();
        // epilogue: this thread's row (warp w reads TMEM lanes 32w..32w+31), the
        // accumulator blocks added in block order (fp32, round to nearest)
        float dot[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) dot[j] = 0.f;
        const unsigned lrow = static_cast<unsigned>(32 * warp) << 16;
        for (int t = 0; t < nblk; ++t) {
            float v[NP];
            if constexpr (NP == 16) umma::tmem_ld16(tbase + lrow + static_cast<unsigned>(t) * NP, v);
            else umma::tmem_ld32(tbase + lrow + static_cast<unsigned>(t) * NP, v);
#pragma unroll
            for (int j = 0; j < NP; ++j) dot[j] = __fadd_rn(dot[j], v[j]);
        }
        if (tid < np) {
            const uint64_t gp = p0 + tid;
            float4* dst = reinterpret_cast<float4*>(a.dot + (static_cast<size_t>(ks) * a.rows + gp) * NP);
#pragma unroll
            for (int q = 0; q < NP / 4; ++q) dst[q] = make_float4(dot[4 * q], dot[4 * q + 1], dot[4 * q + 2], dot[4 * q + 3]);
            reinterpret_cast<float2*>(a.nx)[static_cast<size_t>(ks) * a.rows + gp] = make_float2(nxl, nxh);
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) {
        umma::fence_after();
        umma::tmem_dealloc(tbase, cols);
    }
}

// ---------------------------------------------------------------------------
// k_wide_recheck: 32 points per CTA (rows [32 b, 32 b + 32)), 128 threads.
namespace {
constexpr int kRP = 32;      // points per CTA
constexpr int kRT = 128;     // threads
constexpr int kRD = 32;      // dims per stage
constexpr int kRItems = 4 * kRT;  // items (point, candidate) per streaming round
}  // namespace

// RS stages of [32 rows x 32 dims] fp32 point pieces and [NPR rows x 32 dims]
// fp64 centroid pieces: 16 (NPR 16) or 12 (NPR 32) stages keep enough bytes in
// flight to cover the L2 / HBM latency with one CTA per SM
__host__ __device__ inline size_t wide_recheck_stage_bytes(int npr) {
    return static_cast<size_t>(kRP) * 128 + 2 * static_cast<size_t>(npr) * 128;  // x box + two centroid boxes
}
__host__ __device__ inline size_t wide_recheck_smem_bytes(int rs, int npr) {
    return 1024 + static_cast<size_t>(rs) * wide_recheck_stage_bytes(npr);
}

// 160 threads: warps 0-3 compute (the bounds of 32 points, then up to 4
// chains each per streaming round), warp 4's lane 0 streams the dims: step g
// (round g / nsteps, dims 32 (g % nsteps) ..) into stage g % kRS by TMA; a
// stage is refilled once its 128 readers have arrived (no block barrier per step).
template <int kRS, int NPR>
__global__ void __launch_bounds__(kRT + 32) k_wide_recheck(const __grid_constant__ RecheckArgs a) {
    extern __shared__ __align__(16) unsigned char rsm[];
    __shared__ float ncl[32], nch[32], ncr[32];
    __shared__ unsigned cand[kRP];
    __shared__ int icount[kRP + 1];
    __shared__ short item_p[kRP * 32];
    __shared__ signed char item_j[kRP * 32];
    __shared__ double item_d[kRP * 32];
    __shared__ __align__(8) unsigned long long s_full[kRS], s_empty[kRS];
    pdl_wait();
    if ((a.stop && *a.stop) || (a.go && !*a.go)) return;
    const int tid = threadIdx.x;
    const bool producer = tid == kRT;
    const uint64_t q0 = static_cast<uint64_t>(blockIdx.x) * kRP;
    const int np = static_cast<int>(min(static_cast<uint64_t>(kRP), a.rows - q0));
    const int KA = *a.n_active;
    const float finf = __int_as_float(0x7F800000);
    // stage: [x box: 32 rows x 128 B][centroid box dims 0-15: NPR rows x 128 B][dims 16-31], 128-byte swizzle
    unsigned char* stg = rsm + ((1024u - (umma::smem_addr(rsm) & 1023u)) & 1023u);
    constexpr unsigned kStage = static_cast<unsigned>(kRP * 128 + 2 * NPR * 128);
    const int nsteps = (a.n + kRD - 1) / kRD;
    if (tid == 0) {
        for (int i = 0; i < kRS; ++i) {
            mbar_init(reinterpret_cast<uint64_t*>(&s_full[i]), 1);
            mbar_init(reinterpret_cast<uint64_t*>(&s_empty[i]), kRT);
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int g) {  // global step g (producer only)
        const int st = g % kRS, d0 = (g % nsteps) * kRD;
        unsigned char* b = stg + static_cast<size_t>(st) * kStage;
        uint64_t* bar = reinterpret_cast<uint64_t*>(&s_full[st]);
        mbar_expect_tx(bar, kStage);
        tma_load_2d(b, &a.xmap, bar, d0, static_cast<int>(q0));
        tma_load_2d(b + kRP * 128, &a.cmap, bar, d0, 0);
        tma_load_2d(b + kRP * 128 + NPR * 128, &a.cmap, bar, d0 + 16, 0);
    };
    if (producer) {  // the first stages are in flight while the candidates are found
        tma_prefetch_map(&a.xmap);
        tma_prefetch_map(&a.cmap);
        for (int g = 0; g < kRS && g < nsteps; ++g) issue(g);
    }
    // centroid norms: the atoms' partial norms added (rounded down / up)
    if (tid < KA) {
        float lo = 0.f, hi = 0.f;
        for (int q = 0; q < a.natoms; ++q) {  // the atoms' partial norms (k_wide_prep)
            lo = __fadd_rd(lo, a.nc[(static_cast<size_t>(q) * a.np + tid) * 2]);
            hi = __fadd_ru(hi, a.nc[(static_cast<size_t>(q) * a.np + tid) * 2 + 1]);
        }
        const bool ok = hi <= 1.0e36f;  // beyond: (0, inf, inf) -> L = 0, U = inf (exact fallback)
        ncl[tid] = ok ? lo : 0.f;
        nch[tid] = ok ? hi : finf;
        ncr[tid] = ok ? __fsqrt_ru(hi) : finf;
    }
    __syncthreads();
    // certified bounds (the screen's error model, wide_screen_consts): the KS
    // partial dot products added in split order; candidates j with L_j <= min U
    if (tid < kRP) {
        unsigned bits = 0;
        if (tid < np) {
            const uint64_t gp = q0 + tid;
            float nl = 0.f, nh = 0.f;
            for (int q = 0; q < a.ks; ++q) {
                const float2 v = reinterpret_cast<const float2*>(a.nx)[static_cast<size_t>(q) * a.rows + gp];
                nl = __fadd_rd(nl, v.x);
                nh = __fadd_ru(nh, v.y);
            }
            const bool okx = nh <= 1.0e36f;
            const float pxl = okx ? nl : 0.f, pxh = okx ? nh : finf, pxr = okx ? __fsqrt_ru(nh) : finf;
            float Lj[32];
            float mu = finf;
            for (int j = 0; j < KA; ++j) {
                float ds = 0.f;
                for (int q = 0; q < a.ks; ++q) ds = __fadd_rn(ds, a.dot[(static_cast<size_t>(q) * a.rows + gp) * a.np + j]);
                const float t2 = 2.f * ds;
                const float Sn = __fadd_ru(pxr, ncr[j]);
                const float Al = __fadd_rd(pxl, ncl[j]), Ah = __fadd_ru(pxh, nch[j]);
                float L = 0.f, U = finf;
                if (fabsf(t2) <= 1.0e37f && Sn <= 1.0e18f && Ah <= 1.0e37f) {
                    const float D = __fadd_ru(__fmul_ru(__fmul_ru(a.cst.K, Sn), Sn), a.cst.dabs);
                    L = fmaxf(__fsub_rd(__fsub_rd(Al, t2), D), 0.f);
                    L = __fmul_rd(L, a.cst.lo64);
                    U = __fmul_ru(__fadd_ru(__fsub_ru(Ah, t2), D), a.cst.hi64);
                }
                Lj[j] = L;
                mu = fminf(mu, U);
            }
            for (int j = 0; j < KA; ++j)
                if (Lj[j] <= mu) bits |= 1u << j;
        }
        cand[tid] = bits;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the candidate counts -> item offsets (ascending j per point)
        const int v = __popc(cand[tid]);
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= o) incl += y;
        }
        icount[tid] = incl - v;
        if (tid == 31) icount[kRP] = incl;
        unsigned b = cand[tid];
        int it = incl - v;
        while (b) {
            const int j = __ffs(b) - 1;
            b &= b - 1;
            item_p[it] = static_cast<short>(tid);
            item_j[it] = static_cast<signed char>(j);
            ++it;
        }
    }
    __syncthreads();
    const int NI = icount[kRP];
    const int rounds = (NI + kRItems - 1) / kRItems, total = rounds * nsteps;
    if (producer) {
        for (int g = min(kRS, nsteps); g < total; ++g) {  // (the prologue issued steps < min(kRS, nsteps))
            if (g >= kRS) umma::mbar_wait_parity(&s_empty[g % kRS], ((g / kRS) - 1) & 1);
            issue(g);
        }
    } else if (tid < kRT) {
        // exact fp64 chains (direct form, core.cpp:142-146) of up to 4 items per
        // thread per round; consecutive items on consecutive warps
        const int slot = (tid & 3) * 32 + (tid >> 2);
        for (int rd = 0; rd < rounds; ++rd) {
            const int i0 = rd * kRItems;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            int ip[4], ij[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = i0 + slot + r * kRT;
                ip[r] = i < NI ? item_p[i] : -1;
                ij[r] = i < NI ? item_j[i] : 0;
            }
            for (int t = 0; t < nsteps; ++t) {
                const int g = rd * nsteps + t, st = g % kRS, d0 = t * kRD, dl = min(kRD, a.n - d0);
                mbar_wait(reinterpret_cast<uint64_t*>(&s_full[st]), (g / kRS) & 1);
                const unsigned char* b = stg + static_cast<size_t>(st) * kStage;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (ip[r] < 0) continue;
                    const int pr = ip[r], jr = ij[r];
                    const unsigned char* xrow = b + pr * 128;
                    const unsigned char* c0row = b + kRP * 128 + jr * 128;
                    const unsigned char* c1row = c0row + NPR * 128;
                    auto xq = [&](int c) { return *reinterpret_cast<const float4*>(xrow + ((c ^ (pr & 7)) << 4)); };
                    auto cq = [&](int d) {  // dims d, d+1 (d even)
                        const unsigned char* row = d < 16 ? c0row : c1row;
                        return *reinterpret_cast<const double2*>(row + ((((d & 15) >> 1) ^ (jr & 7)) << 4));
                    };
                    double s_ = acc[r];
                    if (dl == kRD) {
                        // the 32 squared differences first (independent: loads, conversions,
                        // subtractions and products overlap), then the dependent left fold
                        // in dim order (core.cpp:144-145: the same operations, same order)
                        double q[kRD];
#pragma unroll
                        for (int c = 0; c < kRD / 4; ++c) {
                            const float4 xv = xq(c);
                            const double2 c0 = cq(4 * c);
                            const double2 c1 = cq(4 * c + 2);
                            const double e0 = __dsub_rn(static_cast<double>(xv.x), c0.x);
                            const double e1 = __dsub_rn(static_cast<double>(xv.y), c0.y);
                            const double e2 = __dsub_rn(static_cast<double>(xv.z), c1.x);
                            const double e3 = __dsub_rn(static_cast<double>(xv.w), c1.y);
                            q[4 * c] = __dmul_rn(e0, e0);
                            q[4 * c + 1] = __dmul_rn(e1, e1);
                            q[4 * c + 2] = __dmul_rn(e2, e2);
                            q[4 * c + 3] = __dmul_rn(e3, e3);
                        }
#pragma unroll
                        for (int i = 0; i < kRD; ++i) s_ = __dadd_rn(s_, q[i]);
                    } else {
                        for (int d = 0; d < dl; ++d) {
                            const float xv = reinterpret_cast<const float*>(xrow + (((d >> 2) ^ (pr & 7)) << 4))[d & 3];
                            const double cv = (d & 1) ? cq(d & ~1).y : cq(d & ~1).x;
                            s_ = dist_step(s_, static_cast<double>(xv), cv);
                        }
                    }
                    acc[r] = s_;
                }
                mbar_arrive(&s_empty[st]);  // this thread is done with the stage
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = i0 + slot + r * kRT;
                if (i < NI) item_d[i] = acc[r];
            }
        }
    }
    __syncthreads();
    if (tid < np) {  // ascending j, strict < (core.cpp:147)
        double best = __longlong_as_double(0x7FF0000000000000LL);
        int bj = -1;
        for (int i = icount[tid]; i < icount[tid + 1]; ++i)
            if (item_d[i] < best) {
                best = item_d[i];
                bj = item_j[i];
            }
        a.best[q0 + tid] = best;
        a.bj[q0 + tid] = bj;
    }
}

}  // namespace dev

WidePlan wide_plan(int device, uint64_t rows, int n, int k) {
    WidePlan p;
    if (k < 1 || k > 32 || n <= 0 || rows == 0 || rows >= (1ull << 31)) return p;
    p.np = k <= 16 ? 16 : 32;
    p.natoms = (n + 31) / 32;
    p.tiles = static_cast<unsigned>((rows + 127) / 128);
    int sms = 148, optin = 227 * 1024;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    // atoms per split: TMEM (512 columns, one NP-column block per bpa atoms) and
    // shared memory (the split's B operands + the ring) bound it; prefer one wave
    // of CTAs (tiles x splits <= SMs), then one atom per block (tighter bound)
    auto ks_min = [&](int bpa) {
        const int amax = 512 / p.np * bpa;  // TMEM: one NP-column block per bpa atoms
        return (p.natoms + amax - 1) / amax;
    };
    const int fill = std::max<int>(1, sms / static_cast<int>(p.tiles));  // splits that fit one wave
    int ks;
    if (ks_min(1) <= fill) {
        p.bpa = 1;
        ks = std::min(p.natoms, fill);
    } else if (ks_min(2) <= fill) {
        p.bpa = 2;
        ks = std::min(p.natoms, fill);
    } else {
        p.bpa = 1;
        ks = ks_min(1);
    }
    const int na = (p.natoms + ks - 1) / ks;
    ks = (p.natoms + na - 1) / na;  // no empty split
    p.ks = ks;
    p.na = na;
    p.smem = dev::wide_smem_bytes(p.np);
    p.ok = p.na >= 1 && p.smem + 1024 <= static_cast<size_t>(optin);
    return p;
}

dev::ScreenConsts wide_screen_consts(const WidePlan& p, int n) {
    const double u = std::ldexp(1.0, -24);
    auto gam = [&](double m) { return m * u / (1.0 - m * u); };
    // (2 MMAs x 32 dims per atom, bpa atoms per accumulator block; blocks, then splits, added in fp32)
    const double gb = 2.0 * (std::ldexp(1.0, -21) + 64.0 * p.bpa * std::ldexp(1.0, -23) +
                             gam((p.na + p.bpa - 1) / p.bpa) + gam(p.ks));
    const double up = u * (1.0 + 4 * u) / (1.0 - u);
    const double K = gb / 2.0 + 2.0 * up + up * up;
    const double u64 = std::ldexp(1.0, -53);
    const double g64 = (n + 3) * u64 / (1.0 - (n + 3) * u64);
    auto f_ru = [](double x) {
        float f = static_cast<float>(x);
        if (static_cast<double>(f) < x) f = std::nextafter(f, INFINITY);
        return f;
    };
    auto f_rd = [](double x) {
        float f = static_cast<float>(x);
        if (static_cast<double>(f) > x) f = std::nextafter(f, -INFINITY);
        return f;
    };
    dev::ScreenConsts c;
    c.K = f_ru(K * (1.0 + 1e-6));
    c.dabs = std::ldexp(1.0f, -40);
    c.lo64 = f_rd((1.0 - g64) * (1.0 - 4 * u64));
    c.hi64 = f_ru((1.0 + g64) * (1.0 + 4 * u64));
    return c;
}

CUtensorMap wide_cent_map(const double* Cact, int k, int n, int ldc, int np) {
    CUtensorMap m{};
    auto enc = tmap_encoder();
    if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)k};
    const cuuint64_t strides[1] = {(cuuint64_t)ldc * 8};
    const cuuint32_t box[2] = {16u, (cuuint32_t)np};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(Cact), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(wide centroids) failed");
    return m;
}

CUtensorMap wide_rows_map(const void* X, uint64_t rows, int n, uint64_t ld, int box_rows) {
    CUtensorMap m{};
    auto enc = tmap_encoder();
    if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    const cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(wide rows) failed");
    return m;
}

namespace {
std::mutex g_wide_mu;
}

void launch_wide_screen(cudaStream_t st, const WidePlan& p, const dev::WideArgs& a, bool pdl) {
    {  // the B operands and centroid norms of every atom
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(p.natoms));
        cfg.blockDim = dim3(128);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        dev::WideArgs args = a;
        void* kargs[] = {&args};
        const void* fn = p.np == 16 ? reinterpret_cast<const void*>(&dev::k_wide_prep<16>)
                                    : reinterpret_cast<const void*>(&dev::k_wide_prep<32>);
        BM_CUDA(cudaLaunchKernelExC(&cfg, fn, kargs));
    }
    void* fn = p.np == 16 ? reinterpret_cast<void*>(&dev::k_wide_screen<16>) : reinterpret_cast<void*>(&dev::k_wide_screen<32>);
    {
        static std::map<std::pair<int, void*>, size_t> cur;  // per device: raise the attribute, never lower it
        int dev = 0;
        BM_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_wide_mu);
        size_t& c = cur[std::make_pair(dev, fn)];
        if (p.smem > c) {
            BM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)));
            c = p.smem;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.tiles, static_cast<unsigned>(p.ks));
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    dev::WideArgs args = a;
    void* kargs[] = {&args};
    BM_CUDA(cudaLaunchKernelExC(&cfg, fn, kargs));
}

void launch_wide_recheck(cudaStream_t st, const WidePlan& p, const dev::RecheckArgs& a, bool pdl) {
    const int rs = p.np == 16 ? 16 : 12;
    const size_t smem = dev::wide_recheck_smem_bytes(rs, p.np);
    const void* fn = p.np == 16 ? reinterpret_cast<const void*>(&dev::k_wide_recheck<16, 16>)
                                : reinterpret_cast<const void*>(&dev::k_wide_recheck<12, 32>);
    {
        static std::map<std::pair<int, const void*>, bool> done;  // per (device, instance)
        int dev = 0;
        BM_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_wide_mu);
        bool& d = done[std::make_pair(dev, fn)];
        if (!d) {
            BM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            d = true;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.recheck_ctas(a.rows));
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    dev::RecheckArgs args = a;
    void* kargs[] = {&args};
    BM_CUDA(cudaLaunchKernelExC(&cfg, fn, kargs));
}

}  // namespace bm
