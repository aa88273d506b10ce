// finaltc.cu — the final full-data assignment (big_means.cpp:102-107:
// assign_nearest core.cpp:106-161 over all m rows) on the tensor core, for
// fp32 rows exact in tf32 with n <= 88 (c2's integer rows).
//
// Persistent CTAs walk 128-row tiles.  A producer lane streams each tile's
// 32-dim atoms (TMA boxes in the UMMA K-major 128-byte-swizzle layout) through
// a ring; a thread of another warp issues the tile's MMAs (tcgen05.mma kind::tf32, M = 128,
// N = 64 = 32 centroid slots x (hi, lo) parts of fl32(c)) into one of two TMEM
// accumulators, so the next tile's MMAs run while this tile's epilogue runs.
// The epilogue — one thread per row — forms the certified bounds of the chunk
// kernel's tensor-core screen (chunk_screen_consts), rechecks the candidates in
// fp64 direct form (ascending j, strict <) from the staged row and the fp64
// centroids, and writes the label and the distance.  The 1024-row tile
// partials follow from k_tile_sums, as for k_final.
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "device_common.cuh"
#include "finaltc.h"
#include "tma.cuh"
#include "umma.cuh"

namespace bm {
namespace dev {

namespace {
constexpr int kFT = 128;          // epilogue threads (one per tile row)
constexpr int kFS = 3;            // tile stages
constexpr int kFK = 32;           // centroid slots
__device__ __forceinline__ void mbar_arrive_ft(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_addr(bar)) : "memory");
}
}  // namespace

__host__ __device__ inline int ft_cdld(int n) { return n + (n & 1) + 2; }  // fp64 centroid row stride
__host__ __device__ inline size_t ft_smem_bytes(int nka, int n) {
    return 1024 + static_cast<size_t>(kFS) * nka * 16384        // tile stages
           + static_cast<size_t>(nka) * 2 * kFK * 128            // B: per atom [hi 32 rows][lo 32 rows]
           + static_cast<size_t>(kFK) * ft_cdld(n) * 8;          // fp64 centroids
}

template <int NKA>
__global__ void __launch_bounds__(2 * kFT + 64, 1) k_final_tc(const __grid_constant__ FinalTcArgs a) {
    extern __shared__ __align__(16) unsigned char fsm_raw[];
    __shared__ __align__(8) unsigned long long s_full[kFS], s_empty[kFS], s_done[2], s_free[2];
    __shared__ unsigned s_tmem;
    __shared__ float ncl[kFK], nch[kFK], ncr[kFK];
    __shared__ int act[kFK + 1];
    pdl_wait();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool producer = tid == kFT, mma_thread = tid == kFT + 32;  // warps 4 and 5
    // two epilogue groups (warps 0-3 and 6-9): group g takes this CTA's tiles li = g, g + 2, ...
    // (accumulator li & 1 = g), so one tile's exact recheck runs beside the next tile's
    const int eg = warp < 4 ? 0 : warp >= 6 ? 1 : -1;
    const int row = 32 * (warp & 3) + lane;  // this thread's tile row = its TMEM lane (lane quarter warp % 4)
    const int n = a.n, cdld = ft_cdld(n);
    const uint64_t ntiles = (a.rows + 127) / 128;
    const uint64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;  // tiles of this CTA
    constexpr unsigned kTile = NKA * 16384u;
    unsigned char* sm = fsm_raw + ((1024u - (umma::smem_addr(fsm_raw) & 1023u)) & 1023u);
    unsigned char* stg = sm;
    unsigned char* B = sm + static_cast<size_t>(kFS) * kTile;
    double* cd = reinterpret_cast<double*>(B + static_cast<size_t>(NKA) * 2 * kFK * 128);
    constexpr unsigned kIdesc = umma::idesc_tf32<64>();
    if (tid == 0) {
        for (int i = 0; i < kFS; ++i) {
            mbar_init(reinterpret_cast<uint64_t*>(&s_full[i]), 1);
            mbar_init(reinterpret_cast<uint64_t*>(&s_empty[i]), kFT);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(reinterpret_cast<uint64_t*>(&s_done[i]), 1);
            mbar_init(reinterpret_cast<uint64_t*>(&s_free[i]), kFT);
        }
        fence_mbar_init();
    }
    if (tid <= kFK) act[tid] = tid < kFK ? (tid < *a.n_active ? a.act[tid] : 0) : *a.n_active;  // compacted list
    __syncthreads();
    auto load_tile = [&](uint64_t li) {
        const int s = static_cast<int>(li % kFS);
        const uint64_t tile = blockIdx.x + li * gridDim.x;
        uint64_t* bar = reinterpret_cast<uint64_t*>(&s_full[s]);
        mbar_expect_tx(bar, kTile);
        for (int ka = 0; ka < NKA; ++ka)
            tma_load_2d(stg + static_cast<size_t>(s) * kTile + static_cast<size_t>(ka) * 16384, &a.xmap, bar, ka * 32,
                        static_cast<int>(tile * 128));
    };
    if (producer) {
        tma_prefetch_map(&a.xmap);
        for (uint64_t li = 0; li < my && li < static_cast<uint64_t>(kFS); ++li) load_tile(li);
    }
    if (warp == 0) umma::tmem_alloc(&s_tmem, 128);  // two 64-column accumulators
    const int KA = act[kFK];
    // B operands (hi / lo of the compacted fp32 centroids, 0 past KA), fp64 copies, norms
    for (int e = tid; e < NKA * 32 * kFK; e += blockDim.x) {
        const int rk = e / (NKA * 32), d = e - rk * (NKA * 32);
        const double v = rk < KA && d < n ? __ldcg(a.Cact + static_cast<size_t>(rk) * a.ldc + d) : 0.0;
        const float f = __double2float_rn(v), hi = umma::tf32_rna(f);
        const size_t off = static_cast<size_t>(d >> 5) * (2 * kFK * 128) + rk * 128 + ((((d >> 2) & 7) ^ (rk & 7)) << 4) +
                           (d & 3) * 4;
        *reinterpret_cast<float*>(B + off) = hi;
        *reinterpret_cast<float*>(B + off + kFK * 128) = f - hi;
        if (rk < KA && d < n) cd[rk * cdld + d] = v;
    }
    umma::fence_proxy_async_smem();
    __syncthreads();
    for (int rk = warp; rk < KA; rk += blockDim.x / 32) {
        float lo = 0.f, hi = 0.f;
        for (int d = lane; d < n; d += 32) {
            const float f = __double2float_rn(cd[rk * cdld + d]);
            lo = __fmaf_rd(f, f, lo);
            hi = __fmaf_ru(f, f, hi);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = __fadd_rd(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
            hi = __fadd_ru(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
        }
        if (lane == 0) {
            const bool ok = hi <= 1.0e36f;
            ncl[rk] = ok ? lo : 0.f;
            nch[rk] = ok ? hi : __int_as_float(0x7F800000);
            ncr[rk] = ok ? __fsqrt_ru(hi) : __int_as_float(0x7F800000);
        }
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const unsigned tbase = s_tmem;
    const unsigned ust = umma::smem_addr(stg) >> 4, ub = umma::smem_addr(B) >> 4;
    // the MMA thread (warp 5): the MMAs of local tile li into accumulator li % 2
    auto issue = [&](uint64_t li) {
        const int s = static_cast<int>(li % kFS), acc = static_cast<int>(li & 1);
        mbar_wait(reinterpret_cast<uint64_t*>(&s_full[s]), static_cast<unsigned>((li / kFS) & 1));
        if (li >= 2) umma::mbar_wait_parity(&s_free[acc], static_cast<unsigned>(((li / 2) - 1) & 1));
        umma::fence_after();
        for (int ks = 0; ks < NKA * 4; ++ks) {
            if (ks * 8 >= ((a.n + 7) & ~7)) break;  // k-steps past n: zero in both operands
            const unsigned ko = ((ks & 3) * 32) >> 4;
            const unsigned da = ust + static_cast<unsigned>(s) * (kTile >> 4) + ((ks >> 2) * 16384 >> 4) + ko;
            const unsigned db = ub + ((ks >> 2) * (2 * kFK * 128) >> 4) + ko;
            umma::mma_tf32(tbase + 64u * acc, umma::desc_sw128(da), umma::desc_sw128(db), kIdesc, ks > 0);
        }
        umma::commit(&s_done[acc]);
    };
    if (producer) {
        for (uint64_t li = kFS; li < my; ++li) {
            const int s = static_cast<int>(li % kFS);
            umma::mbar_wait_parity(&s_empty[s], static_cast<unsigned>(((li / kFS) - 1) & 1));
            load_tile(li);
        }
    } else if (mma_thread) {
        for (uint64_t li = 0; li < my; ++li) issue(li);
    } else if (eg >= 0) {
        const float finf = __int_as_float(0x7F800000);
        const double dinf = __longlong_as_double(0x7FF0000000000000LL);
        for (uint64_t li = static_cast<uint64_t>(eg); li < my; li += 2) {
            const int s = static_cast<int>(li % kFS), acc = static_cast<int>(li & 1);
            const uint64_t tile = blockIdx.x + li * gridDim.x;
            const uint64_t gp = tile * 128 + row;
            umma::mbar_wait_parity(&s_done[acc], static_cast<unsigned>((li / 2) & 1));
            __syncwarp();  // (tcgen05.ld is warp-aligned)
            umma::fence_after();
            float Lv[32];
            {
                const unsigned ta = tbase + (static_cast<unsigned>(32 * (warp & 3)) << 16) + 64u * acc;
                float Lw[32];
                umma::tmem_ld32(ta, Lv);
                umma::tmem_ld32(ta + 32u, Lw);
#pragma unroll
                for (int j = 0; j < 32; ++j) Lv[j] = __fadd_rn(Lv[j], Lw[j]);
            }
            umma::fence_before();
            mbar_arrive_ft(&s_free[acc]);  // this thread's TMEM reads of the accumulator are done
            const unsigned char* rowb = stg + static_cast<size_t>(s) * kTile + static_cast<size_t>(row) * 128;
            const int sw = row & 7;
            if (gp < a.rows) {
                // this row's squared norm (rounded down / up), from the staged row
                float xl = 0.f, xh = 0.f;
                for (int q = 0; q < (n + 3) / 4; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(rowb + static_cast<size_t>(q >> 3) * 16384 +
                                                                     (((q & 7) ^ sw) << 4));
                    xl = __fmaf_rd(v.x, v.x, xl); xh = __fmaf_ru(v.x, v.x, xh);
                    xl = __fmaf_rd(v.y, v.y, xl); xh = __fmaf_ru(v.y, v.y, xh);
                    xl = __fmaf_rd(v.z, v.z, xl); xh = __fmaf_ru(v.z, v.z, xh);
                    xl = __fmaf_rd(v.w, v.w, xl); xh = __fmaf_ru(v.w, v.w, xh);
                }
                const bool okx = xh <= 1.0e36f;
                const float pxl = okx ? xl : 0.f, pxh = okx ? xh : finf, pxr = okx ? __fsqrt_ru(xh) : finf;
                float mu = finf;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j >= KA) Lv[j] = finf;
                    if (j >= KA) continue;
                    const float t2 = 2.f * Lv[j];
                    const float Sn = __fadd_ru(pxr, ncr[j]);
                    const float Al = __fadd_rd(pxl, ncl[j]), Ah = __fadd_ru(pxh, nch[j]);
                    float L = 0.f, U = finf;
                    if (fabsf(t2) <= 1.0e37f && Sn <= 1.0e18f && Ah <= 1.0e37f) {
                        const float D = __fadd_ru(__fmul_ru(__fmul_ru(a.cst.K, Sn), Sn), a.cst.dabs);
                        L = fmaxf(__fsub_rd(__fsub_rd(Al, t2), D), 0.f);
                        L = __fmul_rd(L, a.cst.lo64);
                        U = __fmul_ru(__fadd_ru(__fsub_ru(Ah, t2), D), a.cst.hi64);
                    }
                    Lv[j] = L;
                    mu = fminf(mu, U);
                }
                unsigned cm = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) cm |= (Lv[j] <= mu ? 1u : 0u) << j;
                // exact fp64 recheck of the candidates: ascending j, strict < (core.cpp:142-153)
                double best = dinf;
                int bj = -1;
                while (cm) {
                    const int j = __ffs(cm) - 1;
                    cm &= cm - 1;
                    const double* c = cd + j * cdld;
                    double sum = 0.0;
                    int d = 0;
                    for (; d + 4 <= n; d += 4) {
                        const int q = d >> 2;
                        const float4 xv = *reinterpret_cast<const float4*>(rowb + static_cast<size_t>(q >> 3) * 16384 +
                                                                          (((q & 7) ^ sw) << 4));
                        sum = dist_step(sum, static_cast<double>(xv.x), c[d]);
                        sum = dist_step(sum, static_cast<double>(xv.y), c[d + 1]);
                        sum = dist_step(sum, static_cast<double>(xv.z), c[d + 2]);
                        sum = dist_step(sum, static_cast<double>(xv.w), c[d + 3]);
                    }
                    for (; d < n; ++d) {
                        const int q = d >> 2;
                        const float x = reinterpret_cast<const float*>(rowb + static_cast<size_t>(q >> 3) * 16384 +
                                                                        (((q & 7) ^ sw) << 4))[d & 3];
                        sum = dist_step(sum, static_cast<double>(x), c[d]);
                    }
                    if (sum < best) {
                        best = sum;
                        bj = j;
                    }
                }
                if (bj < 0) bj = 0;  // (NaN distances only; unreachable for finite data)
                a.labels[gp] = act[bj];
                a.dists[gp] = best;
            }
            mbar_arrive_ft(&s_empty[s]);  // this thread is done with the stage
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) {
        umma::fence_after();
        umma::tmem_dealloc(tbase, 128);
    }
}

}  // namespace dev

namespace {
std::mutex g_ft_mu;
}

bool final_tc_supported(int n, int k) { return n >= 1 && n <= 88 && k >= 1 && k <= 32; }

void launch_final_tc(cudaStream_t st, int device, const dev::FinalTcArgs& a, bool pdl) {
    const int nka = (a.n + 31) / 32;
    const void* fn = nka == 1   ? reinterpret_cast<const void*>(&dev::k_final_tc<1>)
                     : nka == 2 ? reinterpret_cast<const void*>(&dev::k_final_tc<2>)
                                : reinterpret_cast<const void*>(&dev::k_final_tc<3>);
    const size_t smem = dev::ft_smem_bytes(nka, a.n);
    {
        static std::map<std::pair<int, const void*>, size_t> cur;
        std::lock_guard<std::mutex> lk(g_ft_mu);
        size_t& c = cur[std::make_pair(device, fn)];
        if (smem > c) {
            BM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            c = smem;
        }
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t ntiles = (a.rows + 127) / 128;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ntiles < static_cast<uint64_t>(sms) ? ntiles : sms));
    cfg.blockDim = dim3(2 * 128 + 64);  // two epilogue groups + the producer and MMA warps
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    dev::FinalTcArgs args = a;
    void* kargs[] = {&args};
    BM_CUDA(cudaLaunchKernelExC(&cfg, fn, kargs));
}

CUtensorMap final_tc_map(const void* X, uint64_t rows, int n, uint64_t ld) {
    CUtensorMap m{};
    auto enc = tmap_encoder();
    if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    const cuuint32_t box[2] = {32u, 128u};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(final rows) failed");
    return m;
}

}  // namespace bm
