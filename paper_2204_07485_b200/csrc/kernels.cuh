// kernels.cuh — sm_100a kernels of the Big-means hot path.
//
// Bit-exactness contract.  Every fp64 operation that the
// reference performs is performed here with the same operands in the same
// order, with explicit round-to-nearest intrinsics (__dsub_rn/__dmul_rn/
// __dadd_rn) so that nvcc can never contract a*b+c into an FMA (the
// reference's default x86-64 build emits none).  fp32-stored datasets are
// promoted to fp64 exactly ((double)x) before any arithmetic.
//
// Citations are relative to /root/reference/proj.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "device_common.cuh"
#include "mt64.cuh"
#include "tma.cuh"
#include "wide.h"

namespace bm {
namespace dev {

// Optional per-CTA phase timestamps (build with -DBM_KTRACE; tools/ktrace.py).
#ifdef BM_KTRACE
__device__ unsigned long long g_ktrace[1 << 20];
__device__ __forceinline__ void ktrace(int slot, int hm = 0) {  // region by assignment mode (0 / 1 / 2)
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        unsigned long long* row = g_ktrace + (hm == 0 ? 0 : hm == 1 ? 400000 : 470000) + (blockIdx.x & 2047) * 32;
        if (slot == 0)
            for (int i = 1; i < 32; ++i) row[i] = 0;
        row[slot] = t;
    }
}
// region 1: k_update CTAs (linear block id)
__device__ __forceinline__ void ktrace_u(int slot) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const unsigned id = (blockIdx.y * gridDim.x + blockIdx.x) & 2047;
        unsigned long long* row = g_ktrace + 65536 + id * 32;
        if (slot == 0)
            for (int i = 1; i < 32; ++i) row[i] = 0;
        row[slot] = t;
    }
}
// region 2 (index 200000): kernel log.  klog_start by CTA (0,0), klog_end by
// the launch's last CTA: [200000] = count, then (id, start, end) triples.
__device__ unsigned long long g_kstart[32];
__device__ __forceinline__ void klog_start(int id) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_kstart[id] = t;
    }
}
__device__ __forceinline__ void klog_end(int id) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long i = atomicAdd(&g_ktrace[200000], 1ull) % 60000ull;
    g_ktrace[200001 + 3 * i] = static_cast<unsigned long long>(id);
    g_ktrace[200002 + 3 * i] = g_kstart[id];
    g_ktrace[200003 + 3 * i] = t;
}
// an early-exit launch (id + 10): CTA 0's exit time
__device__ __forceinline__ void klog_exit(int id) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const unsigned long long i = atomicAdd(&g_ktrace[200000], 1ull) % 60000ull;
        g_ktrace[200001 + 3 * i] = static_cast<unsigned long long>(id + 10);
        g_ktrace[200002 + 3 * i] = g_kstart[id];
        g_ktrace[200003 + 3 * i] = t;
    }
}
#else
__device__ __forceinline__ void klog_exit(int) {}
__device__ __forceinline__ void ktrace(int, int = 0) {}
__device__ __forceinline__ void ktrace_u(int) {}
__device__ __forceinline__ void klog_start(int) {}
__device__ __forceinline__ void klog_end(int) {}
#endif

}  // namespace dev
}  // namespace bm

#include "kernels_sample.cuh"
#include "kernels_control.cuh"
#include "kernels_assign.cuh"
#include "kernels_update.cuh"
#include "kernels_init.cuh"
#include "kernels_data.cuh"
