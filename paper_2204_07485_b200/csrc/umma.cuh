// umma.cuh — sm_100a tensor-core (tcgen05 / TMEM) helpers shared by the
// persistent chunk kernel (chunk.cu) and the wide-row screen (wide.cu).
// kind::tf32 MMAs with fp32 accumulators in TMEM, K-major operands in the
// 128-byte-swizzle layout (8-row core-matrix groups 1024 B apart).
#pragma once

#include <cuda_runtime.h>

namespace bm {
namespace dev {
namespace umma {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// Shared-memory descriptor: K-major, 128-byte swizzle, SBO 1024 B, LBO unused
// (encoded 1), version 1 (sm_100), from the start address in 16-byte units.
// The two 32-bit halves are joined in PTX: ptxas (CUDA 12.9) was seen to drop
// the constant high half of a 64-bit descriptor built as (const | addr) +
// offset (SBO = 0, no swizzle: garbage MMA results for some code shapes), so
// no 64-bit arithmetic touches it.
__device__ __forceinline__ unsigned long long desc_sw128(unsigned start_units) {
    unsigned long long d;
    asm volatile("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"((start_units & 0x3FFFu) | (1u << 16)),
                 "r"(64u | (1u << 14) | (2u << 29)));
    return d;
}
// Instruction descriptor: D fp32, A / B tf32, both K-major, M = 128, N.
template <int N>
__host__ __device__ constexpr unsigned idesc_tf32() {
    static_assert(N % 16 == 0 && N >= 16 && N <= 256, "UMMA N for M = 128");
    return (1u << 4) | (2u << 7) | (2u << 10) | ((static_cast<unsigned>(N) >> 3) << 17) | ((128u >> 4) << 24);
}
// Issued by ONE thread (the same thread for every MMA and for their commit:
// tcgen05.commit tracks only the executing thread's MMAs).
__device__ __forceinline__ void mma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db, unsigned idesc,
                                         int accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float tf32_rna(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// TMEM columns: a power of two >= 32 covering `need`.
__host__ __device__ inline unsigned tmem_cols(unsigned need) {
    unsigned c = 32;
    while (c < need) c <<= 1;
    return c;
}
__device__ __forceinline__ void tmem_alloc(unsigned* dst_smem, unsigned cols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst_smem)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned taddr, unsigned cols) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
// 32 / 16 consecutive TMEM columns of this thread's lane (row) -> registers
// (the load and its wait in ONE asm statement: the outputs must not be read
// before tcgen05.wait::ld completes).
__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
    unsigned r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace umma
}  // namespace dev
}  // namespace bm
