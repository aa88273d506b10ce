// kernels_data.cuh — dataset helpers: min-max normalisation, finiteness / exactness checks, narrowing, gathers.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

// ===========================================================================
// 8c. io::min_max_normalize (io.cpp:245-264) on the device: per-column min and
// max (exact), then (x - lo) / (hi - lo), constant columns -> 0.0.
// ===========================================================================
__device__ __forceinline__ unsigned long long ordered_bits(double v) {  // total order of doubles as integers
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(unsigned long long o) {
    return __longlong_as_double(static_cast<long long>((o >> 63) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o));
}

template <typename T>
__global__ void k_col_minmax(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
                             unsigned long long* __restrict__ lo, unsigned long long* __restrict__ hi) {
    // grid-stride over rows; each thread keeps one column's running min / max
    const int d = threadIdx.x % n;  // blockDim.x is a multiple of n (host)
    const int lanes = blockDim.x / n, li = threadIdx.x / n;
    if (li >= lanes) return;
    unsigned long long a = ~0ull, b = 0ull;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * lanes + li; i < rows;
         i += static_cast<uint64_t>(gridDim.x) * lanes) {
        const unsigned long long o = ordered_bits(to_f64(X[i * ld + d]));
        a = o < a ? o : a;
        b = o > b ? o : b;
    }
    atomicMin(&lo[d], a);
    atomicMax(&hi[d], b);
}

template <typename T>
__global__ void k_minmax_apply(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
                               const unsigned long long* __restrict__ lo, const unsigned long long* __restrict__ hi,
                               double* __restrict__ out) {  // out: rows x n, row-major (host layout)
    const uint64_t total = rows * static_cast<uint64_t>(n);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int d = static_cast<int>(e % n);
        const double l = from_ordered(lo[d]), h = from_ordered(hi[d]);
        const double range = __dsub_rn(h, l);
        out[e] = range > 0.0 ? __ddiv_rn(__dsub_rn(to_f64(X[(e / n) * ld + d]), l), range) : 0.0;
    }
}

// ===========================================================================
// 9. Dataset helpers.
// ===========================================================================
// Exact-sum statistics (§5b) of one finite value: exponent of its lowest set
// bit, and |x| as bits (ordered like the values for x >= 0).
__device__ __forceinline__ void exact_stats(double x, int& lowexp, unsigned long long& maxbits) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
    if (b == 0) return;
    const int E = static_cast<int>(b >> 52);
    const unsigned long long M = b & 0xFFFFFFFFFFFFFull;
    const int le = E == 0 ? -1074 + __ffsll(static_cast<long long>(M)) - 1
                          : E - 1075 + __ffsll(static_cast<long long>(M | (1ull << 52))) - 1;
    lowexp = min(lowexp, le);
    maxbits = max(maxbits, b);
}

__device__ __forceinline__ void exact_stats_flush(int lowexp, unsigned long long maxbits, int* lowexp_out,
                                                  unsigned long long* maxbits_out) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lowexp = min(lowexp, __shfl_xor_sync(0xFFFFFFFFu, lowexp, o));
        maxbits = max(maxbits, __shfl_xor_sync(0xFFFFFFFFu, maxbits, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (lowexp != 0x7F7F7F7F) atomicMin(lowexp_out, lowexp);
        if (maxbits) atomicMax(maxbits_out, maxbits);
    }
}

template <typename T>
__global__ void k_check_finite(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld, int* bad, int* lowexp_out,
                               unsigned long long* maxbits_out, int* not_tf32) {
    const uint64_t total = rows * static_cast<uint64_t>(n);
    int lowexp = 0x7F7F7F7F;
    unsigned long long maxbits = 0;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const T x = X[(e / n) * ld + (e % n)];
        const double v = to_f64(x);
        if (!isfinite(v)) *bad = 1;
        else exact_stats(v, lowexp, maxbits);
        // fp32 values with more than tf32's 11 significant bits (tensor-core screen bound)
        if (sizeof(T) != 4 || (__float_as_uint(static_cast<float>(x)) & 0x1FFFu) != 0u) *not_tf32 = 1;
    }
    exact_stats_flush(lowexp, maxbits, lowexp_out, maxbits_out);
}

// Lossless storage narrowing: an fp64 dataset whose every value round-trips
// through fp32 exactly is stored as fp32 (every kernel promotes exactly, so all
// results are unchanged) — half the HBM and L2 bytes.
__global__ void k_check_narrow(const double* __restrict__ v, uint64_t count, int* bad, int* inexact,
                               int* lowexp_out, unsigned long long* maxbits_out) {
    int lowexp = 0x7F7F7F7F;
    unsigned long long maxbits = 0;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double x = v[e];
        if (!isfinite(x)) {
            *bad = 1;
            continue;
        }
        if (static_cast<double>(static_cast<float>(x)) != x) *inexact = 1;
        exact_stats(x, lowexp, maxbits);
    }
    exact_stats_flush(lowexp, maxbits, lowexp_out, maxbits_out);
}

// k_check_narrow + k_narrow in one pass over rows [r0, r1): the checks, and
// the fp32 copy written speculatively (discarded when a value is not exact).
__global__ void k_check_narrow_write(const double* __restrict__ v, uint64_t r0, uint64_t r1, int n, int* bad,
                                     int* inexact, int* lowexp_out, unsigned long long* maxbits_out,
                                     float* __restrict__ out, uint64_t ld, int* not_tf32) {
    int lowexp = 0x7F7F7F7F;
    unsigned long long maxbits = 0;
    const uint64_t e0 = r0 * static_cast<uint64_t>(n), e1 = r1 * static_cast<uint64_t>(n);
    for (uint64_t e = e0 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < e1;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double x = v[e];
        const float f = static_cast<float>(x);
        out[(e / n) * ld + (e % n)] = f;
        if (!isfinite(x)) {
            *bad = 1;
            continue;
        }
        if (static_cast<double>(f) != x) *inexact = 1;
        if ((__float_as_uint(f) & 0x1FFFu) != 0u) *not_tf32 = 1;
        exact_stats(x, lowexp, maxbits);
    }
    exact_stats_flush(lowexp, maxbits, lowexp_out, maxbits_out);
}

__global__ void k_narrow(const double* __restrict__ in, uint64_t rows, int n, float* __restrict__ out, uint64_t ld) {
    const uint64_t total = rows * static_cast<uint64_t>(n);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[(e / n) * ld + (e % n)] = static_cast<float>(in[e]);
}

template <typename T>
__global__ void k_promote(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld, double* __restrict__ out) {
    const uint64_t total = rows * static_cast<uint64_t>(n);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[e] = to_f64(X[(e / n) * ld + (e % n)]);
}

template <typename T>
__global__ void k_gather_checked(const T* __restrict__ X, uint64_t ld, int n, const uint64_t* __restrict__ idx,
                                 uint64_t count, T* __restrict__ out, uint64_t out_ld) {
    const uint64_t total = count * static_cast<uint64_t>(n);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = e / n;
        out[r * out_ld + (e % n)] = X[idx[r] * ld + (e % n)];
    }
}

}  // namespace dev
}  // namespace bm
