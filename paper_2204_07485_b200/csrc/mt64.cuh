// mt64.cuh — the reference RNG stream (Rng = std::mt19937_64, common.hpp:13)
// with libstdc++-13 distribution semantics, usable on host AND device.
//
// The stream is consumed in the reference's program order (big_means.hpp:21-23):
// per chunk the s sample draws uniform_int(i, m-1) (big_means.cpp:49-51), then
// only when the incumbent has degenerate rows the K-means++ draws
// (init.cpp:144-196).  The sample draws of a steady-state chunk are produced on
// the device (k_mt_twist, k_mt_emit, k_mt_fix), so the state lives on the device and visits the host
// only for repairs.  Bit-identity with std::mt19937_64 +
// std::uniform_int_distribution / uniform_real_distribution is checked by the
// CPU tests (tests/test_host.py) and the golden vectors.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

namespace bm {

constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ULL, kMtLower = 0x7FFFFFFFULL;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ULL;

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

__host__ __device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t x = (a & kMtUpper) | (b & kMtLower);
    return c ^ (x >> 1) ^ ((x & 1ULL) ? kMtA : 0ULL);
}

// 128-bit product helpers (Lemire's method, uniform_int_dist.h:252-331)
__host__ __device__ __forceinline__ uint64_t mul_hi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// Engine state exactly as std::mt19937_64 holds it (x[312] + position).
struct Mt64State {
    uint64_t x[kMtN];
    uint64_t pos;  // 312 => the next call twists
};

// Host engine.
struct Mt64 {
    Mt64State s;
    explicit Mt64(uint64_t seed = 5489u) { seed_with(seed); }
    void seed_with(uint64_t seed) {
        s.x[0] = seed;
        for (int i = 1; i < kMtN; ++i)
            s.x[i] = 6364136223846793005ULL * (s.x[i - 1] ^ (s.x[i - 1] >> 62)) + static_cast<uint64_t>(i);
        s.pos = kMtN;
    }
    void twist() {
        for (int i = 0; i < kMtN; ++i) s.x[i] = mt_mix(s.x[i], s.x[(i + 1) % kMtN], s.x[(i + kMtM) % kMtN]);
        s.pos = 0;
    }
    uint64_t operator()() {
        if (s.pos >= kMtN) twist();
        return mt_temper(s.x[s.pos++]);
    }
    // uniform_int_distribution<size_t>(a, b)
    uint64_t uniform_int(uint64_t a, uint64_t b) {
        const uint64_t urange = b - a;
        if (urange == ~0ULL) return (*this)() + a;
        const uint64_t r = urange + 1;
        uint64_t y = (*this)();
        uint64_t low = y * r;
        if (low < r) {
            const uint64_t thr = (0 - r) % r;
            while (low < thr) {
                y = (*this)();
                low = y * r;
            }
        }
        return mul_hi64(y, r) + a;
    }
    // uniform_real_distribution<double>(a, b): generate_canonical<double,53>
    double uniform_real(double a, double b) {
        double c = static_cast<double>((*this)()) / 18446744073709551616.0;
        if (c >= 1.0) c = std::nextafter(1.0, 0.0);
        return c * (b - a) + a;
    }
};

}  // namespace bm
