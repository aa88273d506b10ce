// kernels_init.cuh — K-means++ and K-means|| seeding on the device.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

// ===========================================================================
// 8. K-means++ helpers (init.cpp:19-43, 183-198).
// out[c*rows + i] = dist(x_i, x_{cand[c]}), lowered by d2 when given
// (trial = std::min(trial, dist2) -> dist2 < trial ? dist2 : trial).
// ===========================================================================
template <typename T>
__global__ void k_dist_rows(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
                            const uint32_t* __restrict__ cand, int ncand,
                            const double* __restrict__ d2, double* __restrict__ out, const int* skip) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    if (skip && (skip[0] || skip[1])) return;  // device K-means++ step: fallback or direct pick
    const T* x = X + i * ld;
    for (int c = blockIdx.y; c < ncand; c += gridDim.y) {  // one candidate per grid row
        const T* r = X + static_cast<uint64_t>(cand[c]) * ld;
        double sum = 0.0;
        for (int d = 0; d < n; ++d) sum = dist_step(sum, to_f64(x[d]), to_f64(r[d]));
        if (d2) {
            const double o = d2[i];
            if (o < sum) sum = o;
        }
        out[static_cast<uint64_t>(c) * rows + i] = sum;
    }
}

// The same for narrow rows (n <= kDistRowsN) and up to 4 candidates: one thread
// per row takes every candidate at once — the row is read once in 16-byte
// vectors and converted once, the candidate rows sit in shared memory as fp64
// (one conversion each), the chains of the candidates run side by side.  Every
// (row, candidate) chain is the same ascending-d fold as above.
constexpr int kDistRowsN = 128;
template <typename T>
__global__ void __launch_bounds__(128)
k_dist_rows_narrow(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld, const uint32_t* __restrict__ cand,
                   int ncand, const double* __restrict__ d2, double* __restrict__ out, const int* skip) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    if (skip && (skip[0] || skip[1])) return;  // device K-means++ step: fallback or direct pick
    __shared__ __align__(16) double rs[4][kDistRowsN];
    for (int e = threadIdx.x; e < ncand * n; e += blockDim.x) {
        const int c = e / n, d = e - c * n;
        rs[c][d] = to_f64(X[static_cast<uint64_t>(cand[c]) * ld + d]);
    }
    __syncthreads();
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    constexpr int EPC = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte vector (ld is a multiple)
    const T* x = X + i * ld;
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int d0 = 0; d0 < n; d0 += EPC) {
        T v[EPC];
        *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(x + d0);
#pragma unroll
        for (int u = 0; u < EPC; ++u) {
            const int d = d0 + u;
            if (d < n) {
                const double xd = to_f64(v[u]);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < ncand) sum[c] = dist_step(sum[c], xd, rs[c][d]);
            }
        }
    }
    const double o = d2 ? d2[i] : 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (c < ncand) {
            double v = sum[c];
            if (d2 && o < v) v = o;
            out[static_cast<uint64_t>(c) * rows + i] = v;
        }
}

// ---------------------------------------------------------------------------
// Device K-means++ step (init.cpp:171-199) for integer D^2 weights.
// prefix_sums (init.cpp:81-88) is a sequential fp64 fold; when every weight is
// an integer and the total stays below 2^53 every partial sum is exact, so an
// integer scan reproduces it bit for bit.  Otherwise the step reports
// `fallback` (before consuming any draw) and the host path takes over.
// ---------------------------------------------------------------------------
struct PPState {
    int fallback;     // this slot needs the host path (non-integer or huge weights)
    int direct;       // total <= 0: uniform pick, no candidates (:174-180)
    int best;         // candidate chosen by k_pp_best (-1: none)
    int cand_slots;   // slots that evaluated candidates (n_d accounting)
    long long direct_idx;
};

__device__ uint64_t mt_uniform_int(uint64_t* x, int& pos, uint64_t a, uint64_t b) {  // uniform_int_dist.h:252-331
    const uint64_t urange = b - a;
    if (urange == ~0ull) return mt_next_seq(x, pos) + a;
    const uint64_t r = urange + 1;
    uint64_t y = mt_next_seq(x, pos);
    uint64_t low = y * r;
    if (low < r) {
        const uint64_t thr = (0 - r) % r;
        while (low < thr) {
            y = mt_next_seq(x, pos);
            low = y * r;
        }
    }
    return mul_hi64(y, r) + a;
}

__device__ double mt_uniform_real(uint64_t* x, int& pos, double a, double b) {  // generate_canonical<double,53>
    double c = __dmul_rn(__ull2double_rn(mt_next_seq(x, pos)), 0x1p-64);
    if (c >= 1.0) c = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
    return __dadd_rn(__dmul_rn(c, __dsub_rn(b, a)), a);
}

constexpr int kPPThreads = 1024;

// Step A, one CTA per 1024-weight tile: integrality check and the tile's
// inclusive integer scan (coalesced).
__global__ void __launch_bounds__(kPPThreads)
k_pp_scan(const double* __restrict__ d2, uint64_t m, long long* __restrict__ prefix,
          long long* __restrict__ tile_tot, PPState* ps) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    __shared__ long long wsum[kPPThreads / 32];
    if (ps->fallback) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kPPThreads + tid;
    long long v = 0;
    bool bad = false;
    if (i < m) {
        const double x = d2[i];
        if (!(x >= 0.0 && x < 0x1p53 && x == rint(x))) bad = true;
        else v = static_cast<long long>(x);
    }
    if (__syncthreads_or(bad)) {
        if (tid == 0) ps->fallback = 1;  // every tile sees its own weights; any one suffices
        return;
    }
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const long long x = wsum[lane];
        long long w = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w - x;
        if (lane == 31) tile_tot[blockIdx.x] = w;
    }
    __syncthreads();
    if (i < m) prefix[i] = wsum[warp] + incl;
}

// Step B, one CTA: tile offsets, total, the draws (one thread, the reference's
// order) and pick_by_mass (init.cpp:73-79) for each draw.
__global__ void __launch_bounds__(kPPThreads)
k_pp_pick(uint64_t m, Mt64State* __restrict__ mt, int candidates, uint32_t* __restrict__ cand,
          const long long* __restrict__ prefix, const long long* __restrict__ tile_tot, PPState* ps) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    __shared__ uint64_t xs[kMtN];
    __shared__ long long toff[kPPThreads + 1];
    __shared__ double us[8];
    __shared__ int direct_s, tsel, first;
    if (ps->fallback) return;
    const int tid = threadIdx.x;
    const int ntiles = static_cast<int>((m + kPPThreads - 1) / kPPThreads);
    if (ntiles > kPPThreads) {  // beyond one CTA's offset table: host path
        if (tid == 0) ps->fallback = 1;
        return;
    }
    // exclusive offsets of the tiles (<= 1024 exact integer adds): the totals
    // staged in parallel, then one thread's running sum from shared memory
    if (tid < ntiles) toff[tid + 1] = tile_tot[tid];
    if (tid < kMtN) xs[tid] = mt->x[tid];
    __syncthreads();
    if (tid == 0) {
        long long r = 0;
        for (int t = 0; t < ntiles; ++t) {
            const long long v = toff[t + 1];
            toff[t] = r;
            r += v;
        }
        toff[ntiles] = r;
    }
    __syncthreads();
    const long long total = toff[ntiles];
    if (total >= (1ll << 53)) {  // partial sums could round
        if (tid == 0) ps->fallback = 1;
        return;
    }
    if (tid == 0) {
        int pos = static_cast<int>(mt->pos);
        if (total <= 0) {  // :174-180
            ps->direct_idx = static_cast<long long>(mt_uniform_int(xs, pos, 0, m - 1));
            direct_s = 1;
        } else {
            for (int c = 0; c < candidates; ++c) us[c] = mt_uniform_real(xs, pos, 0.0, static_cast<double>(total));
            direct_s = 0;
            ps->cand_slots += 1;
        }
        ps->direct = direct_s;
        mt->pos = static_cast<uint64_t>(pos);
    }
    __syncthreads();
    if (tid < kMtN) mt->x[tid] = xs[tid];
    if (direct_s) return;
    for (int c = 0; c < candidates; ++c) {  // first index whose cumulative exceeds u
        const double u = us[c];
        if (tid == 0) {
            tsel = ntiles;
            first = kPPThreads;
        }
        __syncthreads();
        if (tid < ntiles && static_cast<double>(toff[tid + 1]) > u) atomicMin(&tsel, tid);
        __syncthreads();
        const int t = tsel;
        if (t < ntiles) {
            const uint64_t i = static_cast<uint64_t>(t) * kPPThreads + tid;
            if (i < m && static_cast<double>(toff[t] + prefix[i]) > u) atomicMin(&first, tid);
            __syncthreads();
            if (tid == 0) cand[c] = static_cast<uint32_t>(static_cast<uint64_t>(t) * kPPThreads + first);
        } else if (tid == 0) {
            cand[c] = static_cast<uint32_t>(m - 1);  // upper_bound == end: the last index
        }
        __syncthreads();
    }
}

// Best candidate by potential (block_sum of the trial, :190-195, strict <)
// and set_row(slot) (:197).
template <typename T>
__global__ void k_pp_best(const double* __restrict__ tiles, uint64_t ntiles, int candidates,
                          const uint32_t* __restrict__ cand, PPState* ps, const T* __restrict__ X, uint64_t ld,
                          int n, double* __restrict__ C, uint8_t* __restrict__ mask, int slot) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    __shared__ long long row_s;
    __shared__ __align__(16) double tl[4 * 1024];
    if (ps->fallback) return;
    const bool staged = static_cast<uint64_t>(candidates) * ntiles <= 4 * 1024;
    if (staged && !ps->direct)
        for (uint64_t e = threadIdx.x; e < static_cast<uint64_t>(candidates) * ntiles; e += blockDim.x) tl[e] = tiles[e];
    __syncthreads();
    if (threadIdx.x == 0) {
        long long row = 0;
        int bi = -1;
        if (ps->direct) {
            row = ps->direct_idx;
        } else {
            double best = __longlong_as_double(0x7FF0000000000000LL);
            for (int c = 0; c < candidates; ++c) {
                const double* tc = (staged ? tl : tiles) + static_cast<uint64_t>(c) * ntiles;
                double pot = 0.0;  // block_sum outer fold
                for (uint64_t t = 0; t < ntiles; ++t) pot = __dadd_rn(pot, tc[t]);
                if (pot < best) {
                    best = pot;
                    bi = c;
                    row = cand[c];
                }
            }
        }
        ps->best = bi;
        row_s = row;
    }
    __syncthreads();
    const uint64_t r = static_cast<uint64_t>(row_s);
    for (int d = threadIdx.x; d < n; d += blockDim.x)
        C[static_cast<uint64_t>(slot) * n + d] = to_f64(X[r * ld + d]);
    if (threadIdx.x == 0) mask[slot] = 0;
}

// dist2 := best_trial (:198)
__global__ void k_pp_take(double* __restrict__ pool, uint64_t R, uint64_t m, int d2i, const PPState* ps) {
    pdl_wait();  // (programmatic dependent launch: the previous kernel's writes)
    if (ps->fallback || ps->direct || ps->best < 0) return;
    const double* src = pool + static_cast<uint64_t>(ps->best) * R;
    double* dst = pool + static_cast<uint64_t>(d2i) * R;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

// set_row (core.cpp:78-83 / init.cpp:146,197): centroid j := pool row.
template <typename T>
__global__ void k_set_row(const T* __restrict__ X, uint64_t ld, int n, uint64_t r,
                          double* __restrict__ C, uint8_t* __restrict__ mask, int j) {
    for (int d = threadIdx.x; d < n; d += blockDim.x)
        C[static_cast<uint64_t>(j) * n + d] = to_f64(X[r * ld + d]);
    if (threadIdx.x == 0) mask[j] = 0;
}

// ===========================================================================
// 8b. K-means|| seeding (kmeans_parallel_init init.cpp:209-347) on the device.
// ===========================================================================
// Round draws (:251-258): one uniform_real(0,1) per point in index order (raw
// words from k_mt_twist, tempered here); point i joins with probability
// min(1, l * D2[i] / phi).  Result: one bit per point (ascending order).
__global__ void k_kpar_bern(const uint64_t* __restrict__ raw, const double* __restrict__ d2, uint64_t m, double l,
                            double phi, uint32_t* __restrict__ bits) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool take = false;
    if (i < m) {
        double u = __dmul_rn(__ull2double_rn(mt_temper(raw[i])), 0x1p-64);  // generate_canonical
        if (u >= 1.0) u = 0x1.fffffffffffffp-1;
        u = __dadd_rn(__dmul_rn(u, 1.0), 0.0);  // unit(rng): canon * (1 - 0) + 0
        double p = __ddiv_rn(__dmul_rn(l, d2[i]), phi);
        if (!(p < 1.0)) p = 1.0;  // std::min(1.0, p)
        take = u < p;
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, take);
    if ((threadIdx.x & 31) == 0 && i < m) bits[i >> 5] = b;
}

// lower_to_row (init.cpp:46-70) for a batch of rows: D2[i] = min(D2[i], min over
// the batch of the exact distance).  min is exact, so one pass equals the
// reference's row-by-row passes.
template <typename T>
__global__ void k_kpar_lower(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
                             const uint32_t* __restrict__ cand, int ncand, double* __restrict__ d2) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const T* x = X + i * ld;
    double best = d2[i];
    for (int c = 0; c < ncand; ++c) {
        const T* r = X + static_cast<uint64_t>(cand[c]) * ld;
        double sum = 0.0;
        for (int d = 0; d < n; ++d) sum = dist_step(sum, to_f64(x[d]), to_f64(r[d]));
        if (sum < best) best = sum;
    }
    d2[i] = best;
}

// data.gather(cand_index) (:280) promoted to fp64 rows [count][n].
template <typename T>
__global__ void k_rows_f64(const T* __restrict__ X, uint64_t ld, int n, const uint32_t* __restrict__ idx,
                           uint64_t count, double* __restrict__ out) {
    const uint64_t total = count * static_cast<uint64_t>(n);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[e] = to_f64(X[static_cast<uint64_t>(idx[e / n]) * ld + (e % n)]);
}

// Candidate weights (:292-295): points nearest each candidate (exact integer counts).
__global__ void k_kpar_count(const int32_t* __restrict__ labels, uint64_t m, unsigned long long* __restrict__ cnt) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m && labels[i] >= 0) atomicAdd(&cnt[labels[i]], 1ull);
}

// Exact fp64 distance (init.cpp:32-36) between two fp64 rows.
__device__ __forceinline__ double row_dist64(const double* __restrict__ a, const double* __restrict__ b, int n) {
    double sum = 0.0;
    for (int d = 0; d < n; ++d) sum = dist_step(sum, a[d], b[d]);
    return sum;
}

// Weighted greedy k-means++ over the candidates (:297-339), one CTA: the draws
// from the device-resident stream, the sequential sums (prefix_sums, potential)
// by thread 0, distances by all threads.  scratch: 4 * nc doubles.
__global__ void __launch_bounds__(256)
k_kpar_reduce(const double* __restrict__ Cc, int n, const unsigned long long* __restrict__ cnt, uint64_t nc, int k,
              int candidates, Mt64State* __restrict__ mt, double* __restrict__ scratch, uint32_t* __restrict__ chosen,
              unsigned long long* __restrict__ evals) {
    __shared__ uint64_t xs[kMtN];
    __shared__ int pos;
    __shared__ double total_s;
    __shared__ uint64_t pick_s;
    __shared__ int flip_s;  // which of (trial, best_trial) buffers holds best_trial
    const int tid = threadIdx.x;
    double* cdist2 = scratch;
    double* cum = scratch + nc;
    double* tb[2] = {scratch + 2 * nc, scratch + 3 * nc};
    for (int i = tid; i < kMtN; i += blockDim.x) xs[i] = mt->x[i];
    if (tid == 0) pos = static_cast<int>(mt->pos);
    __syncthreads();
    unsigned long long ev = 0;
    // wcum = prefix_sums(weight); chosen_first = pick_by_mass(wcum, wdraw)  (:297-300)
    if (tid == 0) {
        double run = 0.0;
        for (uint64_t q = 0; q < nc; ++q) {
            run = __dadd_rn(run, static_cast<double>(cnt[q]));
            cum[q] = run;
        }
        int p = pos;
        const double u = mt_uniform_real(xs, p, 0.0, run);
        pos = p;
        uint64_t lo = 0, hi = nc;  // upper_bound, clamped
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (u < cum[mid]) hi = mid;
            else lo = mid + 1;
        }
        pick_s = lo == nc ? nc - 1 : lo;
        chosen[0] = static_cast<uint32_t>(pick_s);
    }
    __syncthreads();
    {
        const double* r = Cc + pick_s * n;
        for (uint64_t q = tid; q < nc; q += blockDim.x) cdist2[q] = row_dist64(Cc + q * n, r, n);  // :302
        ev += nc;
    }
    __syncthreads();
    for (int nch = 1; nch < k; ++nch) {
        if (tid == 0) {  // mass = weight * cdist2; prefix sums (:309-313)
            double run = 0.0;
            for (uint64_t q = 0; q < nc; ++q) {
                run = __dadd_rn(run, __dmul_rn(static_cast<double>(cnt[q]), cdist2[q]));
                cum[q] = run;
            }
            total_s = run;
            flip_s = 0;
        }
        __syncthreads();
        const double total = total_s;
        if (total <= 0.0) {  // :314-317
            if (tid == 0) {
                int p = pos;
                chosen[nch] = static_cast<uint32_t>(mt_uniform_int(xs, p, 0, nc - 1));
                pos = p;
            }
            __syncthreads();
            continue;
        }
        double best_potential = __longlong_as_double(0x7FF0000000000000LL);  // thread 0's view
        uint64_t best_index = 0;
        for (int c = 0; c < candidates; ++c) {  // :321-335
            if (tid == 0) {
                int p = pos;
                const double u = mt_uniform_real(xs, p, 0.0, total);
                pos = p;
                uint64_t lo = 0, hi = nc;
                while (lo < hi) {
                    const uint64_t mid = lo + (hi - lo) / 2;
                    if (u < cum[mid]) hi = mid;
                    else lo = mid + 1;
                }
                pick_s = lo == nc ? nc - 1 : lo;
            }
            __syncthreads();
            double* trial = tb[flip_s ^ 1];
            const double* r = Cc + pick_s * n;
            for (uint64_t q = tid; q < nc; q += blockDim.x) {
                const double t = row_dist64(Cc + q * n, r, n);
                trial[q] = cdist2[q] < t ? cdist2[q] : t;  // std::min(trial, cdist2)
            }
            ev += nc;
            __syncthreads();
            if (tid == 0) {
                double potential = 0.0;
                for (uint64_t q = 0; q < nc; ++q)
                    potential = __dadd_rn(potential, __dmul_rn(static_cast<double>(cnt[q]), trial[q]));
                if (potential < best_potential) {
                    best_potential = potential;
                    best_index = pick_s;
                    flip_s ^= 1;  // swap(trial, best_trial)
                }
            }
            __syncthreads();
        }
        if (tid == 0) chosen[nch] = static_cast<uint32_t>(best_index);
        const double* bt = tb[flip_s];
        for (uint64_t q = tid; q < nc; q += blockDim.x) cdist2[q] = bt[q];  // swap(cdist2, best_trial)
        __syncthreads();
    }
    for (int i = tid; i < kMtN; i += blockDim.x) mt->x[i] = xs[i];
    if (tid == 0) {
        mt->pos = static_cast<uint64_t>(pos);
        *evals = ev;
    }
}

}  // namespace dev
}  // namespace bm
