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

// ===========================================================================
// 1. Chunk sampling: Fisher-Yates resolution of the host's raw draws.
//
// sample_chunk big_means.cpp:49-54 swaps idx[i] <-> idx[j_i] (j_i >= i) for
// i < s and returns sort(idx[0:s]).  Only the SET of the first s positions
// matters (it is sorted).  With W(t) = value at position t just before step t
// (W(t) = W(LT[t]) if LT[t] = max{t' < t : j_t' = t} exists, else t):
//   set ∩ [s,m) = { distinct j_t >= s }
//   set ∩ [0,s) = [0,s) \ { W(t_last(p)) : p >= s targeted, t_last = last step hitting p }
// (a value < s that ends at a position >= s is exactly the one left there by
// the last swap into that position).  All steps are data-parallel.
// ===========================================================================
__device__ __forceinline__ uint32_t hash_slot(uint32_t key, uint32_t hmask) {
    return (key * 2654435761u) & hmask;
}

// All tables are tagged with a per-draw epoch (epoch << 32 | payload): an entry
// of an older epoch reads as empty, so nothing is cleared between chunks.
//   LT[t]   = max{t' < t : j_t' = t}            (atomicMax on the tagged value)
//   hkey/hval: open-addressing map target p >= s -> last step hitting p
//   excl[v] = epoch  when value v < s leaves the first s positions
__device__ __forceinline__ unsigned long long tag(uint32_t epoch, uint32_t v) {
    return (static_cast<unsigned long long>(epoch) << 32) | v;
}

__global__ void k_fy_pass1(const uint32_t* __restrict__ js, const uint32_t* __restrict__ epoch_slot, uint32_t s,
                           unsigned long long* __restrict__ LT, unsigned long long* __restrict__ hkeys,
                           unsigned long long* __restrict__ hvals, uint32_t hmask) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s) return;
    const uint32_t ep = *epoch_slot;
    const uint32_t j = js[t];
    if (j < s) {
        if (j > t) atomicMax(&LT[j], tag(ep, t));
        return;
    }
    uint32_t h = hash_slot(j, hmask);
    const unsigned long long mine = tag(ep, j);
    while (true) {
        unsigned long long cur = hkeys[h];
        if ((cur >> 32) != ep) {  // stale: try to claim it for this epoch
            const unsigned long long prev = atomicCAS(&hkeys[h], cur, mine);
            if (prev != cur) continue;  // raced; re-examine this slot
            cur = mine;
        }
        if (cur == mine) {
            atomicMax(&hvals[h], tag(ep, t));
            return;
        }
        h = (h + 1) & hmask;
    }
}

__global__ void k_fy_pass2(const uint32_t* __restrict__ js, const uint32_t* __restrict__ epoch_slot, uint32_t s,
                           const unsigned long long* __restrict__ LT, const unsigned long long* __restrict__ hkeys,
                           const unsigned long long* __restrict__ hvals, uint32_t hmask,
                           uint32_t* __restrict__ exclbits, uint32_t* __restrict__ bitmap) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s) return;
    const uint32_t ep = *epoch_slot;
    const uint32_t j = js[t];
    if (j < s) return;
    const unsigned long long mine = tag(ep, j);
    uint32_t h = hash_slot(j, hmask);
    while (hkeys[h] != mine) h = (h + 1) & hmask;
    if (hvals[h] != tag(ep, t)) return;  // not the last swap into j
    atomicOr(&bitmap[j >> 5], 1u << (j & 31));
    uint32_t w = t;
    while (true) {
        const unsigned long long v = LT[w];
        if ((v >> 32) != ep) break;
        w = static_cast<uint32_t>(v);
    }
    atomicOr(&exclbits[w >> 5], 1u << (w & 31));
}

// Bitmap -> ascending index list (the std::sort of big_means.cpp:54).  Word q
// covers values 32q..32q+31: bits of values < s come from the exclusion table
// (kept unless excluded this epoch), bits of values >= s from the target
// bitmap, which the emit pass clears for the next chunk.
constexpr int kScanThreads = 256;
constexpr int kWordsPerThread = 8;
constexpr int kWordsPerBlock = kScanThreads * kWordsPerThread;

// The 8 words this thread owns (words base..base+7, base = 8 * global thread
// id): target bits (values >= s) OR'ed with the kept bits of values < s (not
// excluded this chunk).  Both bitmaps are cleared by the emit pass.
__device__ __forceinline__ void chunk_words(const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ exclbits,
                                            uint32_t s, uint32_t nwords, uint32_t words[kWordsPerThread]) {
    const uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * kWordsPerThread;
    const uint32_t low_words = (s + 31u) / 32u;
#pragma unroll
    for (int q = 0; q < kWordsPerThread; ++q) {
        const uint32_t w = base + q;
        uint32_t v = w < nwords ? bitmap[w] : 0u;
        if (w < low_words) {
            const uint32_t lim = s - w * 32u;
            const uint32_t lowmask = lim >= 32u ? 0xFFFFFFFFu : ((1u << lim) - 1u);
            v |= ~exclbits[w] & lowmask;
        }
        words[q] = v;
    }
}

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const uint32_t x = warp_tot[w];
            warp_tot[w] = run;
            run += x;
        }
        *total = run;
    }
    __syncthreads();
    return warp_tot[warp] + incl - v;
}

__global__ void k_bitmap_block_counts(const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ exclbits,
                                      uint32_t s, uint32_t nwords, uint32_t* __restrict__ block_counts) {
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    __shared__ uint32_t total;
    uint32_t words[kWordsPerThread];
    chunk_words(bitmap, exclbits, s, nwords, words);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kWordsPerThread; ++q) c += __popc(words[q]);
    block_exclusive_scan(c, warp_tot, &total);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = total;
}

__global__ void k_bitmap_emit(uint32_t* __restrict__ bitmap, uint32_t* __restrict__ exclbits, uint32_t s,
                              uint32_t nwords, const uint32_t* __restrict__ block_counts, uint32_t* __restrict__ out) {
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    __shared__ uint32_t total;
    __shared__ uint32_t block_off;
    if (threadIdx.x < 32) {  // this block's offset: sum of the preceding blocks' counts
        uint32_t acc = 0;
        for (uint32_t b = threadIdx.x; b < blockIdx.x; b += 32) acc += block_counts[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (threadIdx.x == 0) block_off = acc;
    }
    const uint32_t base = blockIdx.x * kWordsPerBlock + threadIdx.x * kWordsPerThread;
    uint32_t words[kWordsPerThread];
    chunk_words(bitmap, exclbits, s, nwords, words);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kWordsPerThread; ++q) c += __popc(words[q]);
    uint32_t pos = block_exclusive_scan(c, warp_tot, &total) + block_off;
#pragma unroll
    for (int q = 0; q < kWordsPerThread; ++q) {
        uint32_t w = words[q];
        if (base + q < nwords && bitmap[base + q]) bitmap[base + q] = 0u;  // ready for the next chunk
        if (base + q < (s + 31u) / 32u && exclbits[base + q]) exclbits[base + q] = 0u;
        while (w) {
            const int b = __ffs(w) - 1;
            out[pos++] = (base + q) * 32u + static_cast<uint32_t>(b);
            w &= w - 1;
        }
    }
}

__global__ void k_iota(uint32_t* __restrict__ out, uint32_t s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s) out[i] = i;
}

// Next epoch for host-drawn targets (bm_sample_chunk / bm_sample_chunk_draws).
__global__ void k_epoch_bump(uint32_t* counter, uint32_t* slot) {
    if (threadIdx.x == 0) *slot = ++(*counter);
}

// The s raw targets j_i = uniform_int(i, m-1) (big_means.cpp:49-51) drawn on
// the device from the device-resident std::mt19937_64 state.  A Lemire
// rejection (probability < 2^-32 per draw for m < 2^32) shifts every later
// draw; a possible one is detected and the whole draw is redone sequentially
// from the saved state with the exact rejection loop (also forced by
// `force_seq` in tests).
constexpr int kMtThreads = 320;

__device__ uint64_t mt_next_seq(uint64_t* x, int& pos) {
    if (pos >= kMtN) {
        for (int i = 0; i < kMtN; ++i) x[i] = mt_mix(x[i], x[(i + 1) % kMtN], x[(i + kMtM) % kMtN]);
        pos = 0;
    }
    return mt_temper(x[pos++]);
}

// Draw = k_mt_twist (one CTA: the state recurrence, words stored untempered
// in consumption order) + k_mt_emit (all SMs: tempering and Lemire's
// multiply-shift per draw) + k_mt_fix (one thread: the exact sequential redo
// if any draw may have been rejected, or when forced).  The twist is the
// in-place recurrence x[i] = mix(x[i], x[i+1], x[i+156]) with x[j<i] already
// new; double-buffered (A -> B) it is two data-parallel halves per 312 words.
// `snap` receives the input state (host repairs after a speculative draw
// restart from it).
__global__ void __launch_bounds__(kMtThreads)
k_mt_twist(Mt64State* __restrict__ st, Mt64State* __restrict__ snap, uint32_t s, uint64_t* __restrict__ raw,
           int* __restrict__ flag) {
    __shared__ uint64_t xa[kMtN], xb[kMtN];
    const int tid = threadIdx.x;
    for (int i = tid; i < kMtN; i += blockDim.x) {
        const uint64_t v = st->x[i];
        xa[i] = v;
        snap->x[i] = v;
    }
    int pos = static_cast<int>(st->pos);
    if (tid == 0) {
        snap->pos = static_cast<uint64_t>(pos);
        *flag = 0;
    }
    __syncthreads();
    uint64_t* A = xa;
    uint64_t* B = xb;
    uint32_t base = 0;
    if (pos < kMtN) {  // rest of the current block
        const uint32_t take = min(static_cast<uint32_t>(kMtN - pos), s);
        if (tid < static_cast<int>(take)) raw[tid] = A[pos + tid];
        pos += static_cast<int>(take);
        base = take;
    }
    while (base < s) {
        if (tid < kMtM) {
            const uint64_t v = mt_mix(A[tid], A[tid + 1], A[tid + kMtM]);
            B[tid] = v;
            if (base + tid < s) raw[base + tid] = v;
        }
        __syncthreads();
        if (tid >= kMtM && tid < kMtN) {
            const uint64_t v = mt_mix(A[tid], tid + 1 < kMtN ? A[tid + 1] : B[0], B[tid - kMtM]);
            B[tid] = v;
            if (base + tid < s) raw[base + tid] = v;
        }
        __syncthreads();
        uint64_t* t = A;
        A = B;
        B = t;
        const uint32_t take = min(static_cast<uint32_t>(kMtN), s - base);
        pos = static_cast<int>(take);
        base += take;
    }
    for (int i = tid; i < kMtN; i += blockDim.x) st->x[i] = A[i];
    if (tid == 0) st->pos = static_cast<uint64_t>(pos);
}

// j_i = uniform_int(i, m-1) from raw word i (Lemire, uniform_int_dist.h:252-331).
// low < r is necessary for a rejection (threshold (2^64-r) mod r < r); k_mt_fix
// applies the exact test sequentially when any draw sees it.
__global__ void k_mt_emit(const uint64_t* __restrict__ raw, uint64_t m, uint32_t s, uint32_t* __restrict__ js,
                          int* __restrict__ flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s) return;
    const uint64_t y = mt_temper(raw[i]);
    const uint64_t r = m - i;
    if (y * r < r) *flag = 1;
    js[i] = static_cast<uint32_t>(i + mul_hi64(y, r));
}

__global__ void k_mt_fix(Mt64State* __restrict__ st, const Mt64State* __restrict__ snap, uint64_t m, uint32_t s,
                         uint32_t* __restrict__ js, const int* __restrict__ flag, int force_seq,
                         uint32_t* __restrict__ epoch_counter, uint32_t* __restrict__ epoch_slot) {
    __shared__ uint64_t x[kMtN];
    if (threadIdx.x != 0) return;
    if (*flag || force_seq) {  // exact sequential redo from the input state
        for (int i = 0; i < kMtN; ++i) x[i] = snap->x[i];
        int p = static_cast<int>(snap->pos);
        for (uint32_t i = 0; i < s; ++i) {
            const uint64_t r = m - i;
            uint64_t y = mt_next_seq(x, p);
            uint64_t low = y * r;
            if (low < r) {
                const uint64_t thr = (0 - r) % r;
                while (low < thr) {
                    y = mt_next_seq(x, p);
                    low = y * r;
                }
            }
            js[i] = static_cast<uint32_t>(i + mul_hi64(y, r));
        }
        for (int i = 0; i < kMtN; ++i) st->x[i] = x[i];
        st->pos = static_cast<uint64_t>(p);
    }
    *epoch_slot = ++(*epoch_counter);  // tags the resolution tables of these targets
}

// ===========================================================================
// 2. Row gather (Dataset::gather core.cpp:34-44): one warp per output row,
//    16-byte vectors (rows are padded to 16-byte multiples).
// ===========================================================================
//    Xslot (when set) holds the dataset base: graphs captured once serve every
//    dataset of the same shape.
//    A grid of a few CTAs per SM strides over the chunk's 16-byte vectors
//    (every lane busy, four loads in flight per thread) instead of one warp
//    per row (17 of 32 lanes busy on c2) and thousands of short CTAs that
//    compete with the concurrent Lloyd kernels for SM slots.
__global__ void __launch_bounds__(256) k_gather(const uint4* __restrict__ X, const uint4* const* Xslot,
                                                uint32_t row_vecs, const uint32_t* __restrict__ idx, uint32_t s,
                                                uint4* __restrict__ out) {
    if (Xslot) X = *Xslot;
    const uint64_t total = static_cast<uint64_t>(s) * row_vecs;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < total; v0 += 4 * stride) {
        uint4 val[4];
        uint64_t dst[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint64_t v = v0 + r * stride;
            dst[r] = v;
            if (v < total) {
                const uint32_t row = static_cast<uint32_t>(v / row_vecs), col = static_cast<uint32_t>(v - static_cast<uint64_t>(row) * row_vecs);
                val[r] = __ldg(X + static_cast<uint64_t>(__ldg(idx + row)) * row_vecs + col);
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (dst[r] < total) out[dst[r]] = val[r];
    }
}

// Ordered fold of tile partials (block_sum outer loop core.cpp:172).
__device__ __forceinline__ double fold_tiles(const double* tiles, uint64_t ntiles) {
    double total = 0.0;
    uint64_t t = 0;
    for (; t + 8 <= ntiles; t += 8) {  // loads issued ahead of the dependent adds
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = __ldcg(tiles + t + r);  // written by other CTAs
#pragma unroll
        for (int r = 0; r < 8; ++r) total = __dadd_rn(total, v[r]);
    }
    for (; t < ntiles; ++t) total = __dadd_rn(total, __ldcg(tiles + t));
    return total;
}

// Left fold from 0.0 of a 16-byte aligned shared-memory array (one thread).
__device__ __forceinline__ double seq_fold_smem(const double* v, int len) {
    double a = 0.0;
    int i = 0;
    for (; i + 8 <= len; i += 8) {
        const double2 v0 = *reinterpret_cast<const double2*>(v + i);
        const double2 v1 = *reinterpret_cast<const double2*>(v + i + 2);
        const double2 v2 = *reinterpret_cast<const double2*>(v + i + 4);
        const double2 v3 = *reinterpret_cast<const double2*>(v + i + 6);
        a = __dadd_rn(a, v0.x); a = __dadd_rn(a, v0.y);
        a = __dadd_rn(a, v1.x); a = __dadd_rn(a, v1.y);
        a = __dadd_rn(a, v2.x); a = __dadd_rn(a, v2.y);
        a = __dadd_rn(a, v3.x); a = __dadd_rn(a, v3.y);
    }
    for (; i < len; ++i) a = __dadd_rn(a, v[i]);
    return a;
}

// ===========================================================================
// 6. Lloyd control (local_search.cpp:26-54), single thread.  Either its own
// kernel or run by the CTA that completes an assignment's last tile.
// ===========================================================================
__device__ __noinline__ void lloyd_begin_body(LloydStatus* st, const double* tiles, uint64_t ntiles, uint64_t rows,
                                 double* history, const int* n_active) {
    const double f = fold_tiles(tiles, ntiles);  // :27
    if (history) history[0] = f;                 // :28
    st->f = f;
    st->objective = f;
    st->evals = static_cast<unsigned long long>(rows) * *n_active;  // :26 counter
    st->iterations = 0;
    st->parity = 0;
    st->stop = 0;
    st->changed = 0;
    st->state_error = *n_active == 0;
    st->bad_label = 0;
}

__device__ __noinline__ void lloyd_step_body(LloydStatus* st, const double* tiles, uint64_t ntiles, uint64_t rows,
                                unsigned long long max_iterations, double rel_tolerance, double* history,
                                cudaGraphConditionalHandle cond, int use_cond, const int* n_active) {
    if (!st->stop) {
        const double f_new = fold_tiles(tiles, ntiles);  // :35
        st->evals += static_cast<unsigned long long>(rows) * *n_active;
        if (*n_active == 0) st->state_error = 1;
        st->iterations += 1;            // :36
        st->objective = f_new;          // history.push_back (:37)
        if (history) history[st->iterations] = f_new;
        const bool unchanged = __ldcg(&st->changed) == 0;  // :39 (set by other CTAs of this launch)
        st->changed = 0;
        st->parity = st->parity == 0 ? 1 : 0;  // :40-41 advance (the slot the assignment wrote)
        const double f = st->f;
        bool stop = unchanged;                                                      // :42-44
        if (!stop && f <= 0.0) stop = true;                                         // :45-47
        if (!stop && rel_tolerance > 0.0 && __ddiv_rn(__dsub_rn(f, f_new), f) < rel_tolerance)
            stop = true;                                                            // :48-50
        if (!stop) st->f = f_new;                                                   // :51
        if (st->iterations >= max_iterations) stop = true;                          // :32
        if (st->state_error || st->bad_label) stop = true;
        st->stop = stop ? 1 : 0;
    }
    if (use_cond) cudaGraphSetConditional(cond, st->stop ? 0u : 1u);  // graph WHILE node
}

__global__ void k_lloyd_begin(LloydStatus* st, const double* tiles, uint64_t ntiles, uint64_t rows,
                              double* history, const int* n_active) {
    if (threadIdx.x == 0) lloyd_begin_body(st, tiles, ntiles, rows, history, n_active);
}

__global__ void k_lloyd_step(LloydStatus* st, const double* tiles, uint64_t ntiles, uint64_t rows,
                             unsigned long long max_iterations, double rel_tolerance, double* history,
                             cudaGraphConditionalHandle cond, int use_cond, const int* n_active) {
    if (threadIdx.x == 0)
        lloyd_step_body(st, tiles, ntiles, rows, max_iterations, rel_tolerance, history, cond, use_cond, n_active);
}

// Accept step state (big_means.cpp:63-64, 89-94).
struct AcceptArgs {
    double* f_opt;
    double* C;
    uint8_t* mask;
    double* Cinc;
    uint8_t* maskinc;
    int k, n;
    Record* rec_base;
    unsigned long long* chunk_ctr;
    double* Cact;
    int ldc;
    int* act_idx;
    float* CT32;
    double* CactI;   // incumbent's compacted copy (speculative begins read it)
    int* actI;
    float* CT32I;
    GState* gs;
};

// Control fused into an assignment launch: mode 1 = begin, 2 = step.
struct LloydCtl {
    int mode;
    LloydStatus* st;
    GState* gs;
    unsigned* tiles_done;   // arrival counter over the launch's tiles
    uint64_t ntiles;
    unsigned long long max_iterations;
    double rel_tolerance;
    double* history;
    cudaGraphConditionalHandle cond;
    int use_cond;
    int fast;               // fast-sum control (no history; objective computed by k_accept)
    int force_exact;        // test hook: every fast-sum decision takes the exact path
    const double* dists_pair;  // distances of the last two assignments (slot = labels slot)
    uint64_t dstride;
    const int* go;          // when set and *go == 0 the launch does nothing (skipped chunk)
    int begin_kind;         // begin launches: 0 plain, 1 speculative (incumbent copy), 2 redo unless current
    int begin_slot;         // begin launches: the slot the assignment writes (parity after the begin)
    AcceptArgs acc;         // accept state (valid when has_acc)
    // exact-sum mode (sums != nullptr): per-label integer sums of the chunk's
    // points, updated by the assignment (§5b)
    long long* sums;        // this chunk buffer's two halves, each [kSMaxK][n] sums + [kSMaxK] counts
    uint64_t sum_half;      // elements per half
    double sum_scale;       // 2^-e: a stored value times this is an integer
    int sum_which;          // half the launch accumulates into: 0 / 1, or -1: st->sum_sel
    long long* parts;       // begins: per-CTA partial sums [CTA][kSMaxK * n + kSMaxK], merged per group of 8 CTAs
    unsigned* grp_ctr;      // begins: arrival counters of the groups (reset by each group's merger)
    uint64_t pts_rows;      // rows of the launch (point CTAs = ceil(rows / 128))
    int sum_small;          // per-CTA sums of the value units stay below 2^31 (32-bit shared accumulators)
    // exact-sum mode, fused update: the CTA that runs the control (or CTA 0 of
    // a begin that finds the speculative one current) computes the centroids
    // of the next round from the sums when the loop goes on (no k_centroids)
    int sum_fuse;
    double sum_unscale;
    unsigned nblk;          // point blocks when the CTAs loop over them (0: one block per CTA)
    int sum_cluster;        // begins launched as 8-CTA clusters: partials merged through distributed shared memory
    double* cC;
    uint8_t* cmask;
    double* cCact;
    int cldc;
    int* cact;
    int* cn_active;
    float* cCT32;
    float* cdelta;
    int has_acc;
    int accept_run;         // the control runs the accept (:89-94) when the loop stops
    LloydStatus* host_st;   // with acc: the status is also written to mapped host memory
    unsigned long long incomplete_after;  // > 0: no stop after this many rounds -> st->incomplete
    // begin launches with fixup CTAs: exact objective of the pending chunk
    const double* dists_all;  // [2 chunk buffers][2 slots][fix_rows]
    uint64_t fix_rows;
    double* fix_tiles;
};

// The status straight into mapped pinned host memory (no copy node); CTA-wide.
// The host reads it after synchronizing with the kernel's completion, which
// orders the writes (no system fence needed here).
__device__ __forceinline__ void status_to_host(const LloydStatus* st, LloydStatus* host_st) {
    constexpr int kW = sizeof(LloydStatus) / 8;
    for (int i = threadIdx.x; i < kW; i += blockDim.x)
        reinterpret_cast<volatile unsigned long long*>(host_st)[i] =
            reinterpret_cast<const volatile unsigned long long*>(st)[i];
}

// The accept of the chunk's candidate with its exact objective in
// st->objective (k_accept: all threads of one CTA; sm: 2k ints).
__device__ __noinline__ void accept_body(LloydStatus* st, const AcceptArgs& A, int accepted, LloydStatus* host_st,
                                         int* sm) {
    const int k = A.k, n = A.n;
    __shared__ int acc_s;
    __shared__ unsigned long long chunk_s;
    if (threadIdx.x == 0) {
        const unsigned long long chunk = *A.chunk_ctr;
        chunk_s = chunk;
        Record* rec = A.rec_base + chunk;
        if (accepted) *A.f_opt = st->objective;
        rec->candidate_objective = st->objective;
        rec->incumbent_objective = *A.f_opt;
        rec->chunk_index = chunk;
        rec->accepted = accepted;
        rec->degenerate_repaired = static_cast<unsigned long long>(A.gs->inc_degenerate);
        acc_s = accepted;
    }
    __syncthreads();
    accepted = acc_s;
    int* arank = sm;
    int* mk = sm + k;  // incumbent mask staged in shared memory (the rank loop below is serial)
    if (accepted) {
        for (int e0 = threadIdx.x; e0 < k * n; e0 += 8 * blockDim.x) {  // loads batched ahead of the stores
            double v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int e = e0 + r * blockDim.x;
                v[r] = e < k * n ? A.C[e] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int e = e0 + r * blockDim.x;
                if (e < k * n) A.Cinc[e] = v[r];
            }
        }
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const uint8_t v = A.mask[j];
            A.maskinc[j] = v;
            mk[j] = v;
        }
    } else {
        for (int j = threadIdx.x; j < k; j += blockDim.x) mk[j] = A.maskinc[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int dcount = 0, r = 0;
        for (int j = 0; j < k; ++j) {
            dcount += mk[j] ? 1 : 0;
            arank[j] = mk[j] ? -1 : r;
            if (!mk[j]) {
                A.act_idx[r] = j;
                if (accepted && A.actI) A.actI[r] = j;
                ++r;
            }
        }
        A.gs->inc_degenerate = dcount;
        A.gs->go = dcount == 0;
        A.gs->n_active = r;
        if (accepted) A.gs->n_active_inc = r;
        st->inc_degenerate = dcount;
        st->incomplete = 0;
        *A.chunk_ctr = chunk_s + 1;
    }
    __syncthreads();
    // the next chunk's start (:82): (C, mask) := incumbent, and its compacted form
    if (!accepted)
        for (int j = threadIdx.x; j < k; j += blockDim.x) A.mask[j] = static_cast<uint8_t>(mk[j]);
    for (int e0 = threadIdx.x; e0 < k * n; e0 += 8 * blockDim.x) {  // loads batched ahead of the stores
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x;
            v[r] = e < k * n ? A.Cinc[e] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x;
            if (e >= k * n) continue;
            const int j = e / n, d = e - j * n, rk = arank[j];
            if (!accepted) A.C[e] = v[r];
            if (rk < 0) continue;
            A.Cact[static_cast<uint64_t>(rk) * A.ldc + d] = v[r];
            if (A.CT32 && rk < kSMaxK) A.CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v[r]);
            if (accepted && A.CactI) {  // the incumbent's compacted copy
                A.CactI[static_cast<uint64_t>(rk) * A.ldc + d] = v[r];
                if (rk < kSMaxK) A.CT32I[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v[r]);
            }
        }
    }
    if (accepted) {  // published after the copy: a begin that saw the old version is redone
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.gs->inc_version), 1ull);
        }
    }
    if (host_st) {
        __syncthreads();
        status_to_host(st, host_st);
    }
}

// What the accept of the fused control reads, fetched by the last CTA in one
// round trip together with the status (shared memory; k <= kSMaxK).
struct TailIn {
    GState gs;                     // copy; fields this tail changes are written through to global
    unsigned long long chunk;      // *A.chunk_ctr
    unsigned char mk_inc[kSMaxK];  // incumbent mask
    unsigned char mk_cand[kSMaxK]; // candidate mask
    int arank[kSMaxK];             // label -> rank in the next start's compacted rows (-1: degenerate)
    int act[kSMaxK];               // rank -> label
    int na;                        // active labels of the next start
};

// The accept (:89-94) run by the fused control of the stopping round, with a
// deferred exact objective: the record's objectives are filled by fix_commit
// during the next chunk.  All threads of the CTA; inputs prefetched in T;
// stage: k x n doubles of shared memory holding the incumbent's centroids
// (cinc_staged), or room for them, or null.
__device__ __noinline__ void accept_fast(LloydStatus* st, const AcceptArgs& A, int accepted, TailIn* T,
                                         double* stage, bool cinc_staged) {
    const int k = A.k, n = A.n;
    const unsigned char* mk = accepted ? T->mk_cand : T->mk_inc;
    // Thread-serial code issues its global stores last: a generic load
    // behind an outstanding global store of the same thread waits for it.
    if (threadIdx.x < 32) {  // warp 0: ranks of the next start's active labels (k <= 32)
        const int lane = threadIdx.x;
        const bool live = lane < k && !mk[lane];
        const unsigned act = __ballot_sync(0xFFFFFFFFu, live);
        const int r = __popc(act & ((1u << lane) - 1u));
        if (lane < k) T->arank[lane] = live ? r : -1;
        if (live) {
            T->act[r] = lane;
            A.act_idx[r] = lane;
            if (accepted && A.actI) A.actI[r] = lane;
        }
        if (lane == 0) {
            const int na = __popc(act), dcount = k - na;
            T->na = na;
            const unsigned long long chunk = T->chunk;
            const unsigned long long repaired = static_cast<unsigned long long>(T->gs.inc_degenerate);
            const int par = st->parity;
            st->inc_degenerate = dcount;
            st->incomplete = 0;
            ktrace(11, 2);
            Record* rec = A.rec_base + chunk;
            rec->candidate_objective = __longlong_as_double(0x7FF8000000000000LL);
            rec->incumbent_objective = __longlong_as_double(0x7FF8000000000000LL);
            rec->chunk_index = chunk;
            rec->accepted = accepted;
            rec->degenerate_repaired = repaired;
            A.gs->pending_fix = static_cast<int>(chunk);
            A.gs->fix_par = par;
            A.gs->fix_acc = accepted;
            A.gs->inc_degenerate = dcount;
            A.gs->go = dcount == 0;
            A.gs->n_active = na;
            if (accepted) A.gs->n_active_inc = na;
            *A.chunk_ctr = chunk + 1;
            ktrace(9, 2);
        }
    }
    if (threadIdx.x < k) {  // accepted: incumbent mask := candidate's, else the next start's := incumbent's
        if (accepted) A.maskinc[threadIdx.x] = T->mk_cand[threadIdx.x];
        else A.mask[threadIdx.x] = T->mk_inc[threadIdx.x];
    }
    const int kn = k * n;
    if (stage && accepted)  // the candidate becomes the incumbent
        for (int e = threadIdx.x; e < kn; e += blockDim.x) stage[e] = __ldcg(A.C + e);
    __syncthreads();
    if (stage && (accepted || cinc_staged)) {
        // accepted: Cinc := C; the next chunk's start (:82) := incumbent; its
        // compacted forms row by row (Cact) and dimension by dimension (CT32,
        // [d][rank]), all coalesced
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5, na = T->na;
        for (int e = threadIdx.x; e < kn; e += blockDim.x) {
            if (accepted) A.Cinc[e] = stage[e];
            else A.C[e] = stage[e];
        }
        for (int rk = warp; rk < na; rk += nw) {
            const double* src = stage + T->act[rk] * n;
            for (int d = lane; d < n; d += 32) {
                A.Cact[static_cast<uint64_t>(rk) * A.ldc + d] = src[d];
                if (accepted && A.CactI) A.CactI[static_cast<uint64_t>(rk) * A.ldc + d] = src[d];
            }
        }
        if (A.CT32 && lane < na) {
            const double* src = stage + T->act[lane] * n;
            for (int d = warp; d < n; d += nw) {
                const float f = __double2float_rn(src[d]);
                A.CT32[static_cast<uint64_t>(d) * kSMaxK + lane] = f;
                if (accepted && A.CactI) A.CT32I[static_cast<uint64_t>(d) * kSMaxK + lane] = f;
            }
        }
    } else
    for (int e0 = threadIdx.x; e0 < kn; e0 += 8 * blockDim.x) {  // loads batched ahead of the stores
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x;
            v[r] = e >= kn ? 0.0 : accepted ? A.C[e] : A.Cinc[e];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x;
            if (e >= k * n) continue;
            const int j = e / n, d = e - j * n, rk = T->arank[j];
            if (accepted) A.Cinc[e] = v[r];
            else A.C[e] = v[r];
            if (rk < 0) continue;
            A.Cact[static_cast<uint64_t>(rk) * A.ldc + d] = v[r];
            if (A.CT32 && rk < kSMaxK) A.CT32[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v[r]);
            if (accepted && A.CactI) {  // the incumbent's compacted copy
                A.CactI[static_cast<uint64_t>(rk) * A.ldc + d] = v[r];
                if (rk < kSMaxK) A.CT32I[static_cast<uint64_t>(d) * kSMaxK + rk] = __double2float_rn(v[r]);
            }
        }
    }
    if (accepted) {  // published after the copy: a begin that saw the old version is redone
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.gs->inc_version), 1ull);
        }
    }
}

// The pending chunk's record gets its exact objective (thread 0; tiles: the
// ordered tile partials of its final distances).  fix_compute works on the
// state as read (gm: gs itself, or the tail's shared-memory copy, updated);
// fix_commit then writes the record and the state (stores last, see accept_fast).
struct FixOut {
    int pend;
    double fc, fo;
};

__device__ __forceinline__ bool fix_compute(GState* gm, const double* tiles, uint64_t ntiles, FixOut* o) {
    if (gm->pending_fix < 0) return false;
    double fc = 0.0;  // block_sum (:53-54): ordered fold of the tile partials (shared or fresh global memory)
    uint64_t t = 0;
    for (; t + 8 <= ntiles; t += 8) {
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = tiles[t + r];
#pragma unroll
        for (int r = 0; r < 8; ++r) fc = __dadd_rn(fc, v[r]);
    }
    for (; t < ntiles; ++t) fc = __dadd_rn(fc, tiles[t]);
    o->pend = gm->pending_fix;
    o->fc = fc;
    o->fo = gm->fix_acc ? fc : gm->fopt_exact;  // :89-93
    gm->fopt_exact = o->fo;
    gm->pending_fix = -1;
    return true;
}

__device__ __forceinline__ void fix_commit(GState* gs, const AcceptArgs& A, const FixOut& o) {
    Record* rec = A.rec_base + o.pend;
    rec->candidate_objective = o.fc;
    rec->incumbent_objective = o.fo;
    *A.f_opt = o.fo;
    gs->fopt_exact = o.fo;
    gs->pending_fix = -1;
}

// block_sum (core.cpp:165-175) by one thread: ordered tile folds, ordered fold of the tiles.
__device__ __noinline__ double exact_block_sum(const double* v, uint64_t count) {
    double total = 0.0;
    for (uint64_t t0 = 0; t0 < count; t0 += kTile) {
        const uint64_t e = min(count, t0 + kTile);
        double a = 0.0;
        for (uint64_t i = t0; i < e; ++i) a = __dadd_rn(a, __ldcg(v + i));
        total = __dadd_rn(total, a);
    }
    return total;
}

// Fast-sum Lloyd control (thread 0 of the CTA that arrived last).  Returns the
// accept decision (0/1) when the loop stopped and the control runs the accept,
// else -1.  gm: the chain state as read (c.gs, or the tail's prefetched copy).
__device__ __noinline__ int lloyd_fast_control(const LloydCtl& c, LloydStatus* st, uint64_t rows, unsigned ctas,
                                               int n_active, GState* gm, const double* fix_tiles) {
    const double s = st->fsum;
    st->fsum = 0.0;
    st->ctas_done = 0u;
    double lo, hi;
    sum_interval(s, rows, ctas, &lo, &hi);
    const double nan = __longlong_as_double(0x7FF8000000000000LL);
    if (c.mode == 1) {  // :26-28
        st->f = s;
        st->f_lo = lo;
        st->f_hi = hi;
        st->objective = nan;  // exact value: deferred (fix_compute / fix_commit)
        st->evals = static_cast<unsigned long long>(rows) * n_active;
        st->iterations = 0;
        st->parity = c.begin_slot;
        st->stop = 0;
        st->changed = 0;
        st->state_error = n_active == 0;
        st->bad_label = 0;
        st->exact_checks = 0;
        st->incomplete = 0;
        // which incumbent this assignment is valid for: a speculative begin is
        // current only if no accept published a new incumbent since its CTAs started
        const long long v = static_cast<long long>(__ldcg(reinterpret_cast<const unsigned long long*>(&c.gs->inc_version)));
        // (only a speculative begin's result may stand in for a later begin)
        st->begin_version = c.begin_kind == 1 && st->bv_min == v ? v : -1;
        st->sum_sel = c.begin_kind == 2 ? 1 : 0;  // exact-sum mode: the redo begin used the second half
        return -1;
    }
    // the previous chunk's record: its exact objective, before this chunk's accept
    ktrace(6, 2);
    FixOut fx;
    const bool fixed = c.has_acc && fix_tiles && fix_compute(gm, fix_tiles, tiles_of(c.fix_rows), &fx);
    ktrace(7, 2);
    int decision = -1;
    if (!st->stop) {
        st->evals += static_cast<unsigned long long>(rows) * n_active;
        if (n_active == 0) st->state_error = 1;
        st->iterations += 1;  // :36
        st->objective = nan;
        const bool unchanged = st->changed == 0;  // :39
        st->changed = 0;
        const int par = st->parity, out = par == 0 ? 1 : 0;
        st->parity = out;  // :40-41 (the slot this assignment wrote)
        bool stop = unchanged;  // :42-44
        if (!stop) {
            // f <= 0 (:45): terms are >= 0, so the exact f is 0 iff the fast sum is
            if (st->f <= 0.0) {
                stop = true;
            } else if (c.rel_tolerance > 0.0) {  // :48-50 on intervals
                const double flo = fmax(st->f_lo, 0x1p-1074), fhi = st->f_hi;
                bool decided = !c.force_exact && isfinite(fhi) && isfinite(hi);
                if (decided) {
                    const double a_lo = __dsub_rn(flo, hi), a_hi = __dsub_rn(fhi, lo);
                    const double g0 = __ddiv_rn(a_lo, flo), g1 = __ddiv_rn(a_lo, fhi);
                    const double g2 = __ddiv_rn(a_hi, flo), g3 = __ddiv_rn(a_hi, fhi);
                    const double gmin = fmin(fmin(g0, g1), fmin(g2, g3));
                    const double gmax = fmax(fmax(g0, g1), fmax(g2, g3));
                    if (gmax < c.rel_tolerance) stop = true;
                    else if (!(gmin >= c.rel_tolerance)) decided = false;
                }
                if (!decided) {  // exact block sums of both assignments
                    st->exact_checks += 1;
                    const double f = exact_block_sum(c.dists_pair + par * c.dstride, rows);
                    const double f_new = exact_block_sum(c.dists_pair + out * c.dstride, rows);
                    stop = __ddiv_rn(__dsub_rn(f, f_new), f) < c.rel_tolerance;
                }
            }
        }
        if (!stop) {  // :51
            st->f = s;
            st->f_lo = lo;
            st->f_hi = hi;
        }
        if (st->iterations >= c.max_iterations) stop = true;  // :32
        if (st->state_error || st->bad_label) stop = true;
        st->stop = stop ? 1 : 0;
        if (stop && c.accept_run) {  // accept (:89): f < f_opt, strict, on the candidate's interval
            const double fo = gm->fopt_exact;
            if (!c.force_exact && hi < fo) decision = 1;
            else if (!c.force_exact && !(lo < fo)) decision = 0;
            else decision = exact_block_sum(c.dists_pair + st->parity * c.dstride, rows) < fo;
        } else if (!stop && c.incomplete_after && st->iterations >= c.incomplete_after) {
            st->incomplete = 1;  // the host continues this chunk; the queued next chunk stays idle
            c.gs->go = 0;
        }
    }
    ktrace(8, 2);
    if (fixed) fix_commit(c.gs, c.acc, fx);
    if (c.use_cond) cudaGraphSetConditional(c.cond, st->stop ? 0u : 1u);
    return decision;
}

// Called by thread 0 of the CTA that folded a tile: the CTA completing the last
// tile runs the Lloyd control over all tile partials.
__device__ __forceinline__ void tile_done_control(const LloydCtl& c, const double* tiles, uint64_t rows) {
    if (!c.mode) return;
    __threadfence();
    const unsigned done = atomicAdd(c.tiles_done, 1u);
    if (done != c.ntiles - 1) return;
    __threadfence();
    *c.tiles_done = 0u;
    if (c.mode == 1) lloyd_begin_body(c.st, tiles, c.ntiles, rows, c.history, &c.gs->n_active);
    else lloyd_step_body(c.st, tiles, c.ntiles, rows, c.max_iterations, c.rel_tolerance, c.history, c.cond,
                         c.use_cond, &c.gs->n_active);
}

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

struct ScreenSmem {
    union {
        struct {
            float xs[2][kADC][kSXS];    // double-buffered fp32 point slabs [d][p]
            float cs[2][kADC][kSMaxK];  // double-buffered fp32 centroid slabs [d][j]
        } p1;
        struct {
            double item_d[kItemCap];
            short item_p[kItemCap];
            signed char item_j[kItemCap];
        } p2;
        double fold[kTile];
    } u;
    float Ls[kSMaxK][kABP];   // certified lower bounds [j][p]
    float red_u[8][kABP];
    float nx_lo[kABP], nx_hi[kABP], nxr[kABP];
    float nc_lo[kSMaxK], nc_hi[kSMaxK], ncr[kSMaxK];
    float umin[kABP];
    int icount[kABP];
    uint32_t n_items;
    int is_last;
};

template <typename T>
__global__ void __launch_bounds__(kSThreads, 3)
k_assign_screen(const T* __restrict__ X, uint64_t rows, int n, uint64_t ld,
                const double* __restrict__ Cact, int ldc, const int* __restrict__ act_idx,
                const int* __restrict__ n_active_ptr,
                int32_t* __restrict__ labels_pair, uint64_t pair_stride,
                const int* __restrict__ parity_ptr, double* __restrict__ dists_out,
                int* __restrict__ changed_flag, const int* __restrict__ stop_ptr,
                double* __restrict__ tile_out, unsigned* __restrict__ tile_counter,
                unsigned long long* __restrict__ cand_counter, ScreenConsts cst) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScreenSmem& S = *reinterpret_cast<ScreenSmem*>(smem_raw);

    if (stop_ptr && *stop_ptr) return;
    const int KA = *n_active_ptr;
    int32_t* labels_out = labels_pair;
    const int32_t* labels_old = nullptr;
    if (parity_ptr) {
        const int par = *parity_ptr;
        labels_out = labels_pair + (1 - par) * pair_stride;
        labels_old = labels_pair + par * pair_stride;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KG = (KA + kAK - 1) / kAK;
    const bool comp = warp < KG;
    const bool normw = warp == 7;
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * kABP;
    const int np = static_cast<int>(min(static_cast<uint64_t>(kABP), rows - p0));
    const float finf = __int_as_float(0x7F800000);
    const int nslab = (n + kADC - 1) / kADC;

    // ---------------- pass 1: fp32 screen, register-prefetched slabs ----------------
    T xr[8];
    double cr[2];
    auto load_slab = [&](int d0) {
        const int dl = min(kADC, n - d0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + kSThreads * i, p = e >> 4, d = e & 15;
            xr[i] = (p < np && d < dl) ? X[(p0 + p) * ld + d0 + d] : T(0);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + kSThreads * i, d = e >> 5, j = e & 31;
            cr[i] = (j < KA && d < dl) ? Cact[static_cast<uint64_t>(j) * ldc + d0 + d] : 0.0;
        }
    };
    auto store_slab = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + kSThreads * i;
            S.u.p1.xs[buf][e & 15][e >> 4] = static_cast<float>(xr[i]);  // round to nearest
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + kSThreads * i;
            S.u.p1.cs[buf][e >> 5][e & 31] = __double2float_rn(cr[i]);
        }
    };
    load_slab(0);
    store_slab(0);
    if (nslab > 1) load_slab(kADC);
    __syncthreads();

    float2 tot[2][kAK];  // points (4l, 4l+1) and (4l+2, 4l+3) x centroids 4w+u
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < kAK; ++u) tot[h][u] = make_float2(0.f, 0.f);
    float nxl[4] = {0.f, 0.f, 0.f, 0.f}, nxh[4] = {0.f, 0.f, 0.f, 0.f};
    float ncl = 0.f, nch = 0.f;

    for (int sl = 0; sl < nslab; ++sl) {
        const int buf = sl & 1, dl = min(kADC, n - sl * kADC);
        if (comp) {
            float2 part[2][kAK];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < kAK; ++u) part[h][u] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int d = 0; d < dl; ++d) {
                const float4 xv = *reinterpret_cast<const float4*>(&S.u.p1.xs[buf][d][4 * lane]);
                const float4 cv = *reinterpret_cast<const float4*>(&S.u.p1.cs[buf][d][4 * warp]);
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
                const float4 xv = *reinterpret_cast<const float4*>(&S.u.p1.xs[buf][d][4 * lane]);
                nxl[0] = __fmaf_rd(xv.x, xv.x, nxl[0]); nxh[0] = __fmaf_ru(xv.x, xv.x, nxh[0]);
                nxl[1] = __fmaf_rd(xv.y, xv.y, nxl[1]); nxh[1] = __fmaf_ru(xv.y, xv.y, nxh[1]);
                nxl[2] = __fmaf_rd(xv.z, xv.z, nxl[2]); nxh[2] = __fmaf_ru(xv.z, xv.z, nxh[2]);
                nxl[3] = __fmaf_rd(xv.w, xv.w, nxl[3]); nxh[3] = __fmaf_ru(xv.w, xv.w, nxh[3]);
                const float c = S.u.p1.cs[buf][d][lane];
                ncl = __fmaf_rd(c, c, ncl);
                nch = __fmaf_ru(c, c, nch);
            }
        }
        if (sl + 1 < nslab) {
            store_slab(buf ^ 1);  // buf^1 was released by the previous iteration's barrier
            if (sl + 2 < nslab) load_slab((sl + 2) * kADC);
        }
        __syncthreads();
    }
    if (normw) {
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
    // certified bounds
    if (comp) {
        float un[4] = {finf, finf, finf, finf};
#pragma unroll
        for (int u = 0; u < kAK; ++u) {
            const int j = kAK * warp + u;
            if (j >= KA) continue;
            const float cl = S.nc_lo[j], ch = S.nc_hi[j], crr = S.ncr[j];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int p = 4 * lane + q;
                const float sdot = q & 1 ? tot[q >> 1][u].y : tot[q >> 1][u].x;
                const float t2 = 2.f * sdot;  // exact
                const float Sn = __fadd_ru(S.nxr[p], crr);
                const float Al = __fadd_rd(S.nx_lo[p], cl), Ah = __fadd_ru(S.nx_hi[p], ch);
                float L = 0.f, U = finf;
                if (fabsf(t2) <= 1.0e37f && Sn <= 1.0e18f && Ah <= 1.0e37f) {
                    const float D = __fadd_ru(__fmul_ru(__fmul_ru(cst.K, Sn), Sn), cst.dabs);
                    L = fmaxf(__fsub_rd(__fsub_rd(Al, t2), D), 0.f);
                    L = __fmul_rd(L, cst.lo64);
                    U = __fmul_ru(__fadd_ru(__fsub_ru(Ah, t2), D), cst.hi64);
                }
                S.Ls[j][p] = L;
                un[q] = fminf(un[q], U);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) S.red_u[warp][4 * lane + q] = un[q];
    }
    __syncthreads();
    if (tid < kABP) {
        const int p = tid;
        float m = finf;
        for (int g = 0; g < KG; ++g) m = fminf(m, S.red_u[g][p]);
        S.umin[p] = m;
        int c = 0;
        if (p < np)
            for (int j = 0; j < KA; ++j) c += S.Ls[j][p] <= m;
        S.icount[p] = c;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 128 counts -> item offsets
        int v[4], run = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = S.icount[4 * tid + q];
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

    // ---------------- pass 2: exact fp64 recheck of the candidates ----------------
    if (!overflow) {
        if (tid < np) {
            const int p = tid;
            const float m = S.umin[p];
            uint32_t it = S.icount[p];
            for (int j = 0; j < KA; ++j)
                if (S.Ls[j][p] <= m) {
                    S.u.p2.item_p[it] = static_cast<short>(p);
                    S.u.p2.item_j[it] = static_cast<signed char>(j);
                    ++it;
                }
        }
        __syncthreads();
        for (uint32_t i = tid; i < NI; i += kSThreads) {
            const int p = S.u.p2.item_p[i], j = S.u.p2.item_j[i];
            const T* xrow = X + (p0 + p) * ld;
            const double* crow = Cact + static_cast<uint64_t>(j) * ldc;
            double a = 0.0;
            int d = 0;
            for (; d + 8 <= n; d += 8) {
                double xv[8], cv[8];
                if constexpr (sizeof(T) == 8) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 t = *reinterpret_cast<const double2*>(xrow + d + 2 * q);
                        xv[2 * q] = t.x;
                        xv[2 * q + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const float4 t = *reinterpret_cast<const float4*>(xrow + d + 4 * q);
                        xv[4 * q] = t.x;
                        xv[4 * q + 1] = t.y;
                        xv[4 * q + 2] = t.z;
                        xv[4 * q + 3] = t.w;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 t = __ldg(reinterpret_cast<const double2*>(crow + d + 2 * q));
                    cv[2 * q] = t.x;
                    cv[2 * q + 1] = t.y;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) a = dist_step(a, xv[q], cv[q]);
            }
            for (; d < n; ++d) a = dist_step(a, to_f64(xrow[d]), crow[d]);
            S.u.p2.item_d[i] = a;
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
                if (S.u.p2.item_d[i] < best) {
                    best = S.u.p2.item_d[i];
                    bj = S.u.p2.item_j[i];
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
        if (labels_old && labels_old[gp] != label) *changed_flag = 1;
    }
    if (!tile_out) return;
    // ---- fused tile fold: the last CTA of each 1024-point tile ----
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
    if (!S.is_last) return;
    __threadfence();
    const uint64_t tb = tile * kTile;
    const int len = static_cast<int>(min(rows, tb + kTile) - tb);
    double* fold = S.u.fold;
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
        tile_counter[tile] = 0u;  // ready for the next launch
    }
}

constexpr size_t screen_smem_bytes() { return sizeof(ScreenSmem); }

// ---------------------------------------------------------------------------
// 3c. Screened exact assignment, TMA pipeline (v5).  Same mathematics and
// results as k_assign_screen; only the data movement differs:
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
    if (nm == 0 && !(full && ctl.sum_cluster)) return;  // nothing moved in this CTA
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
    const bool clustered = full && ctl.sum_cluster;  // (every CTA of the cluster gets here, np may be 0)
    const bool grouped = full && ctl.parts && !clustered;
    long long* cpart = reinterpret_cast<long long*>(&S.lbs[0][0]);  // clustered: this CTA's partials
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
        if (clustered) cpart[e] = v;
        else if (grouped) slot[e] = v;
        else if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&sg[e]), static_cast<unsigned long long>(v));
    }
    if (clustered) {
        // The 8 CTAs of the cluster merge their partials through distributed
        // shared memory: CTA r sums elements [r E/8, (r+1) E/8) of all eight and
        // issues one atomic per nonzero element into copy (cluster % 8).
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        const int kn = kfull * n, E = kn + kfull;
        if (tid < kfull) cpart[kn + tid] = pc[tid + 1] - pc[tid];
        cl.sync();
        const int r = static_cast<int>(cl.block_rank());
        const int e0 = r * E / 8, e1 = (r + 1) * E / 8;
        const int cidx = static_cast<int>((blockIdx.x / 8) % kSumCopies);
        long long* csg = half + static_cast<uint64_t>(cidx) * kSMaxK * n;
        unsigned long long* ccnt = reinterpret_cast<unsigned long long*>(
            half + static_cast<uint64_t>(kSumCopies) * kSMaxK * n + cidx * kSMaxK);
        for (int e = e0 + tid; e < e1; e += blockDim.x) {
            long long v = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) v += *cl.map_shared_rank(cpart + e, q);
            if (v != 0) {
                if (e >= kn) atomicAdd(&ccnt[e - kn], static_cast<unsigned long long>(v));
                else atomicAdd(reinterpret_cast<unsigned long long*>(&csg[e]), static_cast<unsigned long long>(v));
            }
        }
        cl.sync();        // no CTA leaves (or reuses its shared memory) while others read it
        __threadfence();  // this CTA's atomics before its arrival
        return;
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
    const int tid = threadIdx.x;
    double(*c64)[kSMaxK][kCS] = reinterpret_cast<double(*)[kSMaxK][kCS]>(&S.xs[0][0][0]);
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
        const int st = (qb + sl) % NS, cb = (qb + sl) & 1;
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
    issue(0);
    if (nslab > 1) issue(1);
    for (int sl = 0; sl < nslab; ++sl) {
        const int q = qb + sl, st = q % NS, cb = q & 1;
        if (sl + 1 < nslab) cp_async_wait<1>();
        else cp_async_wait<0>();
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
        if (sl + 2 < nslab) issue(sl + 2);
    }
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
             uint64_t dstride) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
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
            if (NI > static_cast<uint32_t>(kSThreads)) {
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
    if (tid == 0)
        for (int i = 0; i < NS && i < nslab; ++i) issue(i);

    float2 tot[2][kAK];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < kAK; ++u) tot[h][u] = make_float2(0.f, 0.f);
    float nxl[4] = {0.f, 0.f, 0.f, 0.f}, nxh[4] = {0.f, 0.f, 0.f, 0.f};
    float ncl = 0.f, nch = 0.f;
    const int cp_ = tid & (kABP - 1), chalf = tid >> 7;  // conversion: point, 8-dim half

    for (int sl = 0; sl < nslab; ++sl) {
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
    qb += nslab;  // (the screen's slabs; a streamed recheck takes them again below)
    if (normw) {
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
    if (comp) {
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
    if (comp) {
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
        } else if (NI > static_cast<uint32_t>(kSThreads)) {
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
        if (!overflow) {  // ascending j, strict < (core.cpp:147)
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
    if (ctl.sums && (np > 0 || ctl.sum_cluster)) label_sums<T>(S, ctl, X, ld, n, p0, np, labels_old == nullptr, kfull, reuse,
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
