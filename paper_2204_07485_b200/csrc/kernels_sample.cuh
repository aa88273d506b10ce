// kernels_sample.cuh — chunk sampling (Fisher-Yates resolution, device MT19937-64 draws) and the row gather.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

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
constexpr int kMtThreads = 32;

__device__ uint64_t mt_next_seq(uint64_t* x, int& pos) {
    if (pos >= kMtN) {
        for (int i = 0; i < kMtN; ++i) x[i] = mt_mix(x[i], x[(i + 1) % kMtN], x[(i + kMtM) % kMtN]);
        pos = 0;
    }
    return mt_temper(x[pos++]);
}

// Draw = k_mt_twist (one warp: the state recurrence, words stored untempered
// in consumption order) + k_mt_emit (all SMs: tempering and Lemire's
// multiply-shift per draw) + k_mt_fix (one thread: the exact sequential redo
// if any draw may have been rejected, or when forced).
//
// The twist as a stream: with W[0..312) the state, W[312 + i] = mix(W[i],
// W[i+1], W[i+156]) for every i >= 0 (the in-place twist reads x[j < i]
// already new).  A half-block H_k = W[156k .. 156k+156) depends only on
// H_{k-2} (element-aligned, and shifted by one: its last element pairs with
// H_{k-1}[0]) and H_{k-1} (element-aligned), so one warp keeps H_{k-2} and
// H_{k-1} in registers (lane l: elements 5l .. 5l+4; lane 31 holds element 155
// only) and produces H_k with two shuffles, no shared memory and no barrier:
// 320 dependent steps for a 50 000-word draw instead of 320 CTA barriers.
// `snap` receives the input state (host repairs after a speculative draw
// restart from it).
__global__ void __launch_bounds__(kMtThreads)
k_mt_twist(Mt64State* __restrict__ st, Mt64State* __restrict__ snap, uint32_t s, uint64_t* __restrict__ raw,
           int* __restrict__ flag) {
    const int lane = threadIdx.x;
    const int pos = static_cast<int>(st->pos);
    uint64_t a[5], b[5];  // H_{k-2}, H_{k-1}
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int e = 5 * lane + i;
        a[i] = e < kMtM ? st->x[e] : 0ull;
        b[i] = e < kMtM ? st->x[kMtM + e] : 0ull;
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int e = 5 * lane + i;
        if (e < kMtM) {
            snap->x[e] = a[i];
            snap->x[kMtM + e] = b[i];
        }
    }
    if (lane == 0) {
        snap->pos = static_cast<uint64_t>(pos);
        *flag = 0;
    }
    // words consumed: W[pos .. pos + s); T twists happen on the way
    const long long E = static_cast<long long>(pos) + static_cast<long long>(s);
    const long long T = E > kMtN ? (E - kMtN + kMtN - 1) / kMtN : 0;
    auto emit = [&](const uint64_t (&h)[5], long long k) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const int e = 5 * lane + i;
            const long long j = kMtM * k + e - pos;
            if (e < kMtM && j >= 0 && j < static_cast<long long>(s)) raw[j] = h[i];
        }
    };
    emit(a, 0);
    emit(b, 1);
    for (long long k = 2; k < 2 * (T + 1); ++k) {
        const uint64_t up = __shfl_down_sync(0xFFFFFFFFu, a[0], 1);  // H_{k-2}[5l + 5]
        const uint64_t b0 = __shfl_sync(0xFFFFFFFFu, b[0], 0);       // H_{k-1}[0]: follows H_{k-2}[155]
        uint64_t c[5];
        c[0] = mt_mix(a[0], lane == 31 ? b0 : a[1], b[0]);
        c[1] = mt_mix(a[1], a[2], b[1]);
        c[2] = mt_mix(a[2], a[3], b[2]);
        c[3] = mt_mix(a[3], a[4], b[3]);
        c[4] = mt_mix(a[4], up, b[4]);
        emit(c, k);
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            a[i] = b[i];
            b[i] = c[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int e = 5 * lane + i;
        if (e < kMtM) {
            st->x[e] = a[i];
            st->x[kMtM + e] = b[i];
        }
    }
    if (lane == 0) st->pos = static_cast<uint64_t>(E - kMtN * T);
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

}  // namespace dev
}  // namespace bm
