// kernels_control.cuh — Lloyd control, the accept and the deferred exact objectives.
// Part of the sm_100a multi-launch kernels (included, in order, by kernels.cuh;
// see its header for the bit-exactness contract).  Citations are relative to
// /root/reference/proj.
#pragma once

namespace bm {
namespace dev {

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

}  // namespace dev
}  // namespace bm
