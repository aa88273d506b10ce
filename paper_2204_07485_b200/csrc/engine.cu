// engine.cu — host side of the B200-native Big-means hot path and its C-ABI.
//
// One host thread drives one chain on one device stream.  The host owns the
// reference RNG stream (std::mt19937_64 + the libstdc++ distributions, exactly
// the reference's Rng, common.hpp:13) and the few sequential decisions that
// depend on it (K-means++ CDF picks, init.cpp:171-198).  Everything else —
// Fisher-Yates resolution and sort of the sample, gather, assignment, update,
// Lloyd control, accept, final pass — runs on the device.
//
// Citations are relative to /root/reference/proj.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <set>
#include <thread>
#include <unordered_map>
#include <memory>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "bigmeans_b200.h"
#include "chunk.h"
#include "wide.h"
#include "finaltc.h"
#include "common.cuh"
#include "kernels.cuh"
#include "mt64.cuh"
#include "tma.cuh"

struct bm_rng {
    bm::Mt64 eng;  // Rng (common.hpp:13): std::mt19937_64 stream, libstdc++ distributions
};

namespace bm {

thread_local std::string g_last_error;
thread_local bm_profile g_profile{};
thread_local bool g_profiling = false;
thread_local std::vector<bm_chunk_record> g_last_trace;  // every record of the last big_means call

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------------------
// Device memory helpers
// ---------------------------------------------------------------------------
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) BM_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

template <class T>
struct HostBuf {  // pinned
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        release();
        n = count;
        if (count) BM_CUDA(cudaMallocHost(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
    ~HostBuf() { release(); }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        BM_CUDA(cudaGetDevice(&prev));
        if (prev != dev) BM_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Points view: rows x n, row stride ld elements, storage type dtype.
struct Points {
    const void* X;
    bm_dtype dtype;
    uint64_t rows;
    int n;
    uint64_t ld;
    bool tf32_exact = false;  // every value exactly a tf32 (wide rows: tensor-core pre-screen)
};

template <class F>
void dispatch(bm_dtype t, F&& f) {
    if (t == BM_F64) f(double{});
    else f(float{});
}

size_t dtype_size(bm_dtype t) { return t == BM_F64 ? 8 : 4; }

// Row stride: rows padded to 16-byte multiples for vector gathers.
uint64_t padded_ld(uint64_t n, bm_dtype t) {
    const uint64_t per16 = 16 / dtype_size(t);
    return ceil_div(n, per16) * per16;
}

// ---------------------------------------------------------------------------
// Workspace: every device buffer one chain needs, sized for (rows, k, n).
// ---------------------------------------------------------------------------
struct Workspace {
    uint64_t R = 0;  // max rows processed (chunk size s, or m)
    int k = 0, n = 0, ncand = 0;
    int ldc = 0;  // compacted-centroid row stride (even: 16-byte rows)
    uint64_t hist_cap = 0;
    uint64_t tiles = 0;

    DevBuf<int32_t> labels;  // 2 * R (ping-pong)
    DevBuf<double> dists;    // 4 * R
    DevBuf<double> fix_tiles;  // tiles: tile partials of a chunk's exact objective (deferred records)
    DevBuf<double> tile_buf; // max(ncand,1) * tiles
    DevBuf<unsigned> tile_ctr;  // tiles (fused tile-fold arrival counters)
    DevBuf<unsigned> tiles_done;  // tiles completed in the current assignment launch (fused control)
    DevBuf<double> psum;     // tiles * k * n
    DevBuf<double> C, Cact;  // k * n
    DevBuf<float> CT32;      // n * 32: fp32 compacted centroids, transposed [d][j] (TMA screen)
    CUtensorMap tm_ct{};     // tensor map of CT32
    // the incumbent's compacted copy (speculative begins of the next chunk read it)
    DevBuf<double> CactI;
    DevBuf<int> actI;
    DevBuf<float> CT32I;
    CUtensorMap tm_ctI{};
    DevBuf<dev::GState> gs;  // chain state shared by the chunk buffers
    DevBuf<uint8_t> mask;    // k
    DevBuf<int> act;         // k
    DevBuf<dev::LloydStatus> status;
    DevBuf<double> history;
    // certified bounds for the Lloyd-round fast path of the screened assignment
    DevBuf<float> lbk;       // R x 32: lower bound (distance units) of every (point, label) distance
    DevBuf<double> drift_part;  // [n][k]: squared centroid movement of the last update, per d-slab
    int drift_slabs = 0;        // d-slabs of the last update launch (host view at enqueue/capture time)
    DevBuf<float> delta;        // [k]: movement per label of the last update (distance units, rounded up)
    // exact-sum mode (graph chunks of exact-sum datasets): per chunk buffer two
    // halves (speculative begin / redo begin) of [kSMaxK][n] integer sums + [kSMaxK] counts
    DevBuf<long long> sums;
    bool sums_on = false;
    double sum_scale = 1.0, sum_unscale = 1.0;
    bool sums_fuse = false;  // the update runs in the control CTA of the previous launch (LloydCtl::sum_fuse)
    bool sum_small = false;  // per-CTA sums of the value units below 2^31 (bm_dataset::sum_units_max < 2^23)
    uint64_t sum_half() const { return (uint64_t)dev::kSumCopies * dev::kSMaxK * (n + 1); }
    long long* sums_of(int buf) { return sums.p + (uint64_t)buf * 2 * sum_half(); }
    DevBuf<long long> sum_parts;  // begins: per-CTA partials, per chunk buffer
    DevBuf<unsigned> grp_ctr;     // begins: group arrival counters, per chunk buffer
    uint64_t part_ctas() const { return (R + dev::kABP - 1) / dev::kABP; }
    uint64_t part_len() const { return (uint64_t)dev::kSMaxK * n + dev::kSMaxK; }
    DevBuf<unsigned> all_done;  // fused update: mergers finished
    DevBuf<unsigned> slab_ctr, slab_done, slab_tot;  // [n], [n], [n][k]: fused update counters / label totals
    // K-means++ (init.cpp:123-201)
    DevBuf<double> d2pool;   // (ncand + 1) * R
    DevBuf<uint32_t> cand;   // ncand
    DevBuf<Mt64State> ppmt;  // device K-means++: the RNG stream during the device steps
    DevBuf<dev::PPState> pps;
    DevBuf<long long> pprefix;  // R: exact integer prefix sums of the D^2 weights (per 1024-tile)
    DevBuf<long long> pptiles;  // tile totals
    // incumbent (big_means.cpp:63-64, 89-93)
    DevBuf<double> Cinc, fopt;
    DevBuf<uint8_t> maskinc;
    DevBuf<dev::Record> drec;              // per-chunk records (big_means trace)
    DevBuf<unsigned long long> chunk_ctr;  // device-side chunk index
    // persistent chunk kernel (chunk.cu): update partials, tile partials, grid
    // barrier, per-round sums / flags, per-chunk timing stamps
    DevBuf<double> cpart, ctiles, crsum, cdsum;
    DevBuf<int> cdcnt;
    DevBuf<unsigned> cpcnt, cbar;
    DevBuf<int> crchg;
    DevBuf<unsigned long long> ctiming;
    // wide rows (wide.cu): split-K partial dot products / norms per pool slot
    // (0..3: graph chunk buffers, 4: other calls, 5: the final pass), allocated
    // before any graph capture (ensure_wide)
    struct WideSlot {
        DevBuf<float> dot, nx, nc, bops;
        DevBuf<double> best;
        DevBuf<int> bj;
        const void* X = nullptr;
        uint64_t rows = 0, ld = 0;
        int n = 0;
        CUtensorMap map{}, map32{};  // the rows: 128-row boxes (screen), 32-row boxes (recheck)
        const double* C = nullptr;   // the centroid map's source
        int ck = 0, cn = 0, cld = 0, cnp = 0;
        CUtensorMap cmap{};
    } wide[6];
    struct ChunkMap {  // tensor map of chunk buffer i's rows for the current plan
        const void* X = nullptr;
        uint64_t rows = 0, ld = 0;
        int B = 0, xld = 0, n = 0;
        bool tc = false;
        bm_dtype dtype = BM_F64;
        CUtensorMap map{};
    } cmaps[dev::kStateBufs];
    DevBuf<dev::FixJob> cjob;              // [kStateBufs] deferred exact objectives
    DevBuf<unsigned long long> cfix_seq;   // chunks whose exact objective is final
    DevBuf<double> cfix_tiles;
    DevBuf<unsigned> cfix_ctr;
    cudaStream_t fix_stream = nullptr;
    cudaEvent_t ev_chunk[dev::kStateBufs] = {};
    void ensure_chunk(const ChunkPlan& p) {
        if (!cjob.n) {
            cjob.alloc(dev::kStateBufs);
            BM_CUDA(cudaMemset(cjob.p, 0, dev::kStateBufs * sizeof(dev::FixJob)));
            cfix_seq.alloc(1);
            BM_CUDA(cudaMemset(cfix_seq.p, 0, sizeof(unsigned long long)));
            cfix_ctr.alloc(1);
            BM_CUDA(cudaMemset(cfix_ctr.p, 0, sizeof(unsigned)));
            BM_CUDA(cudaStreamCreateWithFlags(&fix_stream, cudaStreamNonBlocking));
            for (auto& e : ev_chunk) BM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        if (cfix_tiles.n < tiles) cfix_tiles.alloc(std::max<uint64_t>(tiles, 1));
        const uint64_t kn = (uint64_t)k * n;
        if (cpart.n < kn * p.grid) cpart.alloc(kn * p.grid);
        if (cpcnt.n < (uint64_t)k * p.grid) cpcnt.alloc((uint64_t)k * p.grid);
        if (ctiles.n < 2 * tiles) ctiles.alloc(2 * tiles);
        if (!cbar.n) {
            cbar.alloc(4);
            BM_CUDA(cudaMemset(cbar.p, 0, 4 * sizeof(unsigned)));
            crsum.alloc(3);
            BM_CUDA(cudaMemset(crsum.p, 0, 3 * sizeof(double)));
            crchg.alloc(3);
            BM_CUDA(cudaMemset(crchg.p, 0, 3 * sizeof(int)));
        }
        if (cdsum.n < 3 * kn) {  // red mode: label-sum deltas, all zero between launches
            cdsum.alloc(3 * kn);
            BM_CUDA(cudaMemset(cdsum.p, 0, 3 * kn * sizeof(double)));
            cdcnt.alloc(3 * (uint64_t)k);
            BM_CUDA(cudaMemset(cdcnt.p, 0, 3 * (uint64_t)k * sizeof(int)));
        }
    }
    // CUDA graphs of one chunk (sample resolution + gather, and the Lloyd loop)
    std::string graph_sig;
    // graph mode: chunk c uses graphs [c % 4]: data and state buffer c % 4, draw buffer c % 2
    cudaGraphExec_t g_prep[dev::kStateBufs] = {};
    cudaGraphExec_t g_lloyd[dev::kStateBufs] = {};
    cudaGraphExec_t g_cont[dev::kStateBufs] = {};   // continuation of an incomplete chunk
    cudaGraphExec_t g_spec[dev::kStateBufs] = {};   // speculative begin (first assignment against the incumbent's copy)
    cudaEvent_t ev_spec[dev::kStateBufs] = {};
    cudaStream_t cap1 = nullptr, cap2 = nullptr;  // capture streams of the IF and WHILE bodies
    cudaEvent_t ev_lloyd[dev::kStateBufs] = {};  // end of the Lloyd graph of the chunk in slot c % 4
    cudaEvent_t ev_prep[dev::kStateBufs] = {};   // its chunk gathered
    void drop_graphs() {
        for (auto* v : {&g_prep, &g_lloyd, &g_cont, &g_spec})
            for (auto& e : *v)
                if (e) {
                    cudaGraphExecDestroy(e);
                    e = nullptr;
                }
        graph_sig.clear();
    }
    ~Workspace() {
        drop_graphs();
        if (fix_stream) cudaStreamDestroy(fix_stream);
        for (auto e : ev_chunk)
            if (e) cudaEventDestroy(e);
        for (auto q : {cap1, cap2})
            if (q) cudaStreamDestroy(q);
        for (auto* v : {&ev_lloyd, &ev_prep, &ev_spec})
            for (auto e : *v)
                if (e) cudaEventDestroy(e);
    }
    // pinned host mirrors
    HostBuf<dev::LloydStatus> h_status;
    HostBuf<double> h_tiles;
    HostBuf<double> h_d2;
    HostBuf<uint8_t> h_mask;
    HostBuf<uint32_t> h_cand;
    HostBuf<Mt64State> h_mt;

    static void encode_ct_map(CUtensorMap* map, float* base, int n) {
        auto enc = tmap_encoder();
        if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
        const cuuint64_t dims[2] = {(cuuint64_t)dev::kSMaxK, (cuuint64_t)n};
        const cuuint64_t strides[1] = {(cuuint64_t)dev::kSMaxK * sizeof(float)};
        const cuuint32_t box[2] = {(cuuint32_t)dev::kSMaxK, (cuuint32_t)dev::kADC};
        const cuuint32_t es[2] = {1, 1};
        if (enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            throw CudaError("cuTensorMapEncodeTiled(centroids) failed");
    }
    void init(uint64_t rows, int k_, int n_, int ncand_, uint64_t hist) {
        R = rows;
        k = k_;
        n = n_;
        ncand = std::max(ncand_, 1);
        ldc = n + (n & 1);
        tiles = tiles_of(rows);
        hist_cap = hist;
        labels.alloc(3 * dev::kStateBufs * R);  // [chunk buffer][slot 0..2][R] (non-graph paths: buffer 0, slots 0/1)
        dists.alloc(3 * dev::kStateBufs * R);   // [chunk buffer][slot 0..2][R], like the labels
        fix_tiles.alloc(std::max<uint64_t>(tiles, 1));
        lbk.alloc(dev::kStateBufs * R * dev::kSMaxK);  // per chunk buffer
        tile_buf.alloc(tiles * ncand);
        tile_ctr.alloc(tiles);
        if (tiles) BM_CUDA(cudaMemset(tile_ctr.p, 0, tiles * sizeof(unsigned)));
        tiles_done.alloc(1);
        BM_CUDA(cudaMemset(tiles_done.p, 0, sizeof(unsigned)));
        psum.alloc((tiles + (tiles & 1)) * (uint64_t)k * n);
        C.alloc((uint64_t)k * n);
        drift_part.alloc((uint64_t)n * k * 8);  // [slabs x mergers][k], slabs x mergers <= n * 8
        BM_CUDA(cudaMemset(drift_part.p, 0, (uint64_t)n * k * 8 * sizeof(double)));
        slab_ctr.alloc(n);
        BM_CUDA(cudaMemset(slab_ctr.p, 0, n * sizeof(unsigned)));
        delta.alloc(k);
        BM_CUDA(cudaMemset(delta.p, 0, k * sizeof(float)));
        all_done.alloc(1);
        BM_CUDA(cudaMemset(all_done.p, 0, sizeof(unsigned)));
        slab_done.alloc(n);
        BM_CUDA(cudaMemset(slab_done.p, 0, n * sizeof(unsigned)));
        slab_tot.alloc((uint64_t)n * k);
        BM_CUDA(cudaMemset(slab_tot.p, 0, (uint64_t)n * k * sizeof(unsigned)));
        Cact.alloc((uint64_t)k * (n + (n & 1)));
        CactI.alloc((uint64_t)k * (n + (n & 1)));
        if (k <= dev::kSMaxK) {
            CT32.alloc((uint64_t)n * dev::kSMaxK);
            BM_CUDA(cudaMemset(CT32.p, 0, (uint64_t)n * dev::kSMaxK * sizeof(float)));
            encode_ct_map(&tm_ct, CT32.p, n);
            CT32I.alloc((uint64_t)n * dev::kSMaxK);
            BM_CUDA(cudaMemset(CT32I.p, 0, (uint64_t)n * dev::kSMaxK * sizeof(float)));
            encode_ct_map(&tm_ctI, CT32I.p, n);
        }
        mask.alloc(k);
        act.alloc(k);
        actI.alloc(k);
        status.alloc(dev::kStateBufs);  // per chunk buffer (non-graph paths: [0])
        BM_CUDA(cudaMemset(status.p, 0, dev::kStateBufs * sizeof(dev::LloydStatus)));
        gs.alloc(1);
        BM_CUDA(cudaMemset(gs.p, 0, sizeof(dev::GState)));
        history.alloc(hist_cap);
        d2pool.alloc((uint64_t)(ncand + 1) * R);
        cand.alloc(ncand);
        Cinc.alloc((uint64_t)k * n);
        fopt.alloc(1);
        maskinc.alloc(k);
        chunk_ctr.alloc(1);
        h_status.alloc(dev::kStateBufs);  // per chunk buffer of the pipelined loop
        h_tiles.alloc(tiles * ncand);
        h_d2.alloc(R);
        h_mask.alloc(k);
        h_cand.alloc(ncand);
        h_mt.alloc(1);
    }
};

// Sampler workspace (sample_chunk big_means.cpp:39-56) for one dataset size m.
struct SamplerWs {
    uint64_t m = 0, s = 0;
    uint32_t hmask = 0;
    uint32_t nwords = 0, nblocks = 0;
    DevBuf<uint32_t> js, js2, bitmap, blockcnt, idx;  // js2: second target buffer (pipelined draws)
    DevBuf<unsigned long long> hkeys, hvals, LT;      // epoch-tagged resolution tables
    DevBuf<uint32_t> exclbits;                        // values < s leaving the first s positions
    // Resolution tables (set 0 = the members above; set 1 = a second copy):
    // the graph pipeline resolves odd chunks (target buffer 1) in set 1 on a
    // second prep stream, so that two chunks' preps overlap.  Each set sees
    // increasing epochs (the draws into its target buffer).
    struct Tabs {
        uint32_t *bitmap, *blockcnt, *idx, *exclbits;
        unsigned long long *hkeys, *hvals, *LT;
    };
    DevBuf<uint32_t> bitmap1, blockcnt1, idx1, exclbits1;
    DevBuf<unsigned long long> hkeys1, hvals1, LT1;
    Tabs tabs(int set) {
        if (set && !idx1.n) {  // allocated on first use (graph pipeline only)
            const size_t h = (size_t)hmask + 1;
            hkeys1.alloc(h);
            hvals1.alloc(h);
            BM_CUDA(cudaMemset(hkeys1.p, 0, h * sizeof(unsigned long long)));
            BM_CUDA(cudaMemset(hvals1.p, 0, h * sizeof(unsigned long long)));
            bitmap1.alloc(nwords);
            BM_CUDA(cudaMemset(bitmap1.p, 0, nwords * sizeof(uint32_t)));
            blockcnt1.alloc(std::max<uint32_t>(nblocks, 1));
            idx1.alloc(s);
            LT1.alloc(s);
            BM_CUDA(cudaMemset(LT1.p, 0, s * sizeof(unsigned long long)));
            exclbits1.alloc(ceil_div(s, 32));
            BM_CUDA(cudaMemset(exclbits1.p, 0, ceil_div(s, 32) * sizeof(uint32_t)));
        }
        if (set) return Tabs{bitmap1.p, blockcnt1.p, idx1.p, exclbits1.p, hkeys1.p, hvals1.p, LT1.p};
        return Tabs{bitmap.p, blockcnt.p, idx.p, exclbits.p, hkeys.p, hvals.p, LT.p};
    }
    DevBuf<uint32_t> epoch;                           // [0] counter, [1+b] epoch of target buffer b
    cudaStream_t rng_stream = nullptr;                      // device draws of the next chunk
    cudaEvent_t drawn[2] = {nullptr, nullptr}, resolved[2] = {nullptr, nullptr};
    DevBuf<Mt64State> mt;           // [0] device-resident RNG stream, [1+b] input state of the draw into buffer b
    DevBuf<uint64_t> raw;           // untempered words of the current draw
    DevBuf<int> mtflag;             // a draw may have been rejected (k_mt_fix redoes it)
    DevBuf<const void*> xslot;      // dataset base read by the prep graphs' gather
    HostBuf<Mt64State> h_mt;
    HostBuf<uint32_t> h_js[2];
    cudaEvent_t js_done[2] = {nullptr, nullptr};
    int cur = 0;

    void init(uint64_t m_, uint64_t s_) {
        m = m_;
        s = s_;
        uint32_t h = 1;
        while (h < 2 * s) h <<= 1;
        hmask = h - 1;
        nwords = (uint32_t)ceil_div(m, 32);
        nblocks = (uint32_t)ceil_div(nwords, dev::kWordsPerBlock);
        js.alloc(s);
        js2.alloc(s);
        hkeys.alloc(h);
        hvals.alloc(h);
        BM_CUDA(cudaMemset(hkeys.p, 0, h * sizeof(unsigned long long)));
        BM_CUDA(cudaMemset(hvals.p, 0, h * sizeof(unsigned long long)));
        bitmap.alloc(nwords);
        blockcnt.alloc(std::max<uint32_t>(nblocks, 1));
        idx.alloc(s);
        LT.alloc(s);
        exclbits.alloc(ceil_div(s, 32));
        epoch.alloc(3);
        BM_CUDA(cudaMemset(LT.p, 0, s * sizeof(unsigned long long)));
        BM_CUDA(cudaMemset(exclbits.p, 0, ceil_div(s, 32) * sizeof(uint32_t)));
        BM_CUDA(cudaMemset(epoch.p, 0, 3 * sizeof(uint32_t)));
        BM_CUDA(cudaMemset(bitmap.p, 0, nwords * sizeof(uint32_t)));
        mt.alloc(3);
        raw.alloc(s);
        mtflag.alloc(1);
        xslot.alloc(1);
        h_mt.alloc(1);
        for (int b = 0; b < 2; ++b) {
            h_js[b].alloc(s);
            if (!js_done[b]) BM_CUDA(cudaEventCreateWithFlags(&js_done[b], cudaEventDisableTiming));
            if (!drawn[b]) BM_CUDA(cudaEventCreateWithFlags(&drawn[b], cudaEventDisableTiming));
            if (!resolved[b]) BM_CUDA(cudaEventCreateWithFlags(&resolved[b], cudaEventDisableTiming));
        }
        if (!rng_stream) {  // highest priority: its single CTA must not wait behind full-GPU Lloyd kernels
            int lo = 0, hi = 0;
            BM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            BM_CUDA(cudaStreamCreateWithPriority(&rng_stream, cudaStreamNonBlocking, hi));
        }
    }
    uint32_t* jsbuf(int b) { return b ? js2.p : js.p; }
    uint32_t* epoch_slot(int b) { return epoch.p + 1 + b; }
    ~SamplerWs() {
        for (auto* arr : {js_done, drawn, resolved})
            for (int b = 0; b < 2; ++b)
                if (arr[b]) cudaEventDestroy(arr[b]);
        if (rng_stream) cudaStreamDestroy(rng_stream);
    }
};

}  // namespace bm

// Device-resident immutable dataset (Dataset core.hpp:13-37).  Immutable and
// shareable: all per-run state lives in the calling thread's DeviceCache.
struct bm_dataset {
    int device = 0;
    uint64_t m = 0, n = 0, ld = 0;
    bm_dtype dtype = BM_F64;
    void* X = nullptr;
    // exact-sum mode (kernels.cuh §5b): every value is a multiple of 2^sum_exp and
    // m * max|x| < 2^53 * 2^sum_exp, so label sums are exact in any order
    bool exact_sums = false;
    int sum_exp = 0;
    double sum_units_max = 0.0;  // max|x| / 2^sum_exp
    // fp32 storage whose every value is exactly a tf32 (11 significant bits):
    // the chunk kernel's tensor-core screen has a tight certified bound
    bool tf32_exact = false;
    cudaStream_t stream = nullptr;  // upload / download only
    ~bm_dataset() {  // X comes from the stream-ordered pool
        if (X) {
            if (stream) {
                cudaFreeAsync(X, stream);
                cudaStreamSynchronize(stream);
            } else {
                cudaFree(X);
            }
        }
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace bm {

// Per (host thread, device) workspaces and stream: one host thread drives one
// chain per device, several threads may share one dataset.
struct DeviceCache {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::map<std::tuple<uint64_t, int, int, int, uint64_t>, std::unique_ptr<Workspace>> ws;
    std::map<std::pair<uint64_t, uint64_t>, std::unique_ptr<SamplerWs>> sws;
    DevBuf<uint8_t> chunk;        // gathered chunk, s * ld * elem
    DevBuf<uint8_t> chunk1, chunk2, chunk3;  // graph mode: chunks c+1..c+3 are gathered while chunk c runs
    cudaStream_t pstream = nullptr;  // graph mode: prep (resolution + gather) of the coming even chunks
    cudaStream_t pstream2 = nullptr; // ... and of the odd chunks (their own resolution tables)
    cudaStream_t sstream = nullptr;  // graph mode: speculative begin of the next chunk
    DevBuf<int32_t> flabels;      // final pass
    DevBuf<double> fdists, ftiles;
    DevBuf<unsigned> fctr;
    ~DeviceCache() {
        ws.clear();
        sws.clear();
        if (stream) cudaStreamDestroy(stream);
        if (pstream) cudaStreamDestroy(pstream);
        if (pstream2) cudaStreamDestroy(pstream2);
        if (sstream) cudaStreamDestroy(sstream);
    }
    void ensure_final(uint64_t rows) {
        if (flabels.n < rows) flabels.alloc(rows);
        if (fdists.n < rows) fdists.alloc(rows);
        const uint64_t t = tiles_of(rows);
        if (ftiles.n < t) ftiles.alloc(t);
        if (fctr.n < t) {
            fctr.alloc(t);
            BM_CUDA(cudaMemset(fctr.p, 0, t * sizeof(unsigned)));
        }
    }
};

thread_local std::map<int, std::unique_ptr<DeviceCache>> t_cache;

DeviceCache& cache_of(int device) {
    auto it = t_cache.find(device);
    if (it != t_cache.end()) return *it->second;
    auto c = std::make_unique<DeviceCache>();
    c->device = device;
    // The engine stream (the chunk chain's critical path) gets a priority above
    // the speculative begins and chunk preps (default priority), the draw
    // stream stays highest.  BM_PRIO=0: default priority (A/B diagnostics).
    const bool prio = true;
    int lo = 0, hi = 0;
    BM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    BM_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio && hi < lo ? hi + 1 : lo));
    auto& ref = *c;
    t_cache.emplace(device, std::move(c));
    return ref;
}

cudaStream_t stream_of(const bm_dataset* d) { return cache_of(d->device).stream; }

}  // namespace bm

namespace bm {
namespace {

Points dataset_points(const bm_dataset* d) { return Points{d->X, d->dtype, d->m, (int)d->n, d->ld, d->tf32_exact}; }

Workspace& get_ws(const bm_dataset* d, uint64_t rows, int k, int ncand, uint64_t hist) {
    DeviceCache& c = cache_of(d->device);
    auto key = std::make_tuple(rows, k, (int)d->n, std::max(ncand, 1), hist);
    auto it = c.ws.find(key);
    if (it != c.ws.end()) return *it->second;
    auto w = std::make_unique<Workspace>();
    w->init(rows, k, (int)d->n, ncand, hist);
    auto& ref = *w;
    c.ws.emplace(key, std::move(w));
    return ref;
}

// ---------------------------------------------------------------------------
// Kernel launch wrappers
// ---------------------------------------------------------------------------
// CUDA-event timing of the launch groups of one big_means call (roofline and
// step-share reporting): events are recorded on the engine stream around
// every launch group while profiling is enabled.
enum Phase { PH_ASSIGN = 0, PH_FINAL, PH_UPDATE, PH_SAMPLE, PH_GATHER, PH_KMEANSPP, PH_CONTROL, PH_COUNT };

struct Profiler {
    std::vector<cudaEvent_t> pool;  // reused across calls: no per-launch creation
    size_t used = 0;
    std::vector<uint64_t> rows;
    std::vector<int> kind;
    cudaStream_t stream = nullptr;
    unsigned long long* d_cand = nullptr;  // [0] screened candidates, [1] screened rows
    void begin(cudaStream_t s) {
        stream = s;
        used = 0;
        rows.clear();
        kind.clear();
        if (!d_cand) BM_CUDA(cudaMalloc(&d_cand, 2 * sizeof(unsigned long long)));
        BM_CUDA(cudaMemsetAsync(d_cand, 0, 2 * sizeof(unsigned long long), s));
    }
    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            BM_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    std::pair<cudaEvent_t, cudaEvent_t> record_start() {
        cudaEvent_t a = next(), b = next();
        BM_CUDA(cudaEventRecord(a, stream));
        return {a, b};
    }
    void record_end(std::pair<cudaEvent_t, cudaEvent_t> p, uint64_t r, int k) {
        BM_CUDA(cudaEventRecord(p.second, stream));
        rows.push_back(r);
        kind.push_back(k);
    }
    void flush(bm_profile& out) {
        for (size_t i = 0; i < rows.size(); ++i) {
            float ms = 0;
            BM_CUDA(cudaEventSynchronize(pool[2 * i + 1]));
            BM_CUDA(cudaEventElapsedTime(&ms, pool[2 * i], pool[2 * i + 1]));
            out.phase_ms[kind[i]] += ms;
            out.phase_count[kind[i]] += 1;
            if (kind[i] == PH_FINAL) {
                out.final_ms += ms;
                out.final_rows += rows[i];
            } else if (kind[i] == PH_ASSIGN) {
                out.assign_ms_total += ms;
                out.assign_launches += 1;
                out.assign_rows_total += rows[i];
            }
        }
        unsigned long long cand[2] = {0, 0};
        BM_CUDA(cudaMemcpyAsync(cand, d_cand, sizeof(cand), cudaMemcpyDeviceToHost, stream));
        BM_CUDA(cudaStreamSynchronize(stream));
        out.screen_candidates += cand[0];
        out.screen_rows += cand[1];
        used = 0;
        rows.clear();
        kind.clear();
    }
};
thread_local Profiler g_prof;

// RAII event bracket around a launch group (no-op unless profiling).
struct PhaseScope {
    int k;
    uint64_t r;
    std::pair<cudaEvent_t, cudaEvent_t> ev{};
    PhaseScope(int kind_, uint64_t rows_) : k(kind_), r(rows_) {
        if (g_profiling) ev = g_prof.record_start();
    }
    ~PhaseScope() {
        if (g_profiling) g_prof.record_end(ev, r, k);
    }
};


void count_launch(uint64_t n = 1) { g_profile.kernel_launches += n; }

// BM_PDL=0 disables programmatic dependent launch.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_PDL");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// Launch with programmatic stream serialization: the kernel's CTAs may start
// while the previous kernel on the stream drains; they wait for its completion
// (griddepcontrol.wait) before touching its results.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BM_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device maximum:
// raise it (never lower it) per (device, kernel), thread-safe (one host thread
// per GPU drives its own chain).
template <class F>
void set_max_smem(F* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    BM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& c = cur[std::make_pair(dev, reinterpret_cast<const void*>(fn))];
    if (bytes > c) {
        BM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        c = bytes;
    }
}

// The kernels that run beside the persistent chunk kernel (draws, sample
// resolution, gather, the deferred objective) ask for the maximum shared-memory
// carveout too: an SM then never has to drain and repartition L1 / shared
// memory between them and a chunk kernel that uses ~200 KB per CTA.
// (BM_CARVEOUT=0 leaves the default for A/B.)
void prefer_max_smem_carveout() {
    static const bool on = !(std::getenv("BM_CARVEOUT") && std::string(std::getenv("BM_CARVEOUT")) == "0");
    if (!on) return;
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    BM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert(dev).second) return;
    const void* ks[] = {reinterpret_cast<const void*>(dev::k_mt_twist), reinterpret_cast<const void*>(dev::k_mt_emit),
                        reinterpret_cast<const void*>(dev::k_mt_fix), reinterpret_cast<const void*>(dev::k_fy_pass1),
                        reinterpret_cast<const void*>(dev::k_fy_pass2),
                        reinterpret_cast<const void*>(dev::k_bitmap_block_counts),
                        reinterpret_cast<const void*>(dev::k_bitmap_emit),
                        reinterpret_cast<const void*>(dev::k_epoch_bump), reinterpret_cast<const void*>(dev::k_gather)};
    for (const void* k : ks)
        BM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    chunk_fix_prefer_max_smem();
}

int assign_threads(int k) {
    const int kg = std::min<int>(dev::kAMaxCG, (int)ceil_div(std::max(k, 1), dev::kAK));
    return dev::kAPG * kg;
}

// fp32 value of x rounded toward -inf / +inf (host-side constant setup)
float f_rd(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -INFINITY);
    return f;
}
float f_ru(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, INFINITY);
    return f;
}

dev::ScreenConsts screen_consts(int n) {
    const double u = std::ldexp(1.0, -24);
    auto gam = [&](double m) { return m * u / (1.0 - m * u); };
    const int nslab = (n + dev::kADC - 1) / dev::kADC;
    const double g16 = gam(std::min(n, dev::kADC));
    const double gb = g16 + gam(nslab) * (1.0 + g16);      // blocked dot-product error
    const double up = u * (1.0 + 4 * u) / (1.0 - u);         // input rounding, incl. x^ vs x norms
    const double K = gb / 2.0 + 2.0 * up + up * up;
    const double u64 = std::ldexp(1.0, -53);
    const double g64 = (n + 3) * u64 / (1.0 - (n + 3) * u64);
    dev::ScreenConsts c;
    c.K = f_ru(K * (1.0 + 1e-6));
    c.dabs = std::ldexp(1.0f, -40);
    c.lo64 = f_rd((1.0 - g64) * (1.0 - 4 * u64));
    c.hi64 = f_ru((1.0 + g64) * (1.0 + 4 * u64));
    return c;
}

// Tensor map of a points view: 2-D [rows][n] (stride ld), box 16 dims x 128 rows.
template <class T>
CUtensorMap points_map(const Points& P) {
    CUtensorMap m{};
    auto enc = tmap_encoder();
    if (!enc) throw CudaError("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)P.n, (cuuint64_t)P.rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(P.ld * sizeof(T))};
    const cuuint32_t box[2] = {(cuuint32_t)dev::kADC, (cuuint32_t)dev::kABP};
    const cuuint32_t es[2] = {1, 1};
    const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const auto sw = sizeof(T) == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if (enc(&m, dt, 2, const_cast<void*>(P.X), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(points) failed");
    return m;
}

// BM_STORAGE=native keeps fp64 datasets in fp64 even when fp32 is lossless.
bool narrow_storage() {
    static const bool on = [] {
        const char* e = std::getenv("BM_STORAGE");
        return !(e && std::string(e) == "native");
    }();
    return on;
}

// BM_SUMS=0 disables the exact-sum update (kernels.cuh §5b) for A/B checks.
bool exact_sums_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_SUMS");
        return !(e && std::string(e) == "0");
    }();
    return on;
}


// BM_HAMERLY=0 disables the bound-based Lloyd-round fast path (A/B checks).
bool hamerly_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_HAMERLY");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// BM_ASSIGN_MODE=exact forces the unscreened kernel (A/B parity checks).
bool screen_enabled(int k) {
    static const bool exact_forced = [] {
        const char* e = std::getenv("BM_ASSIGN_MODE");
        return e && std::string(e) == "exact";
    }();
    return !exact_forced && k <= dev::kSMaxK;
}

void launch_tile_sums(cudaStream_t st, const double* v, uint64_t count, uint64_t stride, int narrays,
                      double* tiles, const int* stop);

// Centroid source of an assignment (default: the working compacted rows; a
// speculative begin reads the incumbent's copy) and its bound storage.
struct AssignSrc {
    const double* Cact;
    const int* act;
    const int* n_active;
    const CUtensorMap* tmc;
    float* lbk;
};

// Diagnostics (library built with -DBM_WIDE_DBG, BM_WIDE_DBG=1): k_wide_screen
// CTA (0,0)'s per-atom stamps [4][64] (TMA issue, data landed, MMAs issued, retired).
unsigned long long* wide_dbg_buffer() {
    static unsigned long long* p = nullptr;
    if (!p && std::getenv("BM_WIDE_DBG")) {
        BM_CUDA(cudaMalloc(&p, 4 * 64 * sizeof(unsigned long long)));
        BM_CUDA(cudaMemset(p, 0, 4 * 64 * sizeof(unsigned long long)));
    }
    return p;
}

// BM_WIDE=0: wide rows keep k_assign_tma's own slab screen (A/B checks).
bool wide_enabled() {
    const char* e = std::getenv("BM_WIDE");
    return !(e && std::string(e) == "0");
}

// The tensor-core pre-screen applies to fp32 rows exact in tf32 that are too
// wide for the persistent chunk kernel (wide.cu).
bool use_wide(const Points& P, int k) {
    return wide_enabled() && P.dtype == BM_F32 && P.tf32_exact && P.n > 88 && k >= 1 && k <= 32 &&
           P.rows < (1ull << 31);
}

int current_device() {
    int d = 0;
    BM_CUDA(cudaGetDevice(&d));
    return d;
}

// Pool slot sized for `rows` (never during a capture: graphs are captured after ensure_wide).
void ensure_wide_slot(Workspace::WideSlot& ws, const WidePlan& wp) {
    if (ws.dot.n < wp.dot_floats()) ws.dot.alloc(wp.dot_floats());
    if (ws.nx.n < wp.nx_floats()) ws.nx.alloc(wp.nx_floats());
    if (ws.nc.n < wp.nc_floats()) ws.nc.alloc(wp.nc_floats());
    if (ws.bops.n < wp.bops_floats()) ws.bops.alloc(wp.bops_floats());
    const size_t rows = static_cast<size_t>(wp.tiles) * 128;
    if (ws.best.n < rows) ws.best.alloc(rows);
    if (ws.bj.n < rows) ws.bj.alloc(rows);
}

void ensure_wide(Workspace& w, const Points& P, int k) {
    if (!use_wide(P, k)) return;
    const WidePlan wp = wide_plan(current_device(), P.rows, P.n, k);
    if (!wp.ok) return;
    for (int i = 0; i < 5; ++i) ensure_wide_slot(w.wide[i], wp);
    (void)wide_dbg_buffer();  // (diagnostics: allocated before any capture)
}

// assign_nearest over P with the compacted centroids of ws (Cact/act/n_active).
// With tile_out the per-1024-row tile partials of the distances are produced
// too (fused into the screened kernel; a separate fold after the exact one).
void launch_assign(cudaStream_t st, const Points& P, Workspace& w, int k, int32_t* labels_pair,
                   uint64_t pair_stride, const int* parity, double* dists, int* changed,
                   const int* stop, bool final_pass = false, double* tile_out = nullptr,
                   unsigned* tile_ctr = nullptr, const dev::LloydCtl* ctl = nullptr, int hmode = 0,
                   uint64_t dstride = 0, unsigned extra_ctas = 0, const AssignSrc* src = nullptr,
                   int wide_slot = 4) {
    const dev::LloydCtl noctl{};
    const AssignSrc def{w.Cact.p, w.act.p, &w.gs.p->n_active, &w.tm_ct, w.lbk.p};
    const AssignSrc& S = src ? *src : def;
    bool fused_ctl = false;
    const unsigned grid = (unsigned)ceil_div(P.rows, dev::kABP) + extra_ctas;  // extra: fixup CTAs (TMA path)
    if (grid == 0) return;
    PhaseScope ps(final_pass ? PH_FINAL : PH_ASSIGN, P.rows);
    const bool screen = screen_enabled(k);
    dispatch(P.dtype, [&](auto tag) {
        using T = decltype(tag);
        if (screen && P.rows < (1ull << 31)) {
            fused_ctl = ctl && (tile_out || ctl->fast);
            // NS-stage TMA slab ring: 2 stages (3 CTAs per SM) for rows of up to
            // 8 slabs, 6 stages (2 CTAs per SM) for wide rows, whose CTAs stream
            // tens to hundreds of slabs each
            // wide fp32 rows exact in tf32: the dot products from the tensor-core
            // pre-screen (split-K over the dims, wide.cu); hmode 0 (no bound rows)
            dev::PreDots pd{};
            if (use_wide(P, k)) {
                const WidePlan wp = wide_plan(current_device(), P.rows, P.n, k);
                if (wp.ok) {
                    Workspace::WideSlot& ws = w.wide[final_pass ? 5 : wide_slot];
                    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                    BM_CUDA(cudaStreamIsCapturing(st, &cs));
                    if (cs == cudaStreamCaptureStatusNone) ensure_wide_slot(ws, wp);
                    else if (ws.dot.n < wp.dot_floats() || ws.nx.n < wp.nx_floats() || ws.nc.n < wp.nc_floats() ||
                             ws.bops.n < wp.bops_floats() || ws.best.n < P.rows)
                        throw CudaError("wide pre-screen buffers not allocated before the graph capture");
                    if (ws.X != P.X || ws.rows != P.rows || ws.n != P.n || ws.ld != P.ld) {
                        ws.map = wide_rows_map(P.X, P.rows, P.n, P.ld);
                        ws.map32 = wide_rows_map(P.X, P.rows, P.n, P.ld, 32);
                        ws.X = P.X;
                        ws.rows = P.rows;
                        ws.n = P.n;
                        ws.ld = P.ld;
                    }
                    dev::WideArgs wa{};
                    wa.xmap = ws.map;
                    wa.Cact = S.Cact;
                    wa.ldc = w.ldc;
                    wa.n_active = S.n_active;
                    wa.rows = P.rows;
                    wa.n = P.n;
                    wa.na = wp.na;
                    wa.bpa = wp.bpa;
                    wa.natoms = wp.natoms;
                    wa.dot = ws.dot.p;
                    wa.nx = ws.nx.p;
                    wa.nc = ws.nc.p;
                    wa.bops = ws.bops.p;
                    wa.stop = stop;
                    wa.go = ctl ? ctl->go : nullptr;
                    wa.dbg = wide_dbg_buffer();
                    launch_wide_screen(st, wp, wa, pdl_enabled());
                    if (ws.C != S.Cact || ws.ck != k || ws.cn != P.n || ws.cld != w.ldc || ws.cnp != wp.np) {
                        ws.cmap = wide_cent_map(S.Cact, k, P.n, w.ldc, wp.np);
                        ws.C = S.Cact;
                        ws.ck = k;
                        ws.cn = P.n;
                        ws.cld = w.ldc;
                        ws.cnp = wp.np;
                    }
                    dev::RecheckArgs ra{};
                    ra.xmap = ws.map32;
                    ra.cmap = ws.cmap;
                    ra.X = static_cast<const float*>(P.X);
                    ra.ld = P.ld;
                    ra.rows = P.rows;
                    ra.n = P.n;
                    ra.Cact = S.Cact;
                    ra.ldc = w.ldc;
                    ra.n_active = S.n_active;
                    ra.dot = ws.dot.p;
                    ra.nx = ws.nx.p;
                    ra.nc = ws.nc.p;
                    ra.ks = wp.ks;
                    ra.natoms = wp.natoms;
                    ra.np = wp.np;
                    ra.cst = wide_screen_consts(wp, P.n);
                    ra.best = ws.best.p;
                    ra.bj = ws.bj.p;
                    ra.stop = stop;
                    ra.go = wa.go;
                    launch_wide_recheck(st, wp, ra, pdl_enabled());
                    count_launch(3);
                    pd = dev::PreDots{ws.best.p, ws.bj.p};
                    hmode = 0;
                }
            }
            auto go = [&](auto ns_tag) {
                constexpr int NS = decltype(ns_tag)::value;
                constexpr size_t shm = dev::tma_smem_bytes<T, NS>();
                set_max_smem(dev::k_assign_tma<T, NS>, shm);
                const CUtensorMap tmx = points_map<T>(P);
                const unsigned lgrid = grid;
                launch_pdl(dev::k_assign_tma<T, NS>, lgrid, dev::kSThreads, shm, st,
                    tmx, *S.tmc, static_cast<const T*>(P.X), P.rows, P.n, P.ld, S.Cact, w.ldc, S.act,
                    S.n_active, labels_pair, pair_stride, parity, dists, changed, stop, tile_out, tile_ctr,
                    g_profiling ? g_prof.d_cand : nullptr, screen_consts(P.n), fused_ctl ? *ctl : noctl,
                    !hamerly_enabled() || (hmode == 2 && w.drift_slabs == 0) ? 0 : hmode, S.lbk, w.delta.p, k,
                    dstride, pd);
            };
            if (P.n > 8 * dev::kADC) go(std::integral_constant<int, 6>{});
            else go(std::integral_constant<int, 2>{});
        } else {
            dev::k_assign<T><<<grid, assign_threads(k), 0, st>>>(
                static_cast<const T*>(P.X), P.rows, P.n, P.ld, w.Cact.p, w.ldc, w.act.p, &w.gs.p->n_active,
                labels_pair, pair_stride, parity, dists, changed, stop);
        }
    });
    BM_LAUNCH();
    count_launch();
    if (tile_out && !screen) launch_tile_sums(st, dists, P.rows, 0, 1, tile_out, stop);
    if (ctl && ctl->mode && !fused_ctl) {  // control as its own kernel
        if (ctl->mode == 1)
            dev::k_lloyd_begin<<<1, 32, 0, st>>>(ctl->st, tile_out, ctl->ntiles, P.rows, ctl->history, S.n_active);
        else
            dev::k_lloyd_step<<<1, 32, 0, st>>>(ctl->st, tile_out, ctl->ntiles, P.rows, ctl->max_iterations,
                                                ctl->rel_tolerance, ctl->history, ctl->cond, ctl->use_cond,
                                                S.n_active);
        BM_LAUNCH();
        count_launch();
    }
}

void launch_tile_sums(cudaStream_t st, const double* v, uint64_t count, uint64_t stride, int narrays,
                      double* tiles, const int* stop) {
    const uint64_t blocks = tiles_of(count) * narrays;
    if (blocks == 0) return;
    launch_pdl(dev::k_tile_sums, (unsigned)blocks, 256, 0, st, v, count, stride, narrays, tiles, stop);
    BM_LAUNCH();
    count_launch();
}

void launch_compact(cudaStream_t st, Workspace& w, const double* C, const uint8_t* mask) {
    dev::k_compact<<<1, 256, w.k * sizeof(int), st>>>(C, mask, w.k, w.n, w.Cact.p, w.ldc, w.act.p,
                                                       &w.gs.p->n_active, w.CT32.p);
    BM_LAUNCH();
    count_launch();
}

// update_centroids (core.cpp:183-244) in one launch: grid (tile, d-slab), the
// slab's last CTA merges it.  Slabs split the dimensions so that the grid
// covers the GPU when there are few tiles and the staged slab fits in shared memory.
void launch_update(cudaStream_t st, const Points& P, Workspace& w, const int* parity, const int* stop,
                   const int* go = nullptr, int32_t* labels = nullptr, int* bad_label = nullptr) {
    PhaseScope ps(PH_UPDATE, P.rows);
    const int k = w.k, n = w.n;
    const uint64_t tiles = tiles_of(P.rows);
    if (tiles == 0) return;
    const size_t es = dtype_size(P.dtype);
    const int V = (int)(16 / es);  // staged rows are whole 16-byte vectors
    const size_t base = ((size_t)(kTile / 2 + (2 + dev::kUWarps) * k) * 4 + 15) & ~size_t(15);
    // about two CTAs per SM in one wave; the staged slab within ~100 KB of shared memory
    int slabs = (int)std::max<uint64_t>(1, std::min<uint64_t>((296 + tiles / 2) / tiles, ceil_div(n, V)));
    int dslab = (int)(ceil_div(ceil_div(n, slabs), V) * V);
    while (dslab > V && base + (size_t)kTile * dslab * es > 100 * 1024) dslab -= V;
    slabs = (int)ceil_div(n, dslab);
    const uint64_t tstride = tiles + (tiles & 1);
    const size_t merge_min = ((((size_t)2 * k * 4 + 15) & ~size_t(15)) + (size_t)k * dslab * 8 + 15) / 16 * 16 +
                             (tstride + 1) * 8 * 16;  // at least 16 (dim, label) pairs per merge round
    const size_t shm = std::max(base + (size_t)kTile * dslab * es, merge_min);
    dim3 grid((unsigned)tiles, (unsigned)slabs);
    // mergers per slab: about 48 (dim, label) pairs each
    // (waiting mergers never exceed one per SM, so the CTAs they wait for always get a slot)
    int G = (int)std::min<uint64_t>({tiles, (uint64_t)8, std::max<uint64_t>(1, ceil_div((uint64_t)k * dslab, 48))});
    while (G > 1 && (uint64_t)G * slabs > 148) --G;
    dev::UpdateArgs u{w.psum.p, tstride, shm, w.slab_ctr.p, w.slab_done.p, G, go, w.all_done.p, w.delta.p, w.slab_tot.p, w.C.p, w.mask.p, w.Cact.p, w.ldc,
                      w.act.p, &w.gs.p->n_active, w.CT32.p, w.drift_part.p,
                      bad_label ? bad_label : &w.status.p->bad_label, stop};
    dispatch(P.dtype, [&](auto tag) {
        using T = decltype(tag);
        if (shm > 48 * 1024) set_max_smem(dev::k_update<T>, shm);
        launch_pdl(dev::k_update<T>, grid, dev::kUThreads, shm, st, static_cast<const T*>(P.X), P.rows, n, P.ld,
                   labels ? labels : w.labels.p, w.R, parity, k, dslab, u);
    });
    BM_LAUNCH();
    count_launch(1);
    w.drift_slabs = slabs * G;
}

// update_centroids in exact-sum mode (kernels.cuh §5b): the label sums the
// assignments keep give the centroids directly (one CTA).
void launch_centroids(cudaStream_t st, Workspace& w, int buf, dev::LloydStatus* sts, const int* go) {
    PhaseScope ps(PH_UPDATE, 0);
    launch_pdl(dev::k_centroids, 1, 1024, 0, st, (const dev::LloydStatus*)sts, (const int*)&sts->stop, go,
               (const long long*)w.sums_of(buf), w.sum_half(), w.sum_unscale, w.k, w.n, w.C.p, w.mask.p, w.Cact.p,
               w.ldc, w.act.p, &w.gs.p->n_active, w.CT32.p, w.delta.p);
    BM_LAUNCH();
    count_launch(1);
    w.drift_slabs = 1;
}

// ---------------------------------------------------------------------------
// lloyd (local_search.cpp:16-60) with the loop state on the device.
// Start centroids in w.C / w.mask.  Kernels of a finished loop early-exit, so
// the host launches rounds in batches and checks the status once per batch.
// ---------------------------------------------------------------------------
struct LloydResult {
    double objective;
    uint64_t evals;
    uint64_t iterations;
    int parity;
};

// BM_FORCE_EXACT_CONTROL=1: every fast-sum stop test takes the exact path (test hook).
bool force_exact_control() {
    static const bool on = std::getenv("BM_FORCE_EXACT_CONTROL") != nullptr;
    return on;
}

dev::LloydCtl make_ctl(Workspace& w, int mode, uint64_t rows, uint64_t max_it = 0, double tol = 0.0,
                       cudaGraphConditionalHandle cond = 0, int use_cond = 0, bool fast = false) {
    dev::LloydCtl c{};
    c.fast = fast ? 1 : 0;
    c.force_exact = force_exact_control() ? 1 : 0;
    c.dists_pair = w.dists.p;
    c.dstride = w.R;
    c.mode = mode;
    c.st = w.status.p;
    c.gs = w.gs.p;
    c.tiles_done = w.tiles_done.p;
    c.ntiles = tiles_of(rows);
    c.max_iterations = max_it;
    c.rel_tolerance = tol;
    c.history = w.hist_cap ? w.history.p : nullptr;
    c.cond = cond;
    c.use_cond = use_cond;
    return c;
}

// compact (unless the compacted start is already in place) + assign (:26) +
// begin (:27-28), the latter fused into the assignment where possible.
// Graph-mode extras of a Lloyd launch sequence.
struct GraphRound {
    int buf = 0;                    // chunk buffer: labels/dists/bounds/status of this buffer
    const int* go = nullptr;        // skip everything when *go == 0
    int begin_kind = 0;             // begin: 1 speculative (incumbent copy), 2 redo unless current
    bool accept = false;            // the control runs the accept when the loop stops
    dev::LloydStatus* host_st = nullptr;
    unsigned long long incomplete_after = 0;
    bool fix = false;               // round 1: fixup CTAs for the previous chunk's record
};

// Per-buffer storage in graph mode: 3 slots of labels/distances (slot 2: the
// begin's assignment), bounds and status.
int32_t* gr_labels(Workspace& w, const GraphRound* g) { return w.labels.p + (g ? 3 * (uint64_t)g->buf * w.R : 0); }
double* gr_dists(Workspace& w, const GraphRound* g) { return w.dists.p + (g ? 3 * (uint64_t)g->buf * w.R : 0); }
dev::LloydStatus* gr_status(Workspace& w, const GraphRound* g) { return w.status.p + (g ? g->buf : 0); }
float* gr_lbk(Workspace& w, const GraphRound* g) {
    return w.lbk.p + (g ? (uint64_t)g->buf * w.R * dev::kSMaxK : 0);
}

dev::AcceptArgs accept_args(Workspace& w);

void apply_graph(dev::LloydCtl& c, Workspace& w, const GraphRound* g) {
    if (!g) return;
    c.dists_pair = gr_dists(w, g);
    c.st = gr_status(w, g);
    c.go = g->go;
    c.begin_kind = g->begin_kind;
    if (g->accept || g->fix) {
        c.acc = accept_args(w);
        c.has_acc = 1;
    }
    c.accept_run = g->accept ? 1 : 0;
    if (w.sums_on) {  // exact-sum mode: the begins fill a half, the rounds move points in the live one
        c.sums = w.sums_of(g->buf);
        c.sum_half = w.sum_half();
        c.sum_scale = w.sum_scale;
        c.sum_which = g->begin_kind == 1 ? 0 : g->begin_kind == 2 ? 1 : -1;
        if (g->begin_kind != 0) {
            c.parts = w.sum_parts.p + (uint64_t)g->buf * w.part_ctas() * w.part_len();
            c.grp_ctr = w.grp_ctr.p + (uint64_t)g->buf * ceil_div(w.part_ctas(), (uint64_t)dev::kSumGroup);
            c.pts_rows = w.R;
        }
        c.sum_small = w.sum_small ? 1 : 0;
        if (w.sums_fuse && g->begin_kind != 1) {  // never the speculative begin: the working centroids are in use
            c.sum_fuse = 1;
            c.sum_unscale = w.sum_unscale;
            c.cC = w.C.p;
            c.cmask = w.mask.p;
            c.cCact = w.Cact.p;
            c.cldc = w.ldc;
            c.cact = w.act.p;
            c.cn_active = &w.gs.p->n_active;
            c.cCT32 = w.CT32.p;
            c.cdelta = w.delta.p;
        }
    }
    c.host_st = g->host_st;
    c.incomplete_after = g->incomplete_after;
    if (g->fix) {
        c.dists_all = w.dists.p;
        c.fix_rows = w.R;
        c.fix_tiles = w.fix_tiles.p;
    }
}

// compact (unless the compacted start is already in place) + assign (:26) +
// begin (:27-28), the latter fused into the assignment where possible.  In
// graph mode the begin's assignment goes to slot 2 of the chunk buffer.
void lloyd_enqueue_begin(cudaStream_t st, const Points& P, Workspace& w, bool do_compact = true,
                         bool fast = false, const GraphRound* g = nullptr) {
    if (do_compact) launch_compact(st, w, w.C.p, w.mask.p);
    dev::LloydCtl ctl = make_ctl(w, 1, P.rows, 0, 0.0, 0, 0, fast);
    apply_graph(ctl, w, g);
    const uint64_t slot = g ? 2 : 0;
    ctl.begin_slot = (int)slot;
    AssignSrc src{w.Cact.p, w.act.p, &w.gs.p->n_active, &w.tm_ct, gr_lbk(w, g)};
    if (g && g->begin_kind == 1) src = AssignSrc{w.CactI.p, w.actI.p, &w.gs.p->n_active_inc, &w.tm_ctI, gr_lbk(w, g)};
    launch_assign(st, P, w, w.k, gr_labels(w, g) + slot * w.R, 0, nullptr, gr_dists(w, g) + slot * w.R, nullptr,
                  nullptr, false, fast ? nullptr : w.tile_buf.p, w.tile_ctr.p, &ctl, 1, 0, 0u, &src, g ? g->buf : 4);
}

// update (:33) + assign (:34-35) + step (:36-51), the step fused into the assignment.
void lloyd_enqueue_round(cudaStream_t st, const Points& P, Workspace& w, uint64_t max_it, double tol,
                         cudaGraphConditionalHandle cond = 0, int use_cond = 0, bool fast = false,
                         const GraphRound* g = nullptr) {
    dev::LloydStatus* sts = gr_status(w, g);
    const int* parity = &sts->parity;
    const int* stop = &sts->stop;
    if (g && w.sums_on && w.sums_fuse) w.drift_slabs = 1;  // computed by the previous launch's control CTA
    else if (g && w.sums_on) launch_centroids(st, w, g->buf, sts, g->go);
    else launch_update(st, P, w, parity, stop, g ? g->go : nullptr, gr_labels(w, g), &sts->bad_label);
    dev::LloydCtl ctl = make_ctl(w, 2, P.rows, max_it, tol, cond, use_cond, fast);
    apply_graph(ctl, w, g);
    AssignSrc src{w.Cact.p, w.act.p, &w.gs.p->n_active, &w.tm_ct, gr_lbk(w, g)};
    launch_assign(st, P, w, w.k, gr_labels(w, g), w.R, parity, gr_dists(w, g), &sts->changed, stop, false,
                  fast ? nullptr : w.tile_buf.p, w.tile_ctr.p, &ctl, 2, fast ? w.R : 0,
                  g && g->fix ? (unsigned)tiles_of(w.R) : 0u, &src, g ? g->buf : 4);
}

// Runs the loop to completion; `between` is called once after the first
// batch is enqueued (used to overlap host RNG work with device work).
template <class Between>
LloydResult lloyd_run(cudaStream_t st, const Points& P, Workspace& w, uint64_t max_it, double tol,
                      Between&& between) {
    lloyd_enqueue_begin(st, P, w);
    uint64_t launched = 0;
    int batch = 2;
    bool first = true;
    while (true) {
        const uint64_t todo = std::min<uint64_t>(batch, max_it - launched);
        for (uint64_t i = 0; i < todo; ++i) lloyd_enqueue_round(st, P, w, max_it, tol);
        launched += todo;
        BM_CUDA(cudaMemcpyAsync(w.h_status.p, w.status.p, sizeof(dev::LloydStatus),
                                cudaMemcpyDeviceToHost, st));
        if (first) {
            between();
            first = false;
        }
        BM_CUDA(cudaStreamSynchronize(st));
        const dev::LloydStatus& s = *w.h_status.p;
        if (s.state_error) throw StateError("assign_nearest: every centroid is degenerate");
        if (s.stop || launched >= max_it) break;
        batch = std::min(batch * 2, 8);
    }
    const dev::LloydStatus& s = *w.h_status.p;
    if (s.bad_label) throw ConfigError("update_centroids: label out of range");
    return LloydResult{s.objective, s.evals, s.iterations, s.parity};
}

LloydResult lloyd_run(cudaStream_t st, const Points& P, Workspace& w, uint64_t max_it, double tol) {
    return lloyd_run(st, P, w, max_it, tol, [] {});
}

// ---------------------------------------------------------------------------
// kmeanspp_fill (init.cpp:123-201).  Centroids in w.C / w.mask (device) with
// the host mask mirror `mask`.  D^2 arrays live on the device; the sequential
// prefix sum, the draws and upper_bound run on the host (the reference RNG).
// ---------------------------------------------------------------------------
template <class T>
void set_row(cudaStream_t st, const Points& P, Workspace& w, uint64_t row, int j) {
    dev::k_set_row<T><<<1, 256, 0, st>>>(static_cast<const T*>(P.X), P.ld, P.n, row, w.C.p, w.mask.p, j);
    BM_LAUNCH();
    count_launch();
}

void set_row_any(cudaStream_t st, const Points& P, Workspace& w, uint64_t row, int j) {
    dispatch(P.dtype, [&](auto tag) { set_row<decltype(tag)>(st, P, w, row, j); });
}

void launch_dist_rows(cudaStream_t st, const Points& P, const uint32_t* cand, int ncand, const double* d2,
                      double* out, const int* skip = nullptr) {
    PhaseScope ps(PH_KMEANSPP, P.rows);
    const dim3 grid((unsigned)ceil_div(P.rows, 128), (unsigned)std::max(1, ncand));
    dispatch(P.dtype, [&](auto tag) {
        using T = decltype(tag);
        static const bool narrow = !(std::getenv("BM_DIST_NARROW") && std::string(std::getenv("BM_DIST_NARROW")) == "0");
        if (narrow && P.n <= dev::kDistRowsN && ncand >= 1 && ncand <= 4)  // narrow rows: every candidate in one thread
            launch_pdl(dev::k_dist_rows_narrow<T>, dim3(grid.x), 128, 0, st, static_cast<const T*>(P.X), P.rows, P.n,
                       P.ld, cand, ncand, d2, out, skip);
        else
            launch_pdl(dev::k_dist_rows<T>, grid, 128, 0, st, static_cast<const T*>(P.X), P.rows, P.n, P.ld, cand,
                       ncand, d2, out, skip);
    });
    BM_LAUNCH();
    count_launch();
}

// pick_by_mass (init.cpp:73-79): upper_bound clamped to the last index.
uint64_t pick_by_mass(const std::vector<double>& cum, double u) {
    auto it = std::upper_bound(cum.begin(), cum.end(), u);
    if (it == cum.end()) --it;
    return (uint64_t)(it - cum.begin());
}

void kmeanspp_fill_device(cudaStream_t st, const Points& P, Workspace& w, std::vector<uint8_t>& mask,
                          int candidates, Mt64& rng, uint64_t& evals) {
    if (candidates < 1) throw ConfigError("kmeanspp_fill: candidates_per_step must be at least 1");
    const uint64_t m = P.rows;
    std::vector<int> degenerate;
    int active = 0;
    for (int j = 0; j < w.k; ++j) {
        if (mask[j]) degenerate.push_back(j);
        else ++active;
    }
    if (degenerate.empty()) return;
    if ((int)w.ncand < candidates) throw ConfigError("kmeanspp_fill: workspace candidate capacity");
    // D^2 pool: trial arrays in slots [0, candidates), D^2 in slot `candidates`.
    auto buf = [&](int i) { return w.d2pool.p + (uint64_t)i * w.R; };
    const int d2i = candidates;
    size_t first_slot = 0;
    if (active == 0) {  // :144-150
        const uint64_t first = rng.uniform_int(0, m - 1);
        const int slot = degenerate.front();
        set_row_any(st, P, w, first, slot);
        mask[slot] = 0;
        first_slot = 1;
        w.h_cand.p[0] = (uint32_t)first;
        BM_CUDA(cudaMemcpyAsync(w.cand.p, w.h_cand.p, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        launch_dist_rows(st, P, w.cand.p, 1, nullptr, buf(d2i));  // distances_to_row :149
        evals += m;
    } else {  // :151-164 — min over active rows == assignment distance
        launch_compact(st, w, w.C.p, w.mask.p);
        launch_assign(st, P, w, w.k, w.labels.p, 0, nullptr, buf(d2i), nullptr, nullptr);
        evals += m * (uint64_t)active;
    }
    const uint64_t ntiles = tiles_of(m);
    // Device steps while the D^2 weights are integers (exact prefix sums); the
    // host path below continues from the first step that is not.
    static const bool dev_pp = !(std::getenv("BM_PP") && std::string(std::getenv("BM_PP")) == "host");
    if (dev_pp && candidates <= 8 && first_slot < degenerate.size()) {
        if (!w.ppmt.n) w.ppmt.alloc(1);
        if (!w.pps.n) w.pps.alloc(1);
        if (w.pprefix.n < w.R) w.pprefix.alloc(w.R);
        if (w.pptiles.n < ceil_div(w.R, dev::kPPThreads)) w.pptiles.alloc(ceil_div(w.R, dev::kPPThreads));
        *w.h_mt.p = rng.s;
        BM_CUDA(cudaMemcpyAsync(w.ppmt.p, w.h_mt.p, sizeof(Mt64State), cudaMemcpyHostToDevice, st));
        BM_CUDA(cudaMemsetAsync(w.pps.p, 0, sizeof(dev::PPState), st));
        const unsigned cgrid = (unsigned)std::min<uint64_t>(ceil_div(m, 256), 296);
        for (size_t q = first_slot; q < degenerate.size(); ++q) {
            launch_pdl(dev::k_pp_scan, (unsigned)ceil_div(m, dev::kPPThreads), dev::kPPThreads, 0, st,
                       (const double*)buf(d2i), m, w.pprefix.p, w.pptiles.p, w.pps.p);
            BM_LAUNCH();
            launch_pdl(dev::k_pp_pick, 1, dev::kPPThreads, 0, st, m, w.ppmt.p, candidates, w.cand.p,
                       (const long long*)w.pprefix.p, (const long long*)w.pptiles.p, w.pps.p);
            BM_LAUNCH();
            // (skipped after a fallback or a direct pick: the first two PPState fields)
            launch_dist_rows(st, P, w.cand.p, candidates, buf(d2i), buf(0), &w.pps.p->fallback);  // :186-189
            launch_tile_sums(st, buf(0), m, w.R, candidates, w.tile_buf.p, &w.pps.p->fallback);  // :190
            dispatch(P.dtype, [&](auto tag) {
                using T = decltype(tag);
                launch_pdl(dev::k_pp_best<T>, 1, 128, 0, st, (const double*)w.tile_buf.p, ntiles, candidates,
                           (const uint32_t*)w.cand.p, w.pps.p, static_cast<const T*>(P.X), P.ld, P.n, w.C.p,
                           w.mask.p, degenerate[q]);
            });
            BM_LAUNCH();
            launch_pdl(dev::k_pp_take, cgrid, 256, 0, st, w.d2pool.p, w.R, m, d2i, (const dev::PPState*)w.pps.p);
            BM_LAUNCH();
            count_launch(3);
        }
        dev::PPState ps{};
        BM_CUDA(cudaMemcpyAsync(&ps, w.pps.p, sizeof(ps), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(w.h_mt.p, w.ppmt.p, sizeof(Mt64State), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        rng.s = *w.h_mt.p;  // the stream after the device steps (a failed step drew nothing)
        evals += m * (uint64_t)candidates * (uint64_t)ps.cand_slots;
        // the slots done on the device: candidate slots + direct picks, in order,
        // up to the first failed one
        if (!ps.fallback) {
            for (size_t q = first_slot; q < degenerate.size(); ++q) mask[degenerate[q]] = 0;
            return;
        }
        // find how many slots completed: the device counts candidate slots only,
        // so replay the completed count from the masks written on the device
        std::vector<uint8_t> dmask(w.k);
        BM_CUDA(cudaMemcpy(dmask.data(), w.mask.p, w.k, cudaMemcpyDeviceToHost));
        size_t q0 = first_slot;
        while (q0 < degenerate.size() && dmask[degenerate[q0]] == 0) mask[degenerate[q0++]] = 0;
        first_slot = q0;
    }
    std::vector<double> cum(m);
    std::vector<uint64_t> picks(candidates);
    for (size_t q = first_slot; q < degenerate.size(); ++q) {  // :171-199
        const int slot = degenerate[q];
        BM_CUDA(cudaMemcpyAsync(w.h_d2.p, buf(d2i), m * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        double running = 0.0;  // prefix_sums :81-88 (sequential)
        for (uint64_t i = 0; i < m; ++i) {
            running += w.h_d2.p[i];
            cum[i] = running;
        }
        const double total = cum.back();
        if (total <= 0.0) {  // :174-180
            set_row_any(st, P, w, rng.uniform_int(0, m - 1), slot);
            mask[slot] = 0;
            continue;
        }
        for (int c = 0; c < candidates; ++c) {  // :183-185
            picks[c] = pick_by_mass(cum, rng.uniform_real(0.0, total));
            w.h_cand.p[c] = (uint32_t)picks[c];
        }
        BM_CUDA(cudaMemcpyAsync(w.cand.p, w.h_cand.p, candidates * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, st));
        const int base = 0;
        launch_dist_rows(st, P, w.cand.p, candidates, buf(d2i), buf(base));  // :186-189
        evals += m * (uint64_t)candidates;
        launch_tile_sums(st, buf(base), m, w.R, candidates, w.tile_buf.p, nullptr);  // :190
        BM_CUDA(cudaMemcpyAsync(w.h_tiles.p, w.tile_buf.p, candidates * ntiles * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        double best_potential = std::numeric_limits<double>::infinity();
        int best = -1;
        uint64_t best_index = 0;
        for (int c = 0; c < candidates; ++c) {
            double potential = 0.0;  // block_sum outer fold
            for (uint64_t t = 0; t < ntiles; ++t) potential += w.h_tiles.p[c * ntiles + t];
            if (potential < best_potential) {  // :191-195
                best_potential = potential;
                best_index = picks[c];
                best = c;
            }
        }
        set_row_any(st, P, w, best_index, slot);  // :197
        mask[slot] = 0;
        if (best >= 0)  // dist2 := best_trial (:198)
            BM_CUDA(cudaMemcpyAsync(buf(d2i), buf(best), m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
}

// ---------------------------------------------------------------------------
// Sampling (sample_chunk big_means.cpp:39-56): host draws, device resolution.
// ---------------------------------------------------------------------------
SamplerWs& get_sws_dev(int device, uint64_t m, uint64_t s) {
    DeviceCache& c = cache_of(device);
    auto key = std::make_pair(m, s);
    auto it = c.sws.find(key);
    if (it != c.sws.end()) return *it->second;
    auto w = std::make_unique<SamplerWs>();
    w->init(m, s);
    auto& ref = *w;
    c.sws.emplace(key, std::move(w));
    return ref;
}

SamplerWs& get_sws(const bm_dataset* d, uint64_t s) {
    DeviceCache& c = cache_of(d->device);
    auto key = std::make_pair(d->m, s);
    auto it = c.sws.find(key);
    if (it != c.sws.end()) return *it->second;
    auto w = std::make_unique<SamplerWs>();
    w->init(d->m, s);
    auto& ref = *w;
    c.sws.emplace(key, std::move(w));
    return ref;
}

// Draw the s raw Fisher-Yates targets j_i = uniform_int(i, m-1) into the
// next pinned buffer (waits until the buffer's previous upload finished).
uint32_t* draw_targets(SamplerWs& sw, Mt64& rng) {
    const int b = sw.cur;
    BM_CUDA(cudaEventSynchronize(sw.js_done[b]));
    uint32_t* out = sw.h_js[b].p;
    const uint64_t m = sw.m;
    for (uint64_t i = 0; i < sw.s; ++i) out[i] = (uint32_t)rng.uniform_int(i, m - 1);  // :50
    return out;
}

// Device-side draws (k_mt_twist, k_mt_emit, k_mt_fix) from the device-resident stream into target buffer b.
void enqueue_device_draw(cudaStream_t st, SamplerWs& sw, int force_seq = 0, int b = 0) {
    const uint32_t s = (uint32_t)sw.s;
    dev::k_mt_twist<<<1, dev::kMtThreads, 0, st>>>(sw.mt.p, sw.mt.p + 1 + b, s, sw.raw.p, sw.mtflag.p);
    BM_LAUNCH();
    dev::k_mt_emit<<<(unsigned)ceil_div(s, 256), 256, 0, st>>>(sw.raw.p, sw.m, s, sw.jsbuf(b), sw.mtflag.p);
    BM_LAUNCH();
    dev::k_mt_fix<<<1, 32, 0, st>>>(sw.mt.p, sw.mt.p + 1 + b, sw.m, s, sw.jsbuf(b), sw.mtflag.p, force_seq,
                                     sw.epoch.p, sw.epoch_slot(b));
    BM_LAUNCH();
    count_launch(3);
}

void put_stream(cudaStream_t st, SamplerWs& sw, const Mt64& rng) {
    *sw.h_mt.p = rng.s;
    BM_CUDA(cudaMemcpyAsync(sw.mt.p, sw.h_mt.p, sizeof(Mt64State), cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaStreamSynchronize(st));
}

// slot 0: the live stream; 1 + b: the input state of the last draw into buffer b
void get_stream(cudaStream_t st, SamplerWs& sw, Mt64& rng, int slot = 0) {
    BM_CUDA(cudaMemcpyAsync(sw.h_mt.p, sw.mt.p + slot, sizeof(Mt64State), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    rng.s = *sw.h_mt.p;
}

// Fisher-Yates resolution of the targets in buffer b (epoch-tagged tables, no
// clearing between chunks); result in the table set's idx (set 0: sw.idx).
void enqueue_resolve_device(cudaStream_t st, SamplerWs& sw, int b = 0, int set = 0) {
    PhaseScope ps(PH_SAMPLE, sw.s);
    const uint32_t s = (uint32_t)sw.s;
    const uint32_t* js = sw.jsbuf(b);
    const uint32_t* ep = sw.epoch_slot(b);
    const unsigned g = (unsigned)ceil_div(s, 256);
    const SamplerWs::Tabs t = sw.tabs(set);
    dev::k_fy_pass1<<<g, 256, 0, st>>>(js, ep, s, t.LT, t.hkeys, t.hvals, sw.hmask);
    dev::k_fy_pass2<<<g, 256, 0, st>>>(js, ep, s, t.LT, t.hkeys, t.hvals, sw.hmask, t.exclbits, t.bitmap);
    dev::k_bitmap_block_counts<<<sw.nblocks, dev::kScanThreads, 0, st>>>(t.bitmap, t.exclbits, s, sw.nwords, t.blockcnt);
    dev::k_bitmap_emit<<<sw.nblocks, dev::kScanThreads, 0, st>>>(t.bitmap, t.exclbits, s, sw.nwords, t.blockcnt, t.idx);
    BM_LAUNCH();
    count_launch(4);
}

// Upload the host-drawn targets of pinned buffer sw.cur into target buffer 0, then resolve.
void enqueue_resolve(cudaStream_t st, SamplerWs& sw) {
    const int b = sw.cur;
    BM_CUDA(cudaMemcpyAsync(sw.js.p, sw.h_js[b].p, sw.s * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaEventRecord(sw.js_done[b], st));
    sw.cur ^= 1;
    dev::k_epoch_bump<<<1, 32, 0, st>>>(sw.epoch.p, sw.epoch_slot(0));
    BM_LAUNCH();
    enqueue_resolve_device(st, sw, 0);
}

void enqueue_gather(cudaStream_t st, const bm_dataset* d, const uint32_t* idx, uint32_t s, void* out,
                    const void* const* xslot = nullptr) {
    PhaseScope ps(PH_GATHER, s);
    const uint64_t row_vecs = d->ld * dtype_size(d->dtype) / 16;
    constexpr unsigned cap = 592u;  // 4 CTAs per SM (148 SMs)
    const unsigned grid = (unsigned)std::min<uint64_t>(cap, ceil_div((uint64_t)s * row_vecs, 4 * 256));
    dev::k_gather<<<grid, 256, 0, st>>>(static_cast<const uint4*>(d->X),
                                        reinterpret_cast<const uint4* const*>(xslot), (uint32_t)row_vecs, idx, s,
                                        static_cast<uint4*>(out));
    BM_LAUNCH();
    count_launch();
}

// ---------------------------------------------------------------------------
// validate (big_means.cpp:16-35)
// ---------------------------------------------------------------------------
void validate(const bm_dataset* d, const bm_config& c) {
    if (c.k < 1) throw ConfigError("big_means: k must be at least 1");
    if (c.chunk_size < c.k) throw ConfigError("big_means: chunk_size must be at least k");
    if (c.chunk_size > d->m) throw ConfigError("big_means: chunk_size exceeds the dataset size");
    if (!c.has_max_cpu_seconds && !c.has_max_chunks)
        throw ConfigError("big_means: no stop condition; set max_cpu_seconds or max_chunks");
    if (c.has_max_cpu_seconds && c.max_cpu_seconds < 0.0)
        throw ConfigError("big_means: max_cpu_seconds must be nonnegative");
    if (c.has_max_chunks && c.max_chunks < 1) throw ConfigError("big_means: max_chunks must be at least 1");
    if (c.max_iterations < 1) throw ConfigError("lloyd: max_iterations must be at least 1");
    if (c.rel_tolerance < 0.0) throw ConfigError("lloyd: rel_tolerance must be nonnegative");
    if (c.candidates_per_step < 1)
        throw ConfigError("kmeanspp_fill: candidates_per_step must be at least 1");
}

// ---------------------------------------------------------------------------
// Final pass: assign all rows [r0, r1) + per-tile partials (big_means.cpp:102-107)
// ---------------------------------------------------------------------------
void final_pass(cudaStream_t st, const bm_dataset* d, Workspace& w, uint64_t r0, uint64_t r1,
                int32_t* labels_host, double* tiles_host, uint64_t* evals) {
    DeviceCache& c = cache_of(d->device);
    Points P = dataset_points(d);
    P.X = static_cast<const uint8_t*>(d->X) + r0 * d->ld * dtype_size(d->dtype);
    P.rows = r1 - r0;
    c.ensure_final(P.rows);
    static const bool final_tc = !(std::getenv("BM_FINAL_TC") && std::string(std::getenv("BM_FINAL_TC")) == "0");
    if (final_tc && P.dtype == BM_F32 && P.tf32_exact && final_tc_supported(P.n, w.k) && P.rows < (1ull << 31)) {
        // fp32 rows exact in tf32: the tensor-core final pass (finaltc.cu); then the tile partials
        PhaseScope ps(PH_FINAL, P.rows);
        dev::FinalTcArgs fa{};
        fa.xmap = final_tc_map(P.X, P.rows, P.n, P.ld);
        fa.rows = P.rows;
        fa.n = P.n;
        fa.Cact = w.Cact.p;
        fa.ldc = w.ldc;
        fa.act = w.act.p;
        fa.n_active = &w.gs.p->n_active;
        fa.cst = chunk_screen_consts(P.n, true, true);
        fa.labels = c.flabels.p;
        fa.dists = c.fdists.p;
        launch_final_tc(st, d->device, fa, pdl_enabled());
        count_launch();
        launch_tile_sums(st, c.fdists.p, P.rows, 0, 1, c.ftiles.p, nullptr);
    } else if (screen_enabled(w.k) && P.n <= dev::kFMaxD && P.rows < (1ull << 31)) {
        // streaming form (k_final): persistent CTAs, one continuous TMA ring; then the tile partials
        PhaseScope ps(PH_FINAL, P.rows);
        dispatch(P.dtype, [&](auto tag) {
            using T = decltype(tag);
            constexpr size_t shm = dev::final_smem_bytes<T>();
            set_max_smem(dev::k_final<T>, shm);
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
            const uint64_t blocks = ceil_div(P.rows, dev::kABP);
            const unsigned grid = (unsigned)std::min<uint64_t>(blocks, 2ull * (uint64_t)sms);
            const CUtensorMap tmx = points_map<T>(P);
            launch_pdl(dev::k_final<T>, grid, dev::kSThreads, shm, st, tmx, static_cast<const T*>(P.X), P.rows, P.n,
                       P.ld, (const double*)w.Cact.p, w.ldc, (const int*)w.act.p, (const int*)&w.gs.p->n_active,
                       (const float*)w.CT32.p, c.flabels.p, c.fdists.p, g_profiling ? g_prof.d_cand : nullptr,
                       screen_consts(P.n));
        });
        BM_LAUNCH();
        count_launch();
        launch_tile_sums(st, c.fdists.p, P.rows, 0, 1, c.ftiles.p, nullptr);
    } else {
        launch_assign(st, P, w, w.k, c.flabels.p, 0, nullptr, c.fdists.p, nullptr, nullptr, true, c.ftiles.p,
                      c.fctr.p);
    }
    BM_CUDA(cudaMemcpyAsync(tiles_host, c.ftiles.p, tiles_of(P.rows) * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (labels_host)
        BM_CUDA(cudaMemcpyAsync(labels_host, c.flabels.p, P.rows * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    int na = 0;
    BM_CUDA(cudaMemcpyAsync(&na, &w.gs.p->n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    if (na == 0) throw StateError("assign_nearest: every centroid is degenerate");
    if (evals) *evals += P.rows * (uint64_t)na;
}

// ---------------------------------------------------------------------------
// big_means (big_means.cpp:58-112)
// ---------------------------------------------------------------------------
// ---- CUDA graphs of one steady-state chunk --------------------------------
// BM_CHUNK_DBG=1: the chunk kernel stamps its phases (bm_debug_chunk_phases).
unsigned long long* chunk_dbg_buffer() {
    static unsigned long long* p = [] {
        unsigned long long* q = nullptr;
        if (std::getenv("BM_CHUNK_DBG")) {
            BM_CUDA(cudaMalloc(&q, 4 * 8 * 16 * sizeof(unsigned long long)));
            BM_CUDA(cudaMemset(q, 0, 4 * 8 * 16 * sizeof(unsigned long long)));
        }
        return q;
    }();
    return p;
}

// The chunk kernel's screen for fp32 rows: tensor core (tcgen05) when the rows
// are exact in tf32 (tight bound), else packed FFMA (BM_TC=1 / 0 force it).
bool tc_screen_enabled(bool tf32_exact) {
    const char* e = std::getenv("BM_TC");
    if (e && std::string(e) == "1") return true;
    if (e && std::string(e) == "0") return false;
    return tf32_exact;
}

// BM_PERSIST=0: the multi-launch chunk graphs instead of the persistent chunk
// kernel (A/B checks; the kernel also needs a plan that fits, chunk_plan).
bool persist_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_PERSIST");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// BM_CHUNK_RED=0: exact-sum chunks keep the two-barrier rounds (tile partials
// merged by their owners) instead of RED deltas with one barrier per round.
bool chunk_red_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_CHUNK_RED");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// BM_CHUNK_FIX=0: the chunk kernel folds its exact objective itself instead of
// leaving it to k_chunk_fix on the side stream.
bool chunk_fix_deferred() {
    static const bool on = !(std::getenv("BM_CHUNK_FIX") && std::string(std::getenv("BM_CHUNK_FIX")) == "0");
    return on;
}

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BM_GRAPHS");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

dev::AcceptArgs accept_args(Workspace& w) {
    dev::AcceptArgs A{};
    A.f_opt = w.fopt.p;
    A.C = w.C.p;
    A.mask = w.mask.p;
    A.Cinc = w.Cinc.p;
    A.maskinc = w.maskinc.p;
    A.k = w.k;
    A.n = w.n;
    A.rec_base = w.drec.p;
    A.chunk_ctr = w.chunk_ctr.p;
    A.Cact = w.Cact.p;
    A.ldc = w.ldc;
    A.act_idx = w.act.p;
    A.CT32 = w.CT32.p;
    A.CactI = w.CactI.p;
    A.actI = w.actI.p;
    A.CT32I = w.CT32I.p;
    A.gs = w.gs.p;
    return A;
}

// The accept (:89-94) with the exact objective of the finished Lloyd loop.
void enqueue_accept(cudaStream_t st, Workspace& w) {
    PhaseScope ps(PH_CONTROL, 0);
    launch_pdl(dev::k_accept, 1, 256, 2 * w.k * sizeof(int), st, w.status.p, accept_args(w),
               (dev::LloydStatus*)nullptr);
    BM_LAUNCH();
    count_launch();
}

// prep[b]: Fisher-Yates resolution of target buffer b, gather (:79-80), start := incumbent (:82)
cudaGraphExec_t capture_prep(cudaStream_t st, const bm_dataset* d, SamplerWs& sw, int b, void* chunk) {
    cudaGraph_t g = nullptr;
    const SamplerWs::Tabs t = sw.tabs(b);  // before the capture: set 1 is allocated on first use
    BM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    enqueue_resolve_device(st, sw, b, b);  // target buffer b in table set b: odd and even chunks' preps overlap
    BM_CUDA(cudaEventRecordWithFlags(sw.resolved[b], st, cudaEventRecordExternal));
    enqueue_gather(st, d, t.idx, (uint32_t)sw.s, chunk, sw.xslot.p);
    BM_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t e = nullptr;
    BM_CUDA(cudaGraphInstantiate(&e, g, 0));
    cudaGraphDestroy(g);
    return e;
}

// One chunk's Lloyd (local_search.cpp:16-60) + accept (:89-94) as a graph:
//   k_guard -> IF(st->go) { assign+begin, WHILE { update, assign+step }, accept } -> status D2H
// The IF lets the host queue chunk c+1 before chunk c's accept is known: when
// that accept leaves degenerate incumbent rows the graph does nothing and the
// host repairs (:83-85) and relaunches it.
void add_conditional(cudaStream_t st, cudaGraphConditionalHandle* h, cudaGraph_t* body, cudaGraphConditionalNodeType type,
                     unsigned dflt) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    BM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    BM_CUDA(cudaGraphConditionalHandleCreate(h, cg, dflt, cudaGraphCondAssignDefault));
    cudaGraphNodeParams prm = {};
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = *h;
    prm.conditional.type = type;
    prm.conditional.size = 1;
    cudaGraphNode_t cn;
    BM_CUDA(cudaGraphAddNode(&cn, cg, deps, nd, &prm));
    BM_CUDA(cudaStreamUpdateCaptureDependencies(st, &cn, 1, cudaStreamSetCaptureDependencies));
    *body = prm.conditional.phGraph_out[0];
}

cudaGraphExec_t capture_lloyd(cudaStream_t st, Workspace& w, const Points& P, uint64_t max_it, double tol, int b) {
    if (!w.cap1) BM_CUDA(cudaStreamCreateWithFlags(&w.cap1, cudaStreamNonBlocking));
    if (!w.cap2) BM_CUDA(cudaStreamCreateWithFlags(&w.cap2, cudaStreamNonBlocking));
    BM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    // fast-sum control whenever the TMA screen (which implements it) runs
    const bool fast = screen_enabled(w.k) && P.rows < (1ull << 31) && !w.hist_cap;
    if (fast) {
        // begin unless the speculative begin (capture_spec) is current ->
        // round 1 (+ fixup CTAs: the previous chunk's exact objective for its
        // record) -> round 2; the control of the round that stops runs the
        // accept.  A chunk still running after round 2 is marked incomplete and
        // continued by the host (capture_cont).  Every kernel of a skipped
        // chunk (go == 0) returns at once.
        GraphRound g;
        g.buf = b;
        g.go = &w.gs.p->go;
        g.begin_kind = 2;
        lloyd_enqueue_begin(st, P, w, /*do_compact=*/false, true, &g);  // accept (or the repair) compacted the start
        GraphRound r = g;
        r.begin_kind = 0;
        r.fix = true;
        r.accept = true;
        r.host_st = w.h_status.p + b;
        lloyd_enqueue_round(st, P, w, max_it, tol, 0, 0, true, &r);
        r.fix = false;
        r.incomplete_after = 2;
        lloyd_enqueue_round(st, P, w, max_it, tol, 0, 0, true, &r);
    } else {  // the guard sets the IF condition inside the graph that owns it
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        BM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, nullptr, nullptr));
        cudaGraphConditionalHandle hif;
        BM_CUDA(cudaGraphConditionalHandleCreate(&hif, cg, 0, cudaGraphCondAssignDefault));
        dev::k_guard<<<1, 1, 0, st>>>(w.gs.p, hif);
        BM_LAUNCH();
        cudaGraphNodeParams prm = {};
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        BM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
        prm.type = cudaGraphNodeTypeConditional;
        prm.conditional.handle = hif;
        prm.conditional.type = cudaGraphCondTypeIf;
        prm.conditional.size = 1;
        cudaGraphNode_t cn;
        BM_CUDA(cudaGraphAddNode(&cn, cg, deps, nd, &prm));
        BM_CUDA(cudaStreamUpdateCaptureDependencies(st, &cn, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t ifbody = prm.conditional.phGraph_out[0];
        BM_CUDA(cudaStreamBeginCaptureToGraph(w.cap1, ifbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        lloyd_enqueue_begin(w.cap1, P, w, /*do_compact=*/false, false);  // accept (or the repair) compacted the start
        cudaGraphConditionalHandle hw;
        cudaGraph_t wbody = nullptr;
        add_conditional(w.cap1, &hw, &wbody, cudaGraphCondTypeWhile, 1);
        BM_CUDA(cudaStreamBeginCaptureToGraph(w.cap2, wbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        lloyd_enqueue_round(w.cap2, P, w, max_it, tol, hw, 1, false);
        BM_CUDA(cudaStreamEndCapture(w.cap2, &wbody));
        enqueue_accept(w.cap1, w);
        BM_CUDA(cudaStreamEndCapture(w.cap1, &ifbody));
        BM_CUDA(cudaMemcpyAsync(w.h_status.p + b, w.status.p, sizeof(dev::LloydStatus), cudaMemcpyDeviceToHost, st));
    }
    cudaGraph_t g = nullptr;
    BM_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t e = nullptr;
    BM_CUDA(cudaGraphInstantiate(&e, g, 0));
    cudaGraphDestroy(g);
    return e;
}

// The rest of an incomplete chunk's Lloyd loop: WHILE { update, assign + step },
// the stopping control running the accept.
cudaGraphExec_t capture_cont(cudaStream_t st, Workspace& w, const Points& P, uint64_t max_it, double tol, int b) {
    if (!w.cap2) BM_CUDA(cudaStreamCreateWithFlags(&w.cap2, cudaStreamNonBlocking));
    BM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cudaGraphConditionalHandle hw;
    cudaGraph_t wbody = nullptr;
    add_conditional(st, &hw, &wbody, cudaGraphCondTypeWhile, 1);
    BM_CUDA(cudaStreamBeginCaptureToGraph(w.cap2, wbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    GraphRound r;
    r.buf = b;
    r.accept = true;
    r.host_st = w.h_status.p + b;
    lloyd_enqueue_round(w.cap2, P, w, max_it, tol, hw, 1, true, &r);
    BM_CUDA(cudaStreamEndCapture(w.cap2, &wbody));
    cudaGraph_t g = nullptr;
    BM_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t e = nullptr;
    BM_CUDA(cudaGraphInstantiate(&e, g, 0));
    cudaGraphDestroy(g);
    return e;
}

// The speculative begin of the chunk in buffer b: its first assignment against
// the incumbent's compacted copy, run while the previous chunk's rounds run.
// Valid only if no accept published a new incumbent meanwhile (inc_version).
cudaGraphExec_t capture_spec(cudaStream_t st, Workspace& w, const Points& P, int b) {
    BM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    BM_CUDA(cudaMemsetAsync(&w.status.p[b].bv_min, 0xFF, sizeof(long long), st));
    // exact-sum mode: both halves of this buffer's sums start at zero (the redo
    // begin of this chunk, if any, runs after this graph)
    if (w.sums_on) BM_CUDA(cudaMemsetAsync(w.sums_of(b), 0, 2 * w.sum_half() * sizeof(long long), st));
    GraphRound g;
    g.buf = b;
    g.begin_kind = 1;
    lloyd_enqueue_begin(st, P, w, /*do_compact=*/false, true, &g);
    cudaGraph_t gr = nullptr;
    BM_CUDA(cudaStreamEndCapture(st, &gr));
    cudaGraphExec_t e = nullptr;
    BM_CUDA(cudaGraphInstantiate(&e, gr, 0));
    cudaGraphDestroy(gr);
    return e;
}

void ensure_graphs(cudaStream_t st, const bm_dataset* d, DeviceCache& dc, SamplerWs& sw, Workspace& w,
                   const Points& P, uint64_t max_it, double tol, bool persist = false) {
    char sig[512];
    // the dataset enters only through shape: its base is read from sw.xslot
    std::snprintf(sig, sizeof(sig), "%llu/%llu/%d/%p/%p/%p/%p/%p/%p/%llu/%a/%llu/%d/%a/%p/%p",
                  (unsigned long long)d->m, (unsigned long long)d->ld, (int)d->dtype, (void*)dc.chunk.p, (void*)dc.chunk1.p,
                  (void*)dc.chunk3.p, (void*)&sw,
                  (void*)w.drec.p, (void*)sw.mt.p, (unsigned long long)max_it, tol, (unsigned long long)w.drec.n,
                  (int)w.sums_on + 2 * (int)w.sum_small + 4 * (int)w.sums_fuse +
                      16 * (int)persist + 32 * (int)use_wide(P, w.k),
                  w.sum_scale, (void*)w.sums.p, (void*)w.wide[0].dot.p);
    if (w.graph_sig == sig && w.g_prep[0]) return;
    w.drop_graphs();
    const uint64_t saved = g_profile.kernel_launches;
    void* bufs[dev::kStateBufs] = {dc.chunk.p, dc.chunk1.p, dc.chunk2.p, dc.chunk3.p};
    const bool fast = screen_enabled(w.k) && P.rows < (1ull << 31) && !w.hist_cap;
    for (int i = 0; i < dev::kStateBufs; ++i) {  // data and state buffer i, draw buffer i % 2
        const int b = i;
        Points Pb = P;
        Pb.X = bufs[i];
        w.g_prep[i] = capture_prep(st, d, sw, i % 2, bufs[i]);
        if (persist) continue;  // the chunk is one persistent kernel launch (launch_chunk)
        w.g_lloyd[i] = capture_lloyd(st, w, Pb, max_it, tol, b);
        if (fast) {
            w.g_cont[i] = capture_cont(st, w, Pb, max_it, tol, b);
            w.g_spec[i] = capture_spec(st, w, Pb, b);
        }
    }
    g_profile.kernel_launches = saved;  // capture is not execution
    w.graph_sig = sig;
}

void big_means(const bm_dataset* d, const bm_config& cfg, bm_outcome* out, bm_chunk_record* trace,
               uint64_t trace_cap) {
    validate(d, cfg);
    DeviceGuard g(d->device);
    DeviceCache& dc = cache_of(d->device);
    cudaStream_t st = dc.stream;
    const uint64_t m = d->m, s = cfg.chunk_size;
    const int k = (int)cfg.k, n = (int)d->n;
    g_profile = bm_profile{};  // launch counts always; event timing only when profiling
    if (g_profiling) g_prof.begin(st);
    g_prof.stream = st;
    Mt64 rng(cfg.seed);  // :62 — moves to the device for the chunk draws
    Workspace& w = get_ws(d, s, k, cfg.candidates_per_step, 0);
    const bool identity = s == m;  // sample_chunk(s == m): whole range, no draws (:46-48)
    SamplerWs* sw = identity ? nullptr : &get_sws(d, s);
    Points chunkP{nullptr, d->dtype, s, n, d->ld, d->tf32_exact};
    if (identity) {
        chunkP = dataset_points(d);
    } else {
        const size_t bytes = s * d->ld * dtype_size(d->dtype);
        if (dc.chunk.n < bytes) dc.chunk.alloc(bytes);
        chunkP.X = dc.chunk.p;
        if (!g_profiling && graphs_enabled() && dc.chunk1.n < bytes) dc.chunk1.alloc(bytes);
        if (!g_profiling && graphs_enabled() && dc.chunk2.n < bytes) dc.chunk2.alloc(bytes);
        if (!g_profiling && graphs_enabled() && dc.chunk3.n < bytes) dc.chunk3.alloc(bytes);
    }
    // one device record per chunk; a time budget starts small and grows (below)
    const uint64_t want_rec = cfg.has_max_chunks && !cfg.has_max_cpu_seconds
                                  ? cfg.max_chunks
                                  : std::min<uint64_t>(cfg.has_max_chunks ? cfg.max_chunks : 1024, 1024);
    if (w.drec.n < want_rec) w.drec.alloc(want_rec);
    // incumbent all degenerate, f_opt = +inf (:63-64), chunk counter 0
    dev::k_run_init<<<1, 256, 0, st>>>(w.status.p, dev::kStateBufs, w.gs.p, w.fopt.p, w.Cinc.p, w.maskinc.p, w.C.p, w.mask.p, k, n,
                                       w.chunk_ctr.p);
    BM_LAUNCH();
    if (!identity) {
        put_stream(st, *sw, rng);
        BM_CUDA(cudaMemcpyAsync(sw->xslot.p, &d->X, sizeof(void*), cudaMemcpyHostToDevice, st));
    }
    const bool use_graphs = !identity && !g_profiling && graphs_enabled();
    // persistent chunk kernel (chunk.cu): one cooperative launch per chunk
    ChunkPlan cplan;
    if (use_graphs && persist_enabled() && !w.hist_cap)
        cplan = chunk_plan(d->device, s, n, k, d->dtype, d->exact_sums && exact_sums_enabled(),
                           d->dtype == BM_F32 && tc_screen_enabled(d->tf32_exact), chunk_red_enabled());
    const bool persist = cplan.ok;
    if (persist) {
        prefer_max_smem_carveout();
        w.ensure_chunk(cplan);
        if (w.ctiming.n < 2 * w.drec.n) w.ctiming.alloc(2 * w.drec.n);
        // (every fix of the previous run finished: its fix stream was synchronized)
        BM_CUDA(cudaMemsetAsync(w.cfix_seq.p, 0, sizeof(unsigned long long), st));
        BM_CUDA(cudaMemsetAsync(w.cjob.p, 0, dev::kStateBufs * sizeof(dev::FixJob), st));
        BM_CUDA(cudaMemsetAsync(w.cdsum.p, 0, w.cdsum.n * sizeof(double), st));
        BM_CUDA(cudaMemsetAsync(w.cdcnt.p, 0, w.cdcnt.n * sizeof(int), st));
    }
    // exact-sum mode for the graph chunks (kernels.cuh §5b)
    // (wide rows keep the ordered update: integer label sums over thousands of
    // dims cost more than k_update — c5: 128 vs 85 ms per step)
    w.sums_on = use_graphs && !persist && d->exact_sums && exact_sums_enabled() && screen_enabled(k) &&
                s < (1ull << 31) && !w.hist_cap && n <= 256;
    if (w.sums_on) {
        w.sum_scale = std::ldexp(1.0, -d->sum_exp);
        w.sum_unscale = std::ldexp(1.0, d->sum_exp);
        w.sum_small = d->sum_units_max < 0x1p23;  // 128 points per CTA: partial sums below 2^30
        static const bool fuse = !(std::getenv("BM_SUMS_FUSE") && std::string(std::getenv("BM_SUMS_FUSE")) == "0");
        w.sums_fuse = fuse;
        const uint64_t nb = dev::kStateBufs;
        if (w.sums.n < 2 * nb * w.sum_half()) w.sums.alloc(2 * nb * w.sum_half());
        if (w.sum_parts.n < nb * w.part_ctas() * w.part_len()) w.sum_parts.alloc(nb * w.part_ctas() * w.part_len());
        if (w.grp_ctr.n < nb * ceil_div(w.part_ctas(), (uint64_t)dev::kSumGroup)) {
            w.grp_ctr.alloc(nb * ceil_div(w.part_ctas(), (uint64_t)dev::kSumGroup));
            BM_CUDA(cudaMemsetAsync(w.grp_ctr.p, 0, w.grp_ctr.n * sizeof(unsigned), st));
        }
    }
    if (!persist) ensure_wide(w, chunkP, k);  // before any capture
    if (use_graphs) ensure_graphs(st, d, dc, *sw, w, chunkP, cfg.max_iterations, cfg.rel_tolerance, persist);
    uint64_t evals = 0, iterations = 0;
    uint64_t chunk_assign_passes = 0, chunk_update_passes = 0;
    int inc_degenerate = k;
    std::vector<uint8_t> hmask(k);

    const auto t_loop = std::chrono::steady_clock::now();
    if (use_graphs) {
        // Graph mode.  Chunk c uses graph slot c % 4: data and state buffer
        // c % 4, draw buffer c % 2.  While chunk c's Lloyd graph runs, chunk
        // c+3's draws, prep (resolution + gather) and speculative begin (its
        // first assignment against the incumbent's copy) run on rng_stream /
        // pstream / sstream (those of chunks c+1, c+2 were enqueued during
        // chunks c-2, c-1); chunk c+1's Lloyd graph is queued
        // behind chunk c's before the host waits.  It runs only if chunk c's
        // accept leaves no degenerate incumbent rows (go) and redoes its begin
        // if an accept published a new incumbent meanwhile (inc_version).  The
        // RNG order (big_means.hpp:21-23) is kept: draws made ahead of a repair
        // are discarded and redone after it.
        if (!dc.pstream) BM_CUDA(cudaStreamCreateWithFlags(&dc.pstream, cudaStreamNonBlocking));
        if (!dc.pstream2) BM_CUDA(cudaStreamCreateWithFlags(&dc.pstream2, cudaStreamNonBlocking));
        for (int i = 0; i < dev::kStateBufs; ++i) {
            if (!w.ev_lloyd[i]) BM_CUDA(cudaEventCreateWithFlags(&w.ev_lloyd[i], cudaEventDisableTiming));
            if (!w.ev_prep[i]) BM_CUDA(cudaEventCreateWithFlags(&w.ev_prep[i], cudaEventDisableTiming));
            if (!w.ev_spec[i]) BM_CUDA(cudaEventCreateWithFlags(&w.ev_spec[i], cudaEventDisableTiming));
            BM_CUDA(cudaEventRecord(w.ev_lloyd[i], st));
            BM_CUDA(cudaEventRecord(w.ev_spec[i], st));
        }
        // BM_PREP_STREAMS=1: every prep on one stream (A/B)
        static const bool one_prep = std::getenv("BM_PREP_STREAMS") && std::string(std::getenv("BM_PREP_STREAMS")) == "1";
        const cudaStream_t pst = dc.pstream, pst2 = one_prep ? dc.pstream : dc.pstream2;
        Points bufP[dev::kStateBufs] = {chunkP, chunkP, chunkP, chunkP};
        bufP[1].X = dc.chunk1.p;
        bufP[2].X = dc.chunk2.p;
        bufP[3].X = dc.chunk3.p;
        // BM_TIMELINE=1: in-stream events around every graph (GPU durations incl. gaps)
        static const bool timeline = std::getenv("BM_TIMELINE") != nullptr;
        // per graph launch: (kind 0 = prep / 1 = Lloyd / 2 = speculative begin, start event, end event)
        struct TlRec { int kind; cudaEvent_t a, b; };
        std::vector<TlRec> tl;
        auto tl_ev = [&](cudaStream_t q) {
            cudaEvent_t e = nullptr;
            if (timeline) {
                BM_CUDA(cudaEventCreate(&e));
                BM_CUDA(cudaEventRecord(e, q));
            }
            return e;
        };
        // chunk c's prep (its draws are enqueued on rng_stream: drawn[c % 2])
        auto launch_prep = [&](uint64_t c) {
            const int i = (int)(c % dev::kStateBufs);
            const cudaStream_t ps = (c & 1) ? pst2 : pst;  // same parity: same target buffer and table set, in order
            BM_CUDA(cudaStreamWaitEvent(ps, sw->drawn[c & 1], 0));
            BM_CUDA(cudaStreamWaitEvent(ps, w.ev_lloyd[i], 0));  // the data buffer's previous chunk (c-4)
            cudaEvent_t e0 = tl_ev(ps);
            BM_CUDA(cudaGraphLaunch(w.g_prep[i], ps));
            if (timeline) tl.push_back({0, e0, tl_ev(ps)});
            BM_CUDA(cudaEventRecord(w.ev_prep[i], ps));
            count_launch(6);
        };
        // BM_SPEC=0: no speculative begins (every chunk graph runs its own)
        static const bool spec_on = !(std::getenv("BM_SPEC") && std::string(std::getenv("BM_SPEC")) == "0");
        const bool spec = spec_on && !persist && w.g_spec[0] != nullptr;
        if (spec && !dc.sstream) BM_CUDA(cudaStreamCreateWithFlags(&dc.sstream, cudaStreamNonBlocking));
        auto launch_spec = [&](uint64_t c) {  // chunk c's first assignment, overlapping chunks c-2 and c-1
            const int i = (int)(c % dev::kStateBufs);
            BM_CUDA(cudaStreamWaitEvent(dc.sstream, w.ev_prep[i], 0));
            BM_CUDA(cudaStreamWaitEvent(dc.sstream, w.ev_lloyd[i], 0));  // the state buffer's previous chunk (c-4)
            cudaEvent_t e0 = tl_ev(dc.sstream);
            BM_CUDA(cudaGraphLaunch(w.g_spec[i], dc.sstream));
            if (timeline) tl.push_back({2, e0, tl_ev(dc.sstream)});
            BM_CUDA(cudaEventRecord(w.ev_spec[i], dc.sstream));
            count_launch(1);
        };
        auto launch_lloyd = [&](uint64_t c) {
            const int i = (int)(c % dev::kStateBufs);
            if (w.sums_on && (c == 0 || !spec))  // no speculative begin zeroed this buffer's sums
                BM_CUDA(cudaMemsetAsync(w.sums_of((int)(c % dev::kStateBufs)), 0, 2 * w.sum_half() * sizeof(long long),
                                        st));
            // (the prep runs chunks ahead: when it has already finished, no wait is enqueued
            // between the chunk kernels)
            if (cudaEventQuery(w.ev_prep[i]) != cudaSuccess) {
                (void)cudaGetLastError();
                BM_CUDA(cudaStreamWaitEvent(st, w.ev_prep[i], 0));
            }
            if (spec) BM_CUDA(cudaStreamWaitEvent(st, w.ev_spec[i], 0));
            cudaEvent_t e0 = tl_ev(st);
            if (persist) {
                dev::ChunkArgs a{};
                {  // the rows' tensor map of this chunk buffer (re-encoded when the buffer or plan changes)
                    auto& cm = w.cmaps[i];
                    if (cm.X != bufP[i].X || cm.rows != s || cm.B != cplan.B || cm.tc != cplan.tc || cm.xld != cplan.xld ||
                        cm.n != n || cm.ld != d->ld || cm.dtype != d->dtype) {
                        cm.map = chunk_rows_map(cplan, d->dtype, bufP[i].X, s, n, d->ld);
                        cm.X = bufP[i].X;
                        cm.rows = s;
                        cm.B = cplan.B;
                        cm.tc = cplan.tc;
                        cm.xld = cplan.xld;
                        cm.n = n;
                        cm.ld = d->ld;
                        cm.dtype = d->dtype;
                    }
                    a.xmap = cm.map;
                }
                a.rows_tf32_exact = d->tf32_exact ? 1 : 0;
                a.X = bufP[i].X;
                a.rows = s;
                a.n = n;
                a.ld = d->ld;
                a.k = k;
                a.C = w.C.p;
                a.mask = w.mask.p;
                a.part = w.cpart.p;
                a.pcnt = w.cpcnt.p;
                a.dists = w.dists.p + 3 * (uint64_t)i * w.R;
                a.tiles = w.ctiles.p;
                a.bar = w.cbar.p;
                a.rsum = w.crsum.p;
                a.rchg = w.crchg.p;
                a.dsum = w.cdsum.p;
                a.dcnt = w.cdcnt.p;
                a.cst = chunk_screen_consts(n, cplan.tc, true);
                a.cst_loose = chunk_screen_consts(n, cplan.tc, false);
                a.max_iterations = cfg.max_iterations;
                a.rel_tolerance = cfg.rel_tolerance;
                a.force_exact = force_exact_control() ? 1 : 0;
                a.f_opt = w.fopt.p;
                a.Cinc = w.Cinc.p;
                a.maskinc = w.maskinc.p;
                a.rec_base = w.drec.p;
                a.chunk_ctr = w.chunk_ctr.p;
                a.gs = w.gs.p;
                a.st = w.status.p + i;
                a.host_st = w.h_status.p + i;
                a.timing = w.ctiming.p;
                a.timing_cap = w.ctiming.n / 2;
                a.dbg = chunk_dbg_buffer();
                a.dbg_mma = a.dbg && std::string(std::getenv("BM_CHUNK_DBG")) == "2";
                const bool defer = chunk_fix_deferred();
                a.job = defer ? w.cjob.p + i : nullptr;
                a.fix_seq = defer ? w.cfix_seq.p : nullptr;
                launch_chunk(st, cplan, d->dtype, a);
                // its exact objective, folded on the side stream during the next chunk
                if (defer) {
                // (one event per chunk kernel: the fix stream and the buffer's next prep both wait on ev_lloyd)
                BM_CUDA(cudaEventRecord(w.ev_lloyd[i], st));
                BM_CUDA(cudaStreamWaitEvent(w.fix_stream, w.ev_lloyd[i], 0));
                dev::FixArgs fa{};
                fa.job = w.cjob.p + i;
                fa.dists = a.dists;
                fa.rows = s;
                fa.tiles = w.cfix_tiles.p;
                fa.counter = w.cfix_ctr.p;
                fa.rec_base = w.drec.p;
                fa.f_opt = w.fopt.p;
                fa.gs = w.gs.p;
                fa.fix_seq = w.cfix_seq.p;
                launch_chunk_fix(w.fix_stream, fa);
                }
                count_launch(defer ? 2 : 1);
            } else {
                BM_CUDA(cudaGraphLaunch(w.g_lloyd[i], st));
            }
            if (timeline) tl.push_back({1, e0, tl_ev(st)});
            if (!(persist && chunk_fix_deferred())) BM_CUDA(cudaEventRecord(w.ev_lloyd[i], st));
        };
        auto draw = [&](uint64_t c) {  // chunk c's sample draws into target buffer c % 2
            if (c >= 2) BM_CUDA(cudaStreamWaitEvent(sw->rng_stream, sw->resolved[c & 1], 0));  // read by chunk c-2
            enqueue_device_draw(sw->rng_stream, *sw, 0, (int)(c & 1));
            BM_CUDA(cudaEventRecord(sw->drawn[c & 1], sw->rng_stream));
        };
        // speculation needs the chunk count to be known in advance (no time budget)
        const bool speculate = !cfg.has_max_cpu_seconds;
        auto exists = [&](uint64_t c) { return !cfg.has_max_chunks || c < cfg.max_chunks; };
        draw(0);
        launch_prep(0);
        // Lloyd graphs queued from `chunk` on (each guarded by go: a chunk after
        // one that needs a repair or more rounds does nothing and is relaunched)
        uint64_t queued = 0;
        constexpr uint64_t lloyd_depth = 2;  // graphs queued beyond the current one
        uint64_t ahead = 0;  // chunks after this one whose draws, prep and speculative begin are enqueued
        for (uint64_t chunk = 0;; ++chunk) {
            if (cfg.has_max_chunks && chunk >= cfg.max_chunks) break;  // :71-73
            if (chunk > 0 && cfg.has_max_cpu_seconds && seconds_since(t_loop) >= cfg.max_cpu_seconds)
                break;  // :74-77
            if (chunk >= w.drec.n) {  // time-budget runs: grow the record buffer (graphs re-captured)
                BM_CUDA(cudaStreamSynchronize(st));
                BM_CUDA(cudaStreamSynchronize(pst));
                BM_CUDA(cudaStreamSynchronize(pst2));
                if (dc.sstream) BM_CUDA(cudaStreamSynchronize(dc.sstream));
                DevBuf<dev::Record> bigger(w.drec.n * 2);
                BM_CUDA(cudaMemcpyAsync(bigger.p, w.drec.p, w.drec.n * sizeof(dev::Record),
                                        cudaMemcpyDeviceToDevice, st));
                BM_CUDA(cudaStreamSynchronize(st));
                std::swap(w.drec.p, bigger.p);
                std::swap(w.drec.n, bigger.n);
                if (persist && w.ctiming.n < 2 * w.drec.n) {
                    DevBuf<unsigned long long> t2(2 * w.drec.n);
                    BM_CUDA(cudaMemcpyAsync(t2.p, w.ctiming.p, w.ctiming.n * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToDevice, st));
                    BM_CUDA(cudaStreamSynchronize(st));
                    std::swap(w.ctiming.p, t2.p);
                    std::swap(w.ctiming.n, t2.n);
                }
                ensure_graphs(st, d, dc, *sw, w, chunkP, cfg.max_iterations, cfg.rel_tolerance, persist);
            }
            const int b = (int)(chunk % dev::kStateBufs), i6 = b;
            if (inc_degenerate > 0) {  // kmeanspp_fill (:84) after this chunk's sample draws
                // (a queued Lloyd graph of this chunk found go == 0 and did nothing)
                BM_CUDA(cudaStreamWaitEvent(st, w.ev_prep[i6], 0));
                BM_CUDA(cudaMemcpyAsync(w.h_mask.p, w.maskinc.p, k, cudaMemcpyDeviceToHost, st));
                BM_CUDA(cudaStreamSynchronize(st));
                std::copy(w.h_mask.p, w.h_mask.p + k, hmask.begin());
                BM_CUDA(cudaStreamSynchronize(sw->rng_stream));
                // the stream right after this chunk's draws: live, or the input
                // state of chunk+1's speculative draws (which are discarded)
                get_stream(st, *sw, rng, ahead > 0 ? 1 + (int)((chunk + 1) & 1) : 0);
                kmeanspp_fill_device(st, bufP[b], w, hmask, cfg.candidates_per_step, rng, evals);
                put_stream(st, *sw, rng);
                launch_compact(st, w, w.C.p, w.mask.p);  // the Lloyd graph starts from Cact
                BM_CUDA(cudaMemsetAsync(&w.gs.p->go, 0x01, sizeof(int), st));
                dev::k_bump_version<<<1, 1, 0, st>>>(w.gs.p);  // the start is no longer the incumbent's copy
                BM_LAUNCH();
                queued = 0;
                ahead = 0;  // the draws, preps and begins made ahead are redone
            }
            if (queued == 0) {
                launch_lloyd(chunk);
                queued = 1;
            }
            // chunks chunk+1 .. chunk+3: draws (the stream is past this chunk's
            // repair, if any), prep and speculative begin, each as soon as its
            // buffers' previous chunk (c-4) is done.  Beyond chunk+1 they assume
            // no repair in between (else they are redone above) and need the
            // chunk count in advance (no time budget).
            const uint64_t depth = speculate ? 3 : 1;
            while (ahead < depth && exists(chunk + 1 + ahead)) {
                const uint64_t c2 = chunk + 1 + ahead;
                draw(c2);
                launch_prep(c2);
                if (spec) launch_spec(c2);
                ++ahead;
            }
            // the next chunks' Lloyd graphs behind this one (each runs iff the chunk
            // before it needed neither a repair nor more rounds)
            while (speculate && queued < 1 + lloyd_depth && exists(chunk + queued)) {
                launch_lloyd(chunk + queued);
                ++queued;
            }
            {
                // BM_HOSTPROF=1: how long the host waits for the device per chunk (0: the loop is host-bound)
                static const bool hostprof = std::getenv("BM_HOSTPROF") != nullptr;
                const auto tw = std::chrono::steady_clock::now();
                BM_CUDA(cudaEventSynchronize(w.ev_lloyd[i6]));
                if (hostprof) {
                    static double waited = 0.0;
                    static uint64_t nwait = 0;
                    waited += seconds_since(tw);
                    if (++nwait % 200 == 0) {
                        std::fprintf(stderr, "[hostprof] %.1f us waiting on the device per chunk (last 200)\n", waited / 200 * 1e6);
                        waited = 0.0;
                    }
                }
            }
            if (w.h_status.p[b].incomplete) {  // more rounds than the graph unrolls
                BM_CUDA(cudaGraphLaunch(w.g_cont[i6], st));
                BM_CUDA(cudaEventRecord(w.ev_lloyd[i6], st));
                BM_CUDA(cudaEventSynchronize(w.ev_lloyd[i6]));
                queued = 1;  // the queued next chunks found go == 0 and did nothing
            }
            const dev::LloydStatus& ls = w.h_status.p[b];
            if (ls.state_error) throw StateError("assign_nearest: every centroid is degenerate");
            if (ls.bad_label) throw ConfigError("update_centroids: label out of range");
            evals += ls.evals;  // lloyd accumulate (local_search.cpp:55-58)
            iterations += ls.iterations;
            chunk_assign_passes += ls.iterations + 1;
            chunk_update_passes += ls.iterations;
            inc_degenerate = ls.inc_degenerate;
            if (!persist) count_launch(3 + 3 * ls.iterations);
            out->chunks = chunk + 1;
            if (ahead) --ahead;
            if (queued) --queued;
        }
        // the last chunk's record gets its exact objective
        if (persist) {
            BM_CUDA(cudaStreamSynchronize(w.fix_stream));
        } else {
            dev::k_fix_final<<<(unsigned)tiles_of(w.R), 256, 0, st>>>(w.gs.p, accept_args(w), w.dists.p, w.R,
                                                                       w.fix_tiles.p, w.tiles_done.p);
            BM_LAUNCH();
        }
        BM_CUDA(cudaStreamSynchronize(st));
        BM_CUDA(cudaStreamSynchronize(pst));
        BM_CUDA(cudaStreamSynchronize(pst2));
        if (dc.sstream) BM_CUDA(cudaStreamSynchronize(dc.sstream));
        if (timeline && tl.size() > 2) {
            double dur[3] = {0, 0, 0}, gap = 0;
            int cnt[3] = {0, 0, 0}, ngap = 0;
            cudaEvent_t prev_end = nullptr, first = nullptr, last = nullptr;
            for (auto& r : tl) {
                float ms = 0;
                BM_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
                dur[r.kind] += ms;
                cnt[r.kind] += 1;
                if (r.kind == 1) {
                    if (prev_end) {
                        BM_CUDA(cudaEventElapsedTime(&ms, prev_end, r.a));
                        gap += ms;
                        ++ngap;
                    }
                    prev_end = r.b;
                    if (!first) first = r.a;
                    last = r.b;
                }
            }
            float total = 0;
            BM_CUDA(cudaEventElapsedTime(&total, first, last));
            std::fprintf(stderr,
                         "[timeline] %.3f ms over %d Lloyd graphs: %.1f us per chunk | Lloyd graph %.1f us | gap "
                         "before the next %.1f us | prep graph %.1f us (%d) | speculative begin %.1f us (%d)\n",
                         total, cnt[1], 1e3 * total / cnt[1], 1e3 * dur[1] / cnt[1], ngap ? 1e3 * gap / ngap : 0.0,
                         cnt[0] ? 1e3 * dur[0] / cnt[0] : 0.0, cnt[0], cnt[2] ? 1e3 * dur[2] / cnt[2] : 0.0, cnt[2]);
            if (std::string(std::getenv("BM_TIMELINE")) == "2")  // raw: kind, start, end (us from the first Lloyd graph)
                for (auto& r : tl) {
                    float a = 0, b2 = 0;
                    BM_CUDA(cudaEventElapsedTime(&a, first, r.a));
                    BM_CUDA(cudaEventElapsedTime(&b2, first, r.b));
                    std::fprintf(stderr, "[tl] %d %.2f %.2f\n", r.kind, 1e3 * a, 1e3 * b2);
                }
            for (auto& r : tl) {
                cudaEventDestroy(r.a);
                cudaEventDestroy(r.b);
            }
        }
    } else {  // host-driven chunk loop (profiling, BM_GRAPHS=0, s == m)
    bool drawn_ahead = false;  // next chunk's targets already being drawn on rng_stream
    for (uint64_t chunk = 0;; ++chunk) {
        if (cfg.has_max_chunks && chunk >= cfg.max_chunks) break;  // :71-73
        if (chunk > 0 && cfg.has_max_cpu_seconds && seconds_since(t_loop) >= cfg.max_cpu_seconds)
            break;  // :74-77
        if (chunk >= w.drec.n) {  // time-budget runs: grow the record buffer (graphs re-captured)
            DevBuf<dev::Record> bigger(w.drec.n * 2);
            BM_CUDA(cudaMemcpyAsync(bigger.p, w.drec.p, w.drec.n * sizeof(dev::Record), cudaMemcpyDeviceToDevice, st));
            BM_CUDA(cudaStreamSynchronize(st));
            std::swap(w.drec.p, bigger.p);
            std::swap(w.drec.n, bigger.n);
            if (use_graphs) ensure_graphs(st, d, dc, *sw, w, chunkP, cfg.max_iterations, cfg.rel_tolerance);
        }
        const int jb = (int)(chunk & 1);
        if (!identity) {  // sample_chunk (:79): draws made on rng_stream, resolution + gather (:80) here
            if (!drawn_ahead) {
                enqueue_device_draw(sw->rng_stream, *sw, 0, jb);
                BM_CUDA(cudaEventRecord(sw->drawn[jb], sw->rng_stream));
            }
            count_launch();
            BM_CUDA(cudaStreamWaitEvent(st, sw->drawn[jb], 0));
        }
        drawn_ahead = false;
        if (use_graphs) {
            BM_CUDA(cudaGraphLaunch(w.g_prep[jb], st));
            count_launch(7);
        } else {
            if (!identity) {
                enqueue_resolve_device(st, *sw, jb);
                BM_CUDA(cudaEventRecord(sw->resolved[jb], st));
                enqueue_gather(st, d, sw->idx.p, (uint32_t)s, dc.chunk.p);
            }
            // start = incumbent (:82)
            BM_CUDA(cudaMemcpyAsync(w.C.p, w.Cinc.p, (size_t)k * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
            BM_CUDA(cudaMemcpyAsync(w.mask.p, w.maskinc.p, k, cudaMemcpyDeviceToDevice, st));
        }
        if (inc_degenerate > 0) {  // kmeanspp_fill (:84) consumes draws before the next sample
            BM_CUDA(cudaMemcpyAsync(w.h_mask.p, w.maskinc.p, k, cudaMemcpyDeviceToHost, st));
            BM_CUDA(cudaStreamSynchronize(st));
            std::copy(w.h_mask.p, w.h_mask.p + k, hmask.begin());
            // the repair draws follow this chunk's sample draws in the stream
            if (!identity) {
                BM_CUDA(cudaStreamSynchronize(sw->rng_stream));
                get_stream(st, *sw, rng);
            }
            kmeanspp_fill_device(st, chunkP, w, hmask, cfg.candidates_per_step, rng, evals);
            if (!identity) {
        put_stream(st, *sw, rng);
        BM_CUDA(cudaMemcpyAsync(sw->xslot.p, &d->X, sizeof(void*), cudaMemcpyHostToDevice, st));
    }
        }
        // The next chunk's sample draws follow this chunk's (repair) draws:
        // start them now on rng_stream, overlapping this chunk's Lloyd.  Its
        // target buffer was last read by the previous chunk's resolution.
        const bool next_exists = !identity && (!cfg.has_max_chunks || chunk + 1 < cfg.max_chunks);
        if (next_exists) {
            if (chunk >= 1) BM_CUDA(cudaStreamWaitEvent(sw->rng_stream, sw->resolved[jb ^ 1], 0));
            enqueue_device_draw(sw->rng_stream, *sw, 0, jb ^ 1);
            BM_CUDA(cudaEventRecord(sw->drawn[jb ^ 1], sw->rng_stream));
            drawn_ahead = true;
        }
        {
            LloydResult lr = lloyd_run(st, chunkP, w, cfg.max_iterations, cfg.rel_tolerance);
            evals += lr.evals;
            iterations += lr.iterations;
            enqueue_accept(st, w);
            BM_CUDA(cudaMemcpyAsync(&w.h_status.p->inc_degenerate, &w.status.p->inc_degenerate, sizeof(int),
                                    cudaMemcpyDeviceToHost, st));
            BM_CUDA(cudaStreamSynchronize(st));
            inc_degenerate = w.h_status.p->inc_degenerate;
        }
        out->chunks = chunk + 1;
    }
    }
    if (sw) BM_CUDA(cudaStreamSynchronize(sw->rng_stream));  // a speculative draw may be in flight
    const double cpu_init = seconds_since(t_loop);  // :96
    std::vector<dev::Record> records(out->chunks);
    if (out->chunks)
        BM_CUDA(cudaMemcpyAsync(records.data(), w.drec.p, out->chunks * sizeof(dev::Record), cudaMemcpyDeviceToHost, st));
    double fopt = 0.0;
    BM_CUDA(cudaMemcpyAsync(&fopt, w.fopt.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaMemcpyAsync(out->centroids, w.Cinc.p, (size_t)k * n * sizeof(double), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaMemcpyAsync(out->mask, w.maskinc.p, k, cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    out->cpu_init = cpu_init;
    out->cpu_full = 0.0;
    if (cfg.final_assignment) {  // :102-107
        const auto t_full = std::chrono::steady_clock::now();
        Workspace& fw = get_ws(d, 0, k, 1, 0);  // centroid state only
        launch_compact(st, fw, w.Cinc.p, w.maskinc.p);
        std::vector<double> tiles(tiles_of(m));
        final_pass(st, d, fw, 0, m, out->labels, tiles.data(), &evals);
        double total = 0.0;  // block_sum outer fold (core.cpp:172)
        for (double t : tiles) total += t;
        out->objective = total;
        out->cpu_full = seconds_since(t_full);
    } else {
        out->objective = fopt;  // :108-110
    }
    out->distance_evals = evals;
    out->iterations = iterations;  // :97
    if (persist && out->chunks) {  // device time of the chunk kernels (globaltimer stamps, timed run)
        const uint64_t nc = std::min<uint64_t>(out->chunks, w.ctiming.n / 2);
        std::vector<unsigned long long> tm(2 * nc);
        BM_CUDA(cudaMemcpy(tm.data(), w.ctiming.p, tm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        double ns = 0.0;
        double gap = 0.0;
        for (uint64_t c = 0; c < nc; ++c) ns += (double)(tm[2 * c + 1] - tm[2 * c]);
        for (uint64_t c = 1; c < nc; ++c)
            if (tm[2 * c] > tm[2 * c - 1]) gap += (double)(tm[2 * c] - tm[2 * c - 1]);
        g_profile.chunk_ms_total = ns * 1e-6;
        g_profile.chunk_gap_ms_total = gap * 1e-6;
        g_profile.chunk_launches = nc;
        g_profile.chunk_assign_passes = chunk_assign_passes;
        g_profile.chunk_update_passes = chunk_update_passes;
        g_profile.chunk_rows = s;
    }
    g_last_trace.resize(out->chunks);
    for (uint64_t i = 0; i < out->chunks; ++i) {
        bm_chunk_record& r = g_last_trace[i];
        r.chunk_index = records[i].chunk_index;
        r.candidate_objective = records[i].candidate_objective;
        r.incumbent_objective = records[i].incumbent_objective;
        r.accepted = records[i].accepted;
        r.degenerate_repaired = records[i].degenerate_repaired;
        if (trace && i < trace_cap) trace[i] = r;
    }
    if (g_profiling) g_prof.flush(g_profile);
}

template <class F>
bm_status guarded(F&& f) {
    try {
        f();
        return BM_OK;
    } catch (const ConfigError& e) {
        g_last_error = e.what();
        return BM_CONFIG_ERROR;
    } catch (const StateError& e) {
        g_last_error = e.what();
        return BM_STATE_ERROR;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return BM_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BM_INTERNAL_ERROR;
    }
}

// Upload host centroids (k*n f64 + mask) into w.C / w.mask and compact.
void upload_centroids(cudaStream_t st, Workspace& w, const double* C, const uint8_t* mask) {
    const size_t kn = (size_t)w.k * w.n;
    std::vector<double> tmp(C, C + kn);
    for (int j = 0; j < w.k; ++j)  // degenerate rows hold 0.0 (core.cpp:50-53)
        if (mask[j]) std::fill(tmp.begin() + (size_t)j * w.n, tmp.begin() + (size_t)(j + 1) * w.n, 0.0);
    BM_CUDA(cudaMemcpyAsync(w.C.p, tmp.data(), kn * sizeof(double), cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaMemcpyAsync(w.mask.p, mask, w.k, cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaStreamSynchronize(st));
}

}  // namespace
}  // namespace bm

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace bm;

namespace bm {

// block_sum (core.cpp:163-175) of a device array: ordered 1024-tile folds on
// the device, the tile partials folded in order here.
double device_block_sum(cudaStream_t st, Workspace& w, const double* v, uint64_t count) {
    const uint64_t tiles = tiles_of(count);
    launch_tile_sums(st, v, count, 0, 1, w.tile_buf.p, nullptr);
    std::vector<double> t(tiles);
    BM_CUDA(cudaMemcpyAsync(t.data(), w.tile_buf.p, tiles * sizeof(double), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    double total = 0.0;
    for (double x : t) total += x;
    return total;
}

// forgy_init (init.cpp:92-115): the partial Fisher-Yates touches k slots, so
// the swapped positions are kept in a map instead of the reference's iota(m);
// the chosen rows go to w.C (all active).  No distance evaluations.
void forgy_device(cudaStream_t st, const Points& P, Workspace& w, uint64_t k, Mt64& rng) {
    std::unordered_map<uint64_t, uint64_t> moved;
    auto at = [&](uint64_t i) {
        auto it = moved.find(i);
        return it == moved.end() ? i : it->second;
    };
    std::vector<uint64_t> rows(k);
    for (uint64_t i = 0; i < k; ++i) {
        const uint64_t j = rng.uniform_int(i, P.rows - 1);
        const uint64_t vi = at(i), vj = at(j);
        moved[i] = vj;
        moved[j] = vi;
        rows[i] = vj;
    }
    for (uint64_t i = 0; i < k; ++i) set_row_any(st, P, w, rows[i], (int)i);
}

// kmeans_parallel_init (init.cpp:209-347) on the device: D^2 passes, per-point
// round draws, candidate weights and the weighted reduction run as kernels;
// the host keeps the stream between them and the short index bookkeeping.
void kmeans_parallel_device(cudaStream_t st, const bm_dataset* d, const Points& P, Workspace& w, uint64_t k,
                            const bm_init_config& cfg, Mt64& rng, uint64_t& evals) {
    const uint64_t m = P.rows;
    const int n = P.n;
    const uint64_t first = rng.uniform_int(0, m - 1);  // :220-221
    if (k == 1) {                                       // :222-225
        set_row_any(st, P, w, first, 0);
        return;
    }
    const double l = cfg.oversampling_l > 0 ? (double)cfg.oversampling_l : 2.0 * (double)k;  // :227-228
    std::vector<uint32_t> cand{(uint32_t)first};
    DevBuf<uint32_t> dcand(1);
    double* d2 = w.d2pool.p;  // dist2 (m)
    BM_CUDA(cudaMemcpyAsync(dcand.p, cand.data(), sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    launch_dist_rows(st, P, dcand.p, 1, nullptr, d2);  // :232
    evals += m;
    int rounds = cfg.rounds_r;  // :234-238
    if (cfg.rounds_rule == 1) {
        const double phi1 = device_block_sum(st, w, d2, m);
        rounds = phi1 > 1.0 ? std::max(1, (int)std::floor(std::log(phi1))) : 1;
    }
    if (rounds < 1) throw ConfigError("kmeans_parallel_init: rounds_r must be at least 1");  // :239-241
    const uint64_t words = ceil_div(m, 32);
    DevBuf<uint32_t> bits(words);
    std::vector<uint32_t> hbits(words);
    DevBuf<Mt64State> dmt(2);
    DevBuf<uint64_t> raw;
    DevBuf<int> flag(1);
    HostBuf<Mt64State> hmt;
    hmt.alloc(1);
    for (int round = 0; round < rounds; ++round) {  // :244-263
        const double phi = device_block_sum(st, w, d2, m);
        if (phi <= 0.0) break;
        // one uniform_real(0, 1) per point, in index order (:251-258)
        if (!raw.n) raw.alloc(m);
        *hmt.p = rng.s;
        BM_CUDA(cudaMemcpyAsync(dmt.p, hmt.p, sizeof(Mt64State), cudaMemcpyHostToDevice, st));
        if (m > 0xFFFFFFFFull) throw ConfigError("kmeans_parallel_init: too many rows for the device draws");
        dev::k_mt_twist<<<1, dev::kMtThreads, 0, st>>>(dmt.p, dmt.p + 1, (uint32_t)m, raw.p, flag.p);
        BM_LAUNCH();
        dev::k_kpar_bern<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(raw.p, d2, m, l, phi, bits.p);
        BM_LAUNCH();
        BM_CUDA(cudaMemcpyAsync(hmt.p, dmt.p, sizeof(Mt64State), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(hbits.data(), bits.p, words * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        rng.s = *hmt.p;
        count_launch(2);
        std::vector<uint32_t> fresh;
        for (uint64_t wi = 0; wi < words; ++wi)
            for (uint32_t b = hbits[wi]; b; b &= b - 1) fresh.push_back((uint32_t)(wi * 32 + __builtin_ctz(b)));
        if (fresh.empty()) continue;
        cand.insert(cand.end(), fresh.begin(), fresh.end());  // :259-262 (lower_to_row per fresh row)
        DevBuf<uint32_t> df(fresh.size());
        BM_CUDA(cudaMemcpyAsync(df.p, fresh.data(), fresh.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        dispatch(P.dtype, [&](auto tag) {
            using T = decltype(tag);
            dev::k_kpar_lower<T><<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(static_cast<const T*>(P.X), m, n, P.ld,
                                                                             df.p, (int)fresh.size(), d2);
        });
        BM_LAUNCH();
        BM_CUDA(cudaStreamSynchronize(st));
        count_launch();
        evals += m * (uint64_t)fresh.size();
    }
    if (cand.size() < k) {  // top-up with distinct uniform rows (:266-278)
        std::vector<uint8_t> used(m, 0);
        for (uint32_t i : cand) used[i] = 1;
        while (cand.size() < k) {
            const uint64_t i = rng.uniform_int(0, m - 1);
            if (!used[i]) {
                used[i] = 1;
                cand.push_back((uint32_t)i);
            }
        }
    }
    const uint64_t nc = cand.size();
    // candidate rows (fp64) and weights: points nearest each candidate (:280-295)
    DevBuf<uint32_t> dall(nc);
    BM_CUDA(cudaMemcpyAsync(dall.p, cand.data(), nc * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    DevBuf<double> Cc(nc * n);
    dispatch(P.dtype, [&](auto tag) {
        using T = decltype(tag);
        dev::k_rows_f64<T><<<(unsigned)std::min<uint64_t>(ceil_div(nc * n, 256), 1184), 256, 0, st>>>(
            static_cast<const T*>(P.X), P.ld, n, dall.p, nc, Cc.p);
    });
    BM_LAUNCH();
    DevBuf<int> act(nc), nact(1);
    {
        std::vector<int> a(nc);
        for (uint64_t q = 0; q < nc; ++q) a[q] = (int)q;
        const int na = (int)nc;
        BM_CUDA(cudaMemcpyAsync(act.p, a.data(), nc * sizeof(int), cudaMemcpyHostToDevice, st));
        BM_CUDA(cudaMemcpyAsync(nact.p, &na, sizeof(int), cudaMemcpyHostToDevice, st));
        BM_CUDA(cudaStreamSynchronize(st));
    }
    int32_t* lab = w.labels.p;
    double* dd = w.dists.p;
    dispatch(P.dtype, [&](auto tag) {  // exact assign_nearest over the candidates (core.cpp:106-161)
        using T = decltype(tag);
        dev::k_assign<T><<<(unsigned)ceil_div(m, dev::kABP), assign_threads((int)nc), 0, st>>>(
            static_cast<const T*>(P.X), m, n, P.ld, Cc.p, n, act.p, nact.p, lab, 0, nullptr, dd, nullptr, nullptr);
    });
    BM_LAUNCH();
    evals += m * nc;
    DevBuf<unsigned long long> cnt(nc);
    BM_CUDA(cudaMemsetAsync(cnt.p, 0, nc * sizeof(unsigned long long), st));
    dev::k_kpar_count<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(lab, m, cnt.p);
    BM_LAUNCH();
    // weighted greedy k-means++ over the candidates (:297-339), one CTA
    DevBuf<double> scratch(4 * nc);
    DevBuf<uint32_t> chosen(k);
    DevBuf<unsigned long long> dev_ev(1);
    *hmt.p = rng.s;
    BM_CUDA(cudaMemcpyAsync(dmt.p, hmt.p, sizeof(Mt64State), cudaMemcpyHostToDevice, st));
    dev::k_kpar_reduce<<<1, 256, 0, st>>>(Cc.p, n, cnt.p, nc, (int)k, std::max(1, cfg.candidates_per_step), dmt.p,
                                          scratch.p, chosen.p, dev_ev.p);
    BM_LAUNCH();
    count_launch(5);
    std::vector<uint32_t> hch(k);
    unsigned long long hev = 0;
    BM_CUDA(cudaMemcpyAsync(hmt.p, dmt.p, sizeof(Mt64State), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaMemcpyAsync(hch.data(), chosen.p, k * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaMemcpyAsync(&hev, dev_ev.p, sizeof(hev), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    rng.s = *hmt.p;
    evals += hev;
    for (uint64_t j = 0; j < k; ++j)  // :341-346
        BM_CUDA(cudaMemcpyAsync(w.C.p + j * n, Cc.p + (uint64_t)hch[j] * n, n * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    BM_CUDA(cudaMemsetAsync(w.mask.p, 0, k, st));
    (void)d;
}

// choose_chunk_size_hint (big_means.cpp:114-160): short big_means probes per
// ladder size; the best mean final objective wins, ties to the smaller size.
uint64_t choose_chunk_size_hint(bm_dataset* d, uint64_t k, std::vector<uint64_t> ladder, uint64_t chunks_per,
                                uint64_t runs_per, uint64_t max_iterations, double rel_tolerance, int candidates,
                                uint64_t seed, double* best_mean_out) {
    const uint64_t m = d->m;
    if (k < 1 || m < k) throw ConfigError("choose_chunk_size_hint: need at least k points");
    if (chunks_per < 1 || runs_per < 1) throw ConfigError("choose_chunk_size_hint: probe budget must be positive");
    if (ladder.empty())
        for (uint64_t div = 64; div >= 1; div /= 2) ladder.push_back(std::max(k, m / div));
    for (uint64_t& s : ladder) s = std::clamp(s, k, m);
    std::sort(ladder.begin(), ladder.end());
    ladder.erase(std::unique(ladder.begin(), ladder.end()), ladder.end());
    double best_mean = std::numeric_limits<double>::infinity();
    uint64_t best_s = ladder.front();
    std::vector<double> C(k * d->n);
    std::vector<uint8_t> mask(k);
    for (uint64_t s : ladder) {
        double sum = 0.0;
        for (uint64_t run = 0; run < runs_per; ++run) {
            bm_config probe{};
            bm_config_init(&probe);
            probe.k = k;
            probe.chunk_size = s;
            probe.has_max_chunks = 1;
            probe.max_chunks = chunks_per;
            probe.max_iterations = max_iterations;
            probe.rel_tolerance = rel_tolerance;
            probe.candidates_per_step = candidates;
            probe.seed = seed + run;
            probe.final_assignment = 1;
            bm_outcome o{};
            o.centroids = C.data();
            o.mask = mask.data();
            big_means(d, probe, &o, nullptr, 0);
            sum += o.objective;
        }
        const double mean = sum / static_cast<double>(runs_per);
        if (mean < best_mean) {  // strict: ties keep the smaller size
            best_mean = mean;
            best_s = s;
        }
    }
    if (best_mean_out) *best_mean_out = best_mean;
    return best_s;
}

// kmeans (local_search.cpp:62-94): init per method (init.seed), then lloyd.
// The initialization stage of kmeans (local_search.cpp:66-83): w.C / w.mask
// hold the start centroids afterwards; returns the init's distance evals.
uint64_t init_stage(cudaStream_t st, const bm_dataset* d, Workspace& w, uint64_t k, const bm_init_config& init) {
    if (k < 1) throw ConfigError("kmeans: k must be at least 1");
    if (d->m < k) throw ConfigError("kmeans: dataset has fewer points than clusters");
    if (init.method < 0 || init.method > 2) throw ConfigError("kmeans: unknown initialization method");
    Mt64 rng(init.seed);  // :71
    BM_CUDA(cudaMemsetAsync(w.C.p, 0, k * d->n * sizeof(double), st));
    BM_CUDA(cudaMemsetAsync(w.mask.p, 1, k, st));
    uint64_t init_evals = 0;
    Points P = dataset_points(d);
    if (init.method == 0) {
        forgy_device(st, P, w, k, rng);
    } else if (init.method == 1) {
        std::vector<uint8_t> hmask(k, 1);
        kmeanspp_fill_device(st, P, w, hmask, init.candidates_per_step, rng, init_evals);
    } else {
        kmeans_parallel_device(st, d, P, w, k, init, rng, init_evals);
    }
    BM_CUDA(cudaStreamSynchronize(st));
    return init_evals;
}

void kmeans(const bm_dataset* d, uint64_t k, const bm_init_config& init, uint64_t max_iterations,
            double rel_tolerance, bm_outcome* out) {
    if (k < 1) throw ConfigError("kmeans: k must be at least 1");
    if (d->m < k) throw ConfigError("kmeans: dataset has fewer points than clusters");
    if (max_iterations < 1) throw ConfigError("lloyd: max_iterations must be at least 1");
    if (rel_tolerance < 0.0) throw ConfigError("lloyd: rel_tolerance must be nonnegative");
    if (init.method < 0 || init.method > 2) throw ConfigError("kmeans: unknown initialization method");
    DeviceGuard g(d->device);
    cudaStream_t st = stream_of(d);
    Workspace& w = get_ws(d, d->m, (int)k, std::max(1, init.candidates_per_step), 0);
    const auto t_init = std::chrono::steady_clock::now();
    const uint64_t init_evals = init_stage(st, d, w, k, init);
    out->cpu_init = seconds_since(t_init);
    const auto t_search = std::chrono::steady_clock::now();
    Points P = dataset_points(d);
    LloydResult r = lloyd_run(st, P, w, max_iterations, rel_tolerance);
    BM_CUDA(cudaMemcpyAsync(out->centroids, w.C.p, k * d->n * sizeof(double), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaMemcpyAsync(out->mask, w.mask.p, k, cudaMemcpyDeviceToHost, st));
    if (out->labels)
        BM_CUDA(cudaMemcpyAsync(out->labels, w.labels.p + (uint64_t)r.parity * w.R, d->m * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    out->cpu_full = seconds_since(t_search);
    out->objective = r.objective;
    out->distance_evals = r.evals + init_evals;
    out->iterations = r.iterations;
    out->chunks = 1;
}

// ---------------------------------------------------------------------------
// Multi-GPU Big-means in one process (paper mode 2):
// chain g = big_means with seed + g and floor(N/G) (+1 for g < N mod G) of the
// N chunks, on its own dataset handle (one per GPU); one host thread per
// device (chains sharing a device run one after the other on that device's
// thread); the lowest-index chain with the minimum f_opt wins; the final pass
// is row-sharded over the distinct devices on 1024-row tiles and the tile
// partials are folded in row order (bit-identical to block_sum, core.cpp:165-175).
// ---------------------------------------------------------------------------
uint64_t chain_chunks(uint64_t N, int g, int G) { return N / G + ((uint64_t)g < N % G ? 1 : 0); }

void big_means_multi(bm_dataset* const* data, int G, const bm_config& cfg, bm_outcome* out, bm_chunk_record* trace,
                     uint64_t trace_cap, uint64_t* chain_chunk_counts, int* winner_out) {
    if (G < 1) throw ConfigError("big_means_multi: at least one chain");
    for (int g = 0; g < G; ++g) {
        if (!data[g]) throw ConfigError("big_means_multi: null dataset handle");
        if (data[g]->m != data[0]->m || data[g]->n != data[0]->n)
            throw ConfigError("big_means_multi: every chain needs the same dataset");
        validate(data[g], cfg);
    }
    if (cfg.has_max_chunks && cfg.max_chunks < (uint64_t)G)
        throw ConfigError("big_means_multi: fewer chunks than chains");
    const uint64_t k = cfg.k, n = data[0]->n, m = data[0]->m;
    struct Chain {
        std::vector<double> C;
        std::vector<uint8_t> mask;
        bm_outcome o{};
        std::vector<bm_chunk_record> recs;
    };
    std::vector<Chain> ch(G);
    std::vector<int> devs;
    for (int g = 0; g < G; ++g)
        if (std::find(devs.begin(), devs.end(), data[g]->device) == devs.end()) devs.push_back(data[g]->device);
    std::vector<std::string> errs(devs.size());
    std::vector<bm_status> codes(devs.size(), BM_OK);
    auto run_threads = [&](auto&& body) {
        std::vector<std::thread> th;
        for (size_t di = 0; di < devs.size(); ++di)
            th.emplace_back([&, di] {
                codes[di] = guarded([&] { body(di, devs[di]); });
                if (codes[di] != BM_OK) errs[di] = g_last_error;
            });
        for (auto& t : th) t.join();
        for (size_t di = 0; di < devs.size(); ++di)
            if (codes[di] != BM_OK) {
                if (codes[di] == BM_CONFIG_ERROR) throw ConfigError(errs[di]);
                if (codes[di] == BM_STATE_ERROR) throw StateError(errs[di]);
                throw CudaError(errs[di]);
            }
    };
    // 1. the chains
    run_threads([&](size_t, int dev) {
        for (int g = 0; g < G; ++g) {
            if (data[g]->device != dev) continue;
            bm_config c = cfg;
            c.seed = cfg.seed + (uint64_t)g;
            if (cfg.has_max_chunks) c.max_chunks = chain_chunks(cfg.max_chunks, g, G);
            c.final_assignment = 0;
            Chain& x = ch[g];
            x.C.assign(k * n, 0.0);
            x.mask.assign(k, 1);
            x.o.centroids = x.C.data();
            x.o.mask = x.mask.data();
            x.o.labels = nullptr;
            big_means(data[g], c, &x.o, nullptr, 0);
            x.recs = g_last_trace;
        }
    });
    // 2. select: the first chain with the minimum f_opt (strict <)
    int w = 0;
    double best = std::numeric_limits<double>::infinity();
    for (int g = 0; g < G; ++g)
        if (ch[g].o.objective < best) {
            best = ch[g].o.objective;
            w = g;
        }
    uint64_t evals = 0, iters = 0, chunks = 0, rec_i = 0;
    double loop_wall = 0.0;
    for (int g = 0; g < G; ++g) {
        evals += ch[g].o.distance_evals;
        iters += ch[g].o.iterations;
        chunks += ch[g].o.chunks;
        loop_wall = std::max(loop_wall, ch[g].o.cpu_init);
        if (chain_chunk_counts) chain_chunk_counts[g] = ch[g].o.chunks;
        for (const auto& r : ch[g].recs)
            if (trace && rec_i < trace_cap) trace[rec_i++] = r;
    }
    std::copy(ch[w].C.begin(), ch[w].C.end(), out->centroids);
    std::copy(ch[w].mask.begin(), ch[w].mask.end(), out->mask);
    out->cpu_init = loop_wall;
    out->cpu_full = 0.0;
    out->objective = best;
    if (cfg.final_assignment) {
        // 3. row-sharded final pass: device di assigns whole tiles [t0, t1)
        const auto t_full = std::chrono::steady_clock::now();
        const uint64_t T = tiles_of(m), D = devs.size();
        std::vector<double> tiles(T);
        std::vector<uint64_t> fe(D, 0);
        run_threads([&](size_t di, int dev) {
            const uint64_t t0 = di * (T / D) + std::min<uint64_t>(di, T % D);
            const uint64_t t1 = t0 + T / D + (di < T % D ? 1 : 0);
            const uint64_t r0 = std::min(m, t0 * kTile), r1 = std::min(m, t1 * kTile);
            if (r1 <= r0) return;
            const bm_dataset* d = nullptr;
            for (int g = 0; g < G; ++g)
                if (data[g]->device == dev) {
                    d = data[g];
                    break;
                }
            DeviceGuard dg(dev);
            Workspace& fw = get_ws(d, 0, (int)k, 1, 0);
            upload_centroids(stream_of(d), fw, ch[w].C.data(), ch[w].mask.data());
            launch_compact(stream_of(d), fw, fw.C.p, fw.mask.p);
            final_pass(stream_of(d), d, fw, r0, r1, out->labels ? out->labels + r0 : nullptr, tiles.data() + t0,
                       &fe[di]);
        });
        double total = 0.0;  // block_sum outer fold over all tiles in row order (core.cpp:172)
        for (double t : tiles) total += t;
        out->objective = total;
        for (uint64_t e : fe) evals += e;
        out->cpu_full = seconds_since(t_full);
    }
    out->distance_evals = evals;
    out->iterations = iters;
    out->chunks = chunks;
    if (winner_out) *winner_out = w;
}

}  // namespace bm

extern "C" {

const char* bm_last_error(void) { return g_last_error.c_str(); }
int bm_abi_version(void) { return BM_ABI_VERSION; }

void bm_config_init(bm_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->max_iterations = 300;   // local_search.hpp:11
    c->rel_tolerance = 1e-4;   // local_search.hpp:14
    c->candidates_per_step = 3;  // init.hpp:18
    c->seed = 123456789ULL;    // kDefaultSeed common.hpp:17
    c->final_assignment = 1;   // big_means.hpp:25
}

bm_status bm_device_count(int* count) {
    return guarded([&] {
        BM_CUDA(cudaGetDeviceCount(count));
        if (*count < 1) throw CudaError("no CUDA device");
    });
}

bm_status bm_dataset_create(const void* values, uint64_t m, uint64_t n, bm_dtype dtype, int device,
                            bm_dataset** out) {
    return guarded([&] {
        *out = nullptr;
        if (m < 1 || n < 1) throw ConfigError("dataset must have at least one row and one column");
        if (dtype != BM_F64 && dtype != BM_F32) throw ConfigError("dataset dtype must be f64 or f32");
        if (m >= 0xFFFFFFFFull) throw ConfigError("dataset too large for 32-bit row indices");
        DeviceGuard g(device);
        auto d = std::make_unique<bm_dataset>();
        d->device = device;
        d->m = m;
        d->n = n;
        d->dtype = dtype;
        BM_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
        // [0] non-finite, [1] not exactly representable in fp32, [2] lowest set
        // bit exponent, [4:6] largest |value| (bits): the exact-sum test
        DevBuf<int> flags(6);
        BM_CUDA(cudaMemsetAsync(flags.p, 0, 6 * sizeof(int), d->stream));
        BM_CUDA(cudaMemsetAsync(flags.p + 2, 0x7F, sizeof(int), d->stream));
        int hf[6] = {0, 0, 0, 0, 0, 0};
        unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(flags.p + 4);
        // datasets come and go (one per e2e step): stream-ordered allocations from a
        // pool that keeps its memory, instead of a fresh cudaMalloc each time
        {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            cudaGetLastError();
        }
        if (dtype == BM_F64 && narrow_storage()) {
            // Stage the fp64 values, check them (Dataset ctor scan core.cpp:27-31 +
            // fp32 round trip), keep fp32 storage when lossless.
            double* tmp = nullptr;
            BM_CUDA(cudaMallocAsync(&tmp, m * n * sizeof(double), d->stream));
            struct Tmp {
                double* p;
                cudaStream_t s;
                ~Tmp() { cudaFreeAsync(p, s); }
            } tmp_guard{tmp, d->stream};
            // Uploaded in row pieces; each piece is checked and narrowed (speculatively,
            // one pass) on a second stream while the next piece is in flight.
            const uint64_t ld32 = padded_ld(n, BM_F32);
            float* x32 = nullptr;
            BM_CUDA(cudaMallocAsync(&x32, m * ld32 * sizeof(float), d->stream));
            cudaStream_t ks = nullptr;
            BM_CUDA(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
            struct KS {
                cudaStream_t s;
                ~KS() { cudaStreamDestroy(s); }
            } ks_guard{ks};
            constexpr int kPieces = 8;
            const uint64_t per = ceil_div(m, (uint64_t)kPieces);
            for (uint64_t r0 = 0; r0 < m; r0 += per) {
                const uint64_t r1 = std::min(m, r0 + per);
                BM_CUDA(cudaMemcpyAsync(tmp + r0 * n, static_cast<const double*>(values) + r0 * n,
                                        (r1 - r0) * n * sizeof(double), cudaMemcpyHostToDevice, d->stream));
                cudaEvent_t ev;
                BM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                BM_CUDA(cudaEventRecord(ev, d->stream));
                BM_CUDA(cudaStreamWaitEvent(ks, ev, 0));
                BM_CUDA(cudaEventDestroy(ev));
                dev::k_check_narrow_write<<<592, 256, 0, ks>>>(tmp, r0, r1, (int)n, flags.p, flags.p + 1, flags.p + 2,
                                                               maxbits, x32, ld32, flags.p + 3);
                BM_LAUNCH();
            }
            BM_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, ks));
            BM_CUDA(cudaStreamSynchronize(ks));
            BM_CUDA(cudaStreamSynchronize(d->stream));
            if (hf[0]) {
                cudaFreeAsync(x32, d->stream);
                throw ConfigError("dataset contains a non-finite value");
            }
            d->dtype = hf[1] ? BM_F64 : BM_F32;
            d->ld = padded_ld(n, d->dtype);
            if (d->dtype == BM_F32) {
                d->X = x32;
            } else {
                BM_CUDA(cudaFreeAsync(x32, d->stream));
                BM_CUDA(cudaMallocAsync(&d->X, m * d->ld * dtype_size(d->dtype), d->stream));
                BM_CUDA(cudaMemcpy2DAsync(d->X, d->ld * sizeof(double), tmp, n * sizeof(double), n * sizeof(double),
                                          m, cudaMemcpyDeviceToDevice, d->stream));
            }
            BM_CUDA(cudaStreamSynchronize(d->stream));
        } else {
            d->ld = padded_ld(n, dtype);
            const size_t es = dtype_size(dtype);
            BM_CUDA(cudaMallocAsync(&d->X, m * d->ld * es, d->stream));
            if (d->ld == n) {
                BM_CUDA(cudaMemcpyAsync(d->X, values, m * n * es, cudaMemcpyHostToDevice, d->stream));
            } else {
                BM_CUDA(cudaMemcpy2DAsync(d->X, d->ld * es, values, n * es, n * es, m, cudaMemcpyHostToDevice,
                                          d->stream));
            }
            // Dataset ctor finiteness scan (core.cpp:27-31)
            dispatch(dtype, [&](auto tag) {
                using T = decltype(tag);
                dev::k_check_finite<T><<<1184, 256, 0, d->stream>>>(static_cast<const T*>(d->X), m, (int)n, d->ld,
                                                                    flags.p, flags.p + 2, maxbits, flags.p + 3);
            });
            BM_LAUNCH();
            BM_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, d->stream));
            BM_CUDA(cudaStreamSynchronize(d->stream));
            if (hf[0]) throw ConfigError("dataset contains a non-finite value");
        }
        d->tf32_exact = d->dtype == BM_F32 && hf[3] == 0;
        {  // exact-sum test (kernels.cuh §5b): every value k * 2^e, m * max|x| < 2^52 * 2^e
            unsigned long long mb = 0;
            std::memcpy(&mb, hf + 4, sizeof(mb));
            double mx = 0.0;
            std::memcpy(&mx, &mb, sizeof(mx));
            const int e = hf[2] == 0x7F7F7F7F ? 0 : hf[2];  // all zeros: any exponent
            if (e >= -960 && e <= 960) {
                const double units = std::ldexp(mx, -e);  // an integer (exact)
                d->exact_sums = units * (double)m < 0x1p52;
                d->sum_exp = e;
                d->sum_units_max = units;
            }
        }
        *out = d.release();
    });
}

bm_status bm_dataset_destroy(bm_dataset* d) {
    return guarded([&] {
        if (!d) return;
        DeviceGuard g(d->device);
        delete d;
    });
}

bm_status bm_dataset_storage(const bm_dataset* d, bm_dtype* storage) {
    return guarded([&] { *storage = d->dtype; });
}

bm_status bm_dataset_sum_mode(const bm_dataset* d, int32_t* exact, int32_t* exponent) {
    return guarded([&] {
        *exact = d->exact_sums ? 1 : 0;
        *exponent = d->sum_exp;
    });
}

bm_status bm_dataset_min_max_normalize(const bm_dataset* d, bm_dataset** out) {
    return guarded([&] {
        *out = nullptr;
        DeviceGuard g(d->device);
        cudaStream_t st = stream_of(d);
        const int n = (int)d->n;
        DevBuf<unsigned long long> lo(n), hi(n);
        BM_CUDA(cudaMemsetAsync(lo.p, 0xFF, n * sizeof(unsigned long long), st));
        BM_CUDA(cudaMemsetAsync(hi.p, 0, n * sizeof(unsigned long long), st));
        DevBuf<double> tmp(d->m * d->n);
        dispatch(d->dtype, [&](auto tag) {
            using T = decltype(tag);
            const int threads = std::max(1, 256 / n) * n;  // whole rows per CTA pass
            if (n <= 256) {
                dev::k_col_minmax<T><<<592, threads, 0, st>>>(static_cast<const T*>(d->X), d->m, n, d->ld, lo.p,
                                                               hi.p);
            } else {
                for (int c0 = 0; c0 < n; c0 += 256) {  // column blocks of 256 (one row per thread group)
                    const int nc = std::min(256, n - c0);
                    dev::k_col_minmax<T><<<592, nc, 0, st>>>(static_cast<const T*>(d->X) + c0, d->m, nc, d->ld,
                                                              lo.p + c0, hi.p + c0);
                }
            }
            BM_LAUNCH();
            dev::k_minmax_apply<T><<<1184, 256, 0, st>>>(static_cast<const T*>(d->X), d->m, n, d->ld, lo.p, hi.p,
                                                         tmp.p);
            BM_LAUNCH();
        });
        std::vector<double> host(d->m * d->n);  // the normalized values re-enter through the dataset checks
        BM_CUDA(cudaMemcpyAsync(host.data(), tmp.p, host.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        const bm_status s = bm_dataset_create(host.data(), d->m, d->n, BM_F64, d->device, out);
        if (s != BM_OK) throw StateError(bm_last_error());
    });
}

bm_status bm_dataset_shape(const bm_dataset* d, uint64_t* m, uint64_t* n) {
    return guarded([&] {
        *m = d->m;
        *n = d->n;
    });
}

bm_status bm_dataset_gather(const bm_dataset* d, const uint64_t* rows, uint64_t count, bm_dataset** out) {
    return guarded([&] {
        *out = nullptr;
        for (uint64_t i = 0; i < count; ++i)
            if (rows[i] >= d->m) throw ConfigError("gather index out of range");
        if (count < 1) throw ConfigError("dataset must have at least one row and one column");
        DeviceGuard g(d->device);
        auto o = std::make_unique<bm_dataset>();
        o->device = d->device;
        o->m = count;
        o->n = d->n;
        o->dtype = d->dtype;
        o->ld = d->ld;
        o->exact_sums = d->exact_sums;  // a subset of the rows keeps the exact-sum property
        o->tf32_exact = d->tf32_exact;
        o->sum_exp = d->sum_exp;
        o->sum_units_max = d->sum_units_max;
        BM_CUDA(cudaStreamCreateWithFlags(&o->stream, cudaStreamNonBlocking));
        BM_CUDA(cudaMallocAsync(&o->X, count * o->ld * dtype_size(o->dtype), o->stream));
        DevBuf<uint64_t> idx(count);
        BM_CUDA(cudaMemcpyAsync(idx.p, rows, count * sizeof(uint64_t), cudaMemcpyHostToDevice, o->stream));
        dispatch(d->dtype, [&](auto tag) {
            using T = decltype(tag);
            dev::k_gather_checked<T><<<592, 256, 0, o->stream>>>(static_cast<const T*>(d->X), d->ld, (int)d->n,
                                                                 idx.p, count, static_cast<T*>(o->X), o->ld);
        });
        BM_LAUNCH();
        BM_CUDA(cudaStreamSynchronize(o->stream));
        *out = o.release();
    });
}

bm_status bm_dataset_download(const bm_dataset* d, double* out) {
    return guarded([&] {
        DeviceGuard g(d->device);
        DevBuf<double> tmp(d->m * d->n);
        dispatch(d->dtype, [&](auto tag) {
            using T = decltype(tag);
            dev::k_promote<T><<<592, 256, 0, d->stream>>>(static_cast<const T*>(d->X), d->m, (int)d->n, d->ld, tmp.p);
        });
        BM_LAUNCH();
        BM_CUDA(cudaMemcpyAsync(out, tmp.p, d->m * d->n * sizeof(double), cudaMemcpyDeviceToHost, d->stream));
        BM_CUDA(cudaStreamSynchronize(d->stream));
    });
}

bm_status bm_rng_create(uint64_t seed, bm_rng** out) {
    return guarded([&] { *out = new bm_rng{Mt64(seed)}; });
}
bm_status bm_rng_destroy(bm_rng* r) {
    return guarded([&] { delete r; });
}
uint64_t bm_rng_next(bm_rng* r) { return r->eng(); }
uint64_t bm_rng_uniform_int(bm_rng* r, uint64_t a, uint64_t b) { return r->eng.uniform_int(a, b); }
double bm_rng_uniform_real(bm_rng* r, double a, double b) { return r->eng.uniform_real(a, b); }

bm_status bm_sample_chunk_device(const bm_dataset* d, uint64_t s, bm_rng* rng, int force_sequential,
                                 uint64_t* out) {
    return guarded([&] {
        const uint64_t m = d->m;
        if (s < 1 || s >= m) throw ConfigError("sample_chunk_device: need 1 <= s < m");
        DeviceGuard g(d->device);
        SamplerWs& sw = get_sws(d, s);
        cudaStream_t st = stream_of(d);
        put_stream(st, sw, rng->eng);
        enqueue_device_draw(st, sw, force_sequential);
        enqueue_resolve_device(st, sw);
        std::vector<uint32_t> tmp(s);
        BM_CUDA(cudaMemcpyAsync(tmp.data(), sw.idx.p, s * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        get_stream(st, sw, rng->eng);
        for (uint64_t i = 0; i < s; ++i) out[i] = tmp[i];
    });
}

bm_status bm_sample_chunk(const bm_dataset* dc, uint64_t s, bm_rng* rng, uint64_t* out) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        const uint64_t m = d->m;
        if (s < 1 || s > m) throw ConfigError("sample_chunk: chunk size must be in [1, m]");
        if (s == m) {  // :46-48
            for (uint64_t i = 0; i < m; ++i) out[i] = i;
            return;
        }
        DeviceGuard g(d->device);
        SamplerWs& sw = get_sws(d, s);
        draw_targets(sw, rng->eng);
        enqueue_resolve(stream_of(d), sw);
        std::vector<uint32_t> tmp(s);
        BM_CUDA(cudaMemcpyAsync(tmp.data(), sw.idx.p, s * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream_of(d)));
        BM_CUDA(cudaStreamSynchronize(stream_of(d)));
        for (uint64_t i = 0; i < s; ++i) out[i] = tmp[i];
    });
}

bm_status bm_sample_chunk_draws(uint64_t m, uint64_t s, const uint32_t* draws, int device, uint64_t* out) {
    return guarded([&] {
        if (s < 1 || s >= m) throw ConfigError("sample_chunk_draws: need 1 <= s < m");
        if (m >= 0xFFFFFFFFull) throw ConfigError("dataset too large for 32-bit row indices");
        for (uint64_t i = 0; i < s; ++i)
            if (draws[i] < i || draws[i] >= m) throw ConfigError("sample_chunk_draws: draw out of range");
        DeviceGuard g(device);
        SamplerWs& sw = get_sws_dev(device, m, s);
        cudaStream_t st = cache_of(device).stream;
        BM_CUDA(cudaEventSynchronize(sw.js_done[sw.cur]));
        std::memcpy(sw.h_js[sw.cur].p, draws, s * sizeof(uint32_t));
        enqueue_resolve(st, sw);
        std::vector<uint32_t> tmp(s);
        BM_CUDA(cudaMemcpyAsync(tmp.data(), sw.idx.p, s * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < s; ++i) out[i] = tmp[i];
    });
}

bm_status bm_assign_nearest(const bm_dataset* dc, const double* C, const uint8_t* mask, uint64_t k,
                            int32_t* labels, double* dists, uint64_t* evals) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        if (k < 1) throw ConfigError("centroids must have at least one row and one column");
        DeviceGuard g(d->device);
        Workspace& w = get_ws(d, 0, (int)k, 1, 0);
        upload_centroids(stream_of(d), w, C, mask);
        launch_compact(stream_of(d), w, w.C.p, w.mask.p);
        DevBuf<int32_t> dl(d->m);
        DevBuf<double> dd(d->m);
        Points P = dataset_points(d);
        launch_assign(stream_of(d), P, w, (int)k, dl.p, 0, nullptr, dd.p, nullptr, nullptr);
        int na = 0;
        BM_CUDA(cudaMemcpyAsync(&na, &w.gs.p->n_active, sizeof(int), cudaMemcpyDeviceToHost, stream_of(d)));
        BM_CUDA(cudaStreamSynchronize(stream_of(d)));
        if (na == 0) throw StateError("assign_nearest: every centroid is degenerate");
        BM_CUDA(cudaMemcpyAsync(labels, dl.p, d->m * sizeof(int32_t), cudaMemcpyDeviceToHost, stream_of(d)));
        if (dists) BM_CUDA(cudaMemcpyAsync(dists, dd.p, d->m * sizeof(double), cudaMemcpyDeviceToHost, stream_of(d)));
        BM_CUDA(cudaStreamSynchronize(stream_of(d)));
        if (evals) *evals += d->m * (uint64_t)na;
    });
}

bm_status bm_assign_rows(const bm_dataset* dc, const double* C, const uint8_t* mask, uint64_t k,
                         uint64_t row_begin, uint64_t row_end, int32_t* labels, double* tile_partials,
                         uint64_t* evals) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        if (k < 1) throw ConfigError("centroids must have at least one row and one column");
        if (row_begin % kTile != 0 || row_begin > row_end || row_end > d->m)
            throw ConfigError("assign_rows: row range must start on a 1024-row tile and lie in [0, m]");
        if (row_begin == row_end) return;
        DeviceGuard g(d->device);
        Workspace& w = get_ws(d, 0, (int)k, 1, 0);
        upload_centroids(stream_of(d), w, C, mask);
        launch_compact(stream_of(d), w, w.C.p, w.mask.p);
        final_pass(stream_of(d), d, w, row_begin, row_end, labels, tile_partials, evals);
    });
}

bm_status bm_objective(const bm_dataset* d, const double* C, const uint8_t* mask, uint64_t k, double* objective,
                       uint64_t* evals) {
    return guarded([&] {
        std::vector<double> tiles(tiles_of(d->m));
        bm_status rc = bm_assign_rows(d, C, mask, k, 0, d->m, nullptr, tiles.data(), evals);
        if (rc != BM_OK) {
            if (rc == BM_CONFIG_ERROR) throw ConfigError(g_last_error);
            if (rc == BM_STATE_ERROR) throw StateError(g_last_error);
            throw std::runtime_error(g_last_error);
        }
        double total = 0.0;
        for (double t : tiles) total += t;
        *objective = total;
    });
}

bm_status bm_block_sum(const double* values, uint64_t count, int device, double* out) {
    return guarded([&] {
        if (count == 0) {
            *out = 0.0;
            return;
        }
        DeviceGuard g(device);
        DevBuf<double> dv(count), dt(tiles_of(count));
        BM_CUDA(cudaMemcpy(dv.p, values, count * sizeof(double), cudaMemcpyHostToDevice));
        launch_tile_sums(0, dv.p, count, 0, 1, dt.p, nullptr);
        std::vector<double> tiles(tiles_of(count));
        BM_CUDA(cudaMemcpy(tiles.data(), dt.p, tiles.size() * sizeof(double), cudaMemcpyDeviceToHost));
        double total = 0.0;
        for (double t : tiles) total += t;
        *out = total;
    });
}

bm_status bm_update_centroids(const bm_dataset* dc, const int32_t* labels, uint64_t k, double* C, uint8_t* mask) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        for (uint64_t i = 0; i < d->m; ++i)
            if (labels[i] < 0 || (uint64_t)labels[i] >= k) throw ConfigError("update_centroids: label out of range");
        DeviceGuard g(d->device);
        Workspace& w = get_ws(d, d->m, (int)k, 1, 0);
        cudaStream_t st = stream_of(d);
        BM_CUDA(cudaMemcpyAsync(w.labels.p, labels, d->m * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        launch_update(st, dataset_points(d), w, nullptr, nullptr);
        BM_CUDA(cudaMemcpyAsync(C, w.C.p, k * d->n * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(mask, w.mask.p, k, cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
    });
}

bm_status bm_kmeanspp_fill(const bm_dataset* dc, double* C, uint8_t* mask, uint64_t k, int32_t candidates,
                           bm_rng* rng, uint64_t* evals) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        if (candidates < 1) throw ConfigError("kmeanspp_fill: candidates_per_step must be at least 1");
        DeviceGuard g(d->device);
        Workspace& w = get_ws(d, d->m, (int)k, candidates, 0);
        upload_centroids(stream_of(d), w, C, mask);
        std::vector<uint8_t> hmask(mask, mask + k);
        uint64_t ev = 0;
        kmeanspp_fill_device(stream_of(d), dataset_points(d), w, hmask, candidates, rng->eng, ev);
        BM_CUDA(cudaMemcpyAsync(C, w.C.p, k * d->n * sizeof(double), cudaMemcpyDeviceToHost, stream_of(d)));
        BM_CUDA(cudaMemcpyAsync(mask, w.mask.p, k, cudaMemcpyDeviceToHost, stream_of(d)));
        BM_CUDA(cudaStreamSynchronize(stream_of(d)));
        if (evals) *evals += ev;
    });
}

bm_status bm_lloyd(const bm_dataset* dc, double* C, uint8_t* mask, uint64_t k, uint64_t max_iterations,
                   double rel_tolerance, int32_t* labels, double* history, uint64_t history_capacity,
                   uint64_t* history_len, double* objective, uint64_t* evals, uint64_t* iterations) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        if (max_iterations < 1) throw ConfigError("lloyd: max_iterations must be at least 1");
        if (rel_tolerance < 0.0) throw ConfigError("lloyd: rel_tolerance must be nonnegative");
        DeviceGuard g(d->device);
        Workspace& w = get_ws(d, d->m, (int)k, 1, max_iterations + 1);
        cudaStream_t st = stream_of(d);
        upload_centroids(st, w, C, mask);
        LloydResult r = lloyd_run(st, dataset_points(d), w, max_iterations, rel_tolerance);
        const uint64_t hl = r.iterations + 1;
        std::vector<double> h(hl);
        BM_CUDA(cudaMemcpyAsync(h.data(), w.history.p, hl * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(C, w.C.p, k * d->n * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(mask, w.mask.p, k, cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(labels, w.labels.p + (uint64_t)r.parity * w.R, d->m * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < hl && i < history_capacity; ++i) history[i] = h[i];
        if (history_len) *history_len = hl;
        *objective = r.objective;
        *evals = r.evals;
        *iterations = r.iterations;
    });
}

bm_status bm_choose_chunk_size_hint(bm_dataset* data, uint64_t k, const uint64_t* ladder, uint64_t ladder_len,
                                    uint64_t chunks_per_candidate, uint64_t runs_per_candidate,
                                    uint64_t max_iterations, double rel_tolerance, int32_t candidates_per_step,
                                    uint64_t seed, uint64_t* chunk_size, double* best_mean) {
    return guarded([&] {
        std::vector<uint64_t> l(ladder, ladder + (ladder ? ladder_len : 0));
        *chunk_size = choose_chunk_size_hint(data, k, l, chunks_per_candidate, runs_per_candidate, max_iterations,
                                             rel_tolerance, candidates_per_step, seed, best_mean);
    });
}

bm_status bm_kmeans(const bm_dataset* data, uint64_t k, const bm_init_config* init, uint64_t max_iterations,
                    double rel_tolerance, bm_outcome* out) {
    return guarded([&] { kmeans(data, k, *init, max_iterations, rel_tolerance, out); });
}

bm_status bm_init_centroids(const bm_dataset* dc, uint64_t k, const bm_init_config* init, double* centroids,
                            uint8_t* mask, uint64_t* evals) {
    return guarded([&] {
        DeviceGuard g(dc->device);
        cudaStream_t st = stream_of(dc);
        Workspace& w = get_ws(dc, dc->m, (int)k, std::max(1, init->candidates_per_step), 0);
        const uint64_t e = init_stage(st, dc, w, k, *init);
        BM_CUDA(cudaMemcpyAsync(centroids, w.C.p, k * dc->n * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(mask, w.mask.p, k, cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        if (evals) *evals = e;
    });
}

bm_status bm_kmeans_pp(const bm_dataset* dc, uint64_t k, int32_t candidates, uint64_t seed,
                       uint64_t max_iterations, double rel_tolerance, bm_outcome* out) {
    return guarded([&] {
        bm_dataset* d = const_cast<bm_dataset*>(dc);
        if (k < 1) throw ConfigError("kmeans: k must be at least 1");
        if (d->m < k) throw ConfigError("kmeans: dataset has fewer points than clusters");
        if (max_iterations < 1) throw ConfigError("lloyd: max_iterations must be at least 1");
        if (rel_tolerance < 0.0) throw ConfigError("lloyd: rel_tolerance must be nonnegative");
        DeviceGuard g(d->device);
        cudaStream_t st = stream_of(d);
        Workspace& w = get_ws(d, d->m, (int)k, candidates, 0);
        Mt64 rng(seed);  // local_search.cpp:69
        const auto t_init = std::chrono::steady_clock::now();
        BM_CUDA(cudaMemsetAsync(w.C.p, 0, k * d->n * sizeof(double), st));
        BM_CUDA(cudaMemsetAsync(w.mask.p, 1, k, st));
        std::vector<uint8_t> hmask(k, 1);
        uint64_t init_evals = 0;
        Points P = dataset_points(d);
        kmeanspp_fill_device(st, P, w, hmask, candidates, rng, init_evals);
        BM_CUDA(cudaStreamSynchronize(st));
        out->cpu_init = seconds_since(t_init);
        const auto t_search = std::chrono::steady_clock::now();
        LloydResult r = lloyd_run(st, P, w, max_iterations, rel_tolerance);
        BM_CUDA(cudaMemcpyAsync(out->centroids, w.C.p, k * d->n * sizeof(double), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaMemcpyAsync(out->mask, w.mask.p, k, cudaMemcpyDeviceToHost, st));
        if (out->labels)
            BM_CUDA(cudaMemcpyAsync(out->labels, w.labels.p + (uint64_t)r.parity * w.R, d->m * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        out->cpu_full = seconds_since(t_search);
        out->objective = r.objective;
        out->distance_evals = r.evals + init_evals;
        out->iterations = r.iterations;
        out->chunks = 1;
    });
}

bm_status bm_big_means(bm_dataset* d, const bm_config* cfg, bm_outcome* out, bm_chunk_record* trace,
                       uint64_t trace_capacity) {
    return guarded([&] { big_means(d, *cfg, out, trace, trace_capacity); });
}

bm_status bm_big_means_multi(bm_dataset* const* data, int32_t chains, const bm_config* cfg, bm_outcome* out,
                             bm_chunk_record* trace, uint64_t trace_capacity, uint64_t* chain_chunks,
                             int32_t* winner) {
    return guarded([&] { big_means_multi(data, chains, *cfg, out, trace, trace_capacity, chain_chunks, winner); });
}

bm_status bm_last_trace(bm_chunk_record* out, uint64_t capacity, uint64_t* count) {
    return guarded([&] {
        if (count) *count = g_last_trace.size();
        if (out)
            std::copy(g_last_trace.begin(), g_last_trace.begin() + std::min<uint64_t>(capacity, g_last_trace.size()),
                      out);
    });
}

// Debug: k_wide_screen's per-atom stamps (BM_WIDE_DBG=1, -DBM_WIDE_DBG build).
extern "C" bm_status bm_debug_wide_stamps(uint64_t* out) {
    return bm::guarded([&] {
        unsigned long long* p = bm::wide_dbg_buffer();
        if (!p) throw bm::ConfigError("set BM_WIDE_DBG=1");
        BM_CUDA(cudaDeviceSynchronize());
        BM_CUDA(cudaMemcpy(out, p, 4 * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    });
}

// Debug: the chunk kernel's phase stamps ([4][8][16] globaltimer values; BM_CHUNK_DBG=1).
bm_status bm_debug_chunk_phases(uint64_t* out) {
    return guarded([&] {
        unsigned long long* p = chunk_dbg_buffer();
        if (!p) throw ConfigError("set BM_CHUNK_DBG=1");
        BM_CUDA(cudaMemcpy(out, p, 4 * 8 * 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    });
}

// Debug: per-CTA phase timestamps of the screened assignment (-DBM_KTRACE builds only).
bm_status bm_debug_ktrace(uint64_t* out, uint64_t count) {
    return guarded([&] {
#ifdef BM_KTRACE
        BM_CUDA(cudaMemcpyFromSymbol(out, dev::g_ktrace, std::min<uint64_t>(count, 1u << 20) * sizeof(uint64_t)));
#else
        (void)out;
        (void)count;
        throw ConfigError("library built without -DBM_KTRACE");
#endif
    });
}

bm_status bm_set_profiling(int enabled) {
    g_profiling = enabled != 0;
    return BM_OK;
}

bm_status bm_last_profile(bm_profile* out) {
    *out = g_profile;
    return BM_OK;
}

}  // extern "C"
