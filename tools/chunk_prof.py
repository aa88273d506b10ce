"""Per-chunk kernel time of the persistent chunk kernel (globaltimer stamps)
and the graph timeline, for one config: python tools/chunk_prof.py c2 [chunks]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_07485_b200 as bm  # noqa: E402
from paper_2204_07485_b200 import synthetic  # noqa: E402

key = sys.argv[1]
w = synthetic.CONFIGS[key]
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else w.chunks
X = synthetic.generate(key)
d = bm.Dataset(X)
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=chunks, seed=w.seed)
import time
for rep in range(3):
    t0 = time.perf_counter()
    out, tr = bm.big_means(d, cfg, want_labels=False)
    wall = time.perf_counter() - t0
    p = bm.last_profile()
    n = max(p["chunk_launches"], 1)
    print(f"{key} rep{rep}: wall {wall*1e3:.2f} ms, cpu_init {out.counter.cpu_init*1e3:.2f} ms, final {out.counter.cpu_full*1e3:.2f} ms, "
          f"chunk kernels {p['chunk_launches']} avg {p['chunk_ms_total']/n*1e3:.1f} us, gap avg {p['chunk_gap_ms_total']/max(n-1,1)*1e3:.1f} us, "
          f"assign passes/chunk {p['chunk_assign_passes']/n:.2f}, iters {out.counter.iterations}", flush=True)

if os.environ.get("BM_CHUNK_DBG"):
    import ctypes as C
    import numpy as np
    from paper_2204_07485_b200 import _capi
    buf = np.zeros(4 * 8 * 16, np.uint64)
    _capi.load().bm_debug_chunk_phases(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
    buf = buf.reshape(4, 8, 16).astype(np.int64)
    names = ["start", "cent", "screen", "recheck", "fold", "barA", "ctl", "merge", "barB"]
    for c in range(4):
        t0 = buf[c, 0, 0]
        if t0 == 0:
            continue
        print(f"chunk%4={c}")
        for r in range(7):
            row = buf[c, r]
            if row[0] == 0:
                continue
            segs = [f"{names[i]}->{names[i+1]} {(row[i+1]-row[i])/1e3:.1f}" for i in range(8) if row[i + 1] >= row[i] > 0]
            if row[10] and row[11] and row[15]:  # inside load_centroids
                segs.append(f"[cent: sums {(row[10]-row[0])/1e3:.1f} active {(row[11]-row[10])/1e3:.1f} "
                            + (f"copy {(row[13]-row[11])/1e3:.1f} norms {(row[15]-row[13])/1e3:.1f}]" if row[13] > row[11]
                               else f"copy+norms {(row[15]-row[11])/1e3:.1f}]"))
            if row[14] > row[12] > 0:
                segs.append(f"[fold loops {(row[14]-row[12])/1e3:.1f} rest {(row[4]-row[14])/1e3:.1f}]")
            if row[15] > row[0] > 0:
                segs.append(f"[cent-load {(row[15]-row[0])/1e3:.1f}]")
            if row[12] > row[3] > 0:
                segs.append(f"[sort {(row[12]-row[3])/1e3:.1f} fold {(row[4]-row[12])/1e3:.1f}]")
            print(f"  r{r} @{(row[0]-t0)/1e3:.1f}us: " + " | ".join(segs))
        tail = buf[c, 7]
        print(f"  prologue {(buf[c,0,0]-tail[13])/1e3:.1f} us (rows landed at {(buf[c,0,13]-tail[13])/1e3:.1f}); max MMA dot error / (|x||c|) "
              f"{np.array([tail[14] & 0xFFFFFFFF], np.uint32).view(np.float32)[0]:.3g}")
        if tail[10] and tail[11]:
            print(f"  tail: loop-end @{(tail[9]-t0)/1e3:.1f} fold {(tail[10]-tail[9])/1e3:.1f} bar {(tail[11]-tail[10])/1e3:.1f} accept {(tail[12]-tail[11])/1e3:.1f}")
        else:
            print(f"  tail: loop-end @{(tail[9]-t0)/1e3:.1f}, accept + record + next start {(tail[12]-tail[9])/1e3:.1f} (exact objective deferred)")
