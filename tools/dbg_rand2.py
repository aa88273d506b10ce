import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2204_07485_b200 as bm
from oracle.oracle import port
P = port()
for seed in [int(x) for x in os.environ.get("SEEDS", "2,5,8,11").split(",")]:
    rng = np.random.default_rng(500 + seed)
    m = int(rng.integers(300, 20000)); n = int(rng.integers(1, 40)); k = int(rng.integers(1, 30))
    s = int(rng.integers(k, min(m, 5000) + 1))
    X = (rng.normal(size=(m, n)) * rng.uniform(0.1, 30)).astype(np.float32)
    for rep in range(2):
        out, trace = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=8, seed=seed))
        p = P.big_means(X.astype(np.float64), k, s, 8, seed=seed)
        got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted, r.degenerate_repaired) for r in trace.records]
        print(seed, m, n, k, s, "ok" if got == p.trace else "MISMATCH", got[0][1], p.trace[0][1], flush=True)
    if os.environ.get("BM_CHUNK_DBG") == "2":
        import ctypes as C
        from paper_2204_07485_b200 import _capi
        buf = np.zeros(4 * 8 * 16, np.uint64)
        _capi.load().bm_debug_chunk_phases(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
        b = buf.reshape(4, 8, 16)
        print("  max mma err", [float(np.array([b[c, 7, 14] & 0xFFFFFFFF], np.uint32).view(np.float32)[0]) for c in range(4)])
if os.environ.get("BM_CHUNK_DBG") == "2":
    b = buf.reshape(4, 8, 16)
    for c in range(4):
        r = b[c, 6]
        if r[0]:
            print("first bad: p", r[1], "j", r[2], "round", r[3], "tc", np.array([r[4]], np.uint64).view(np.float64)[0],
                  "exact", np.array([r[5]], np.uint64).view(np.float64)[0], "KA", r[6], "np", r[7])
    print("bad per tile (round 0, all chunks):", b[0, 5, :8].tolist(), "per row&7:", b[0, 5, 8:16].tolist())
