import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2204_07485_b200 as bm
from oracle.oracle import port
P = port()
os.environ["BM_TC"] = "1"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rng = np.random.default_rng(1000 + n)
m, k, s = 9000, 11, 2100
X = (rng.normal(size=(m, n)) * 5.0 + rng.integers(0, 3, (m, 1)) * 4.0).astype(np.float32)
Xi = X if os.environ.get('FLOATDATA') else np.rint(X)
if os.environ.get('FLOAT_FIRST'):
    bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=5, seed=n))
cfg = bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=5, seed=n)
p = P.big_means(np.asarray(Xi, np.float64), k, s, 5, seed=n)
for rep in range(3):
    out, trace = bm.big_means(bm.Dataset(Xi), cfg)
    got = [(r.chunk_index, r.candidate_objective, r.accepted) for r in trace.records]
    ok = got == [(t[0], t[1], t[3]) for t in p.trace]
    prof = bm.last_profile()
    print("rep", rep, "ok" if ok else "MISMATCH", got[:2], [(t[0], t[1], t[3]) for t in p.trace][:2], "chunk kernels", prof["chunk_launches"], flush=True)

if os.environ.get("BM_CHUNK_DBG") == "2":
    import ctypes as C
    from paper_2204_07485_b200 import _capi
    buf = np.zeros(4 * 8 * 16, np.uint64)
    _capi.load().bm_debug_chunk_phases(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
    buf = buf.reshape(4, 8, 16)
    print("bad counts by tile", buf[0, 5, :8], "by p&7", buf[0, 5, 8:])
    for c in range(4):
        sl = buf[c, 6]
        if sl[0]:
            print("chunk%4", c, "p", sl[1], "j", sl[2], "r", sl[3], "mma", sl[4:5].view(np.float64), "exact", sl[5:6].view(np.float64), "KA", sl[6], "np", sl[7], "row match", sl[8], "centroid match", sl[9], "next", np.array(sl[10:12], np.uint64).astype(np.uint32).view(np.float32))
        print("max err", np.array([buf[c, 7, 14] & 0xFFFFFFFF], np.uint32).view(np.float32))
    print("rows diag: bad", buf[2, 7, 15], "sample p,d", buf[1, 7, 1], buf[1, 7, 2], "got/want", buf[1, 7, 3:5].view(np.float64))
    print("B operand diag: bad", buf[3, 7, 15], "smem base etc")
    print("theory counts [neither, laneA only, sboB only, both]", buf[1, 5, :4])
