"""TC screen check across row widths: max MMA dot error (BM_CHUNK_DBG=2) and oracle parity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import _capi
from oracle.oracle import port
P = port()
for n in [int(x) for x in os.environ.get("NS", "3,6,8,12,16,20,24,28,32,36,40,68").split(",")]:
    buf = np.zeros(4 * 8 * 16, np.uint64)
    lib = _capi.load()
    rng = np.random.default_rng(n)
    m, k, s = 6000, 10, 1500
    X = (rng.normal(size=(m, n)) * 7.0).astype(np.float32)
    # reset the diagnostic slots by reading them (the device buffer persists; record deltas)
    lib.bm_debug_chunk_phases(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
    before = buf.reshape(4, 8, 16)[0, 5, :8].sum()
    out, trace = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=4, seed=1))
    p = P.big_means(X.astype(np.float64), k, s, 4, seed=1)
    got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted, r.degenerate_repaired) for r in trace.records]
    lib.bm_debug_chunk_phases(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
    b = buf.reshape(4, 8, 16)
    print(n, "ok" if got == p.trace else "MISMATCH", "bad dots (round 0)", int(b[0, 5, :8].sum() - before), flush=True)
