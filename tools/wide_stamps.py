"""k_wide_screen per-atom timeline of CTA (0,0) (library built with -DBM_WIDE_DBG):
BM_WIDE_DBG=1 BM_LIB_PATH=... python tools/wide_stamps.py c5"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_07485_b200 as bm  # noqa: E402
from paper_2204_07485_b200 import _capi, synthetic  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = synthetic.CONFIGS[key]
d = bm.Dataset(synthetic.generate(key))
out, tr = bm.big_means(d, bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=3, seed=w.seed), want_labels=False)
buf = np.zeros(4 * 64, np.uint64)
lib = _capi.load()
lib.bm_debug_wide_stamps.argtypes = [C.POINTER(C.c_uint64)]
lib.bm_debug_wide_stamps(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
b = buf.reshape(4, 64).astype(np.int64)
t0 = b[0, 0]
print("atom  issued  landed  mma-issued  retired   (us from the first TMA issue)")
for t in range(64):
    if b[1, t] == 0:
        break
    print(f"{t:3d} " + " ".join(f"{(b[r, t] - t0) / 1e3:8.2f}" if b[r, t] else "       -" for r in range(4)))
