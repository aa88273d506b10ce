"""Per-CTA phase timeline of the screened assignment kernel (debug tool).

  python tools/ktrace.py --build        # builds tools/_ktrace/libbigmeans_b200.so with -DBM_KTRACE
  python tools/ktrace.py [m] [n] [k]    # one assign_nearest launch, prints phase percentiles (us)
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "_ktrace", "libbigmeans_b200.so")

if "--build" in sys.argv:
    from paper_2204_07485_b200 import build as b
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run([b.NVCC, *b.FLAGS, "-DBM_KTRACE", "-o", LIB, *b.SOURCES], check=True)
    sys.exit(0)

from paper_2204_07485_b200 import _capi  # noqa: E402
_capi.LIB_PATH = LIB
import paper_2204_07485_b200 as bm  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 68
k = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rng = np.random.default_rng(0)
X = np.rint(rng.normal(size=(m, n)) * 5 + rng.integers(0, 20, (m, 1)))
C0 = X[rng.choice(m, k, replace=False)] + 0.3
d = bm.Dataset(X)
cent = bm.Centroids(C0, np.zeros(k, np.uint8))
for _ in range(3):
    bm.assign_nearest(d, cent)
buf = np.zeros(2048 * 16, np.uint64)
lib = _capi.load()
assert lib.bm_debug_ktrace(buf.ctypes.data_as(_capi.P_u64), buf.size) == 0
ctas = (m + 127) // 128
T = buf[: min(ctas, 2048) * 16].reshape(-1, 16).astype(np.int64)
t0 = T[:, 0].min()
names = ["start", "slab0", "slab1", "slab2", "slab3", "slab4", "slab5", "bounds", "items", "recheck",
         "out", "lastwait", "fold"]
print(f"m={m} n={n} k={k} ctas={ctas}")
for i, nm in enumerate(names):
    col = T[:, i]
    v = col[col > 0] - t0
    if v.size:
        print(f"{nm:9s} n={v.size:5d}  p10={np.percentile(v,10)/1e3:8.2f}  p50={np.percentile(v,50)/1e3:8.2f}  "
              f"p90={np.percentile(v,90)/1e3:8.2f}  max={v.max()/1e3:8.2f} us")
