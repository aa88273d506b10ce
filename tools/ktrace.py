"""Per-CTA phase timeline of the screened assignment kernel (debug tool).

  python tools/ktrace.py --build        # builds tools/_ktrace/libbigmeans_b200.so with -DBM_KTRACE
  python tools/ktrace.py [m] [n] [k]    # one assign_nearest launch, prints phase percentiles (us)
  python tools/ktrace.py lloyd [m] [n] [k]  # the last launch of a 1-round Lloyd (bound fast path)
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

args = [a for a in sys.argv[1:] if a != "lloyd"]
lloyd_mode = "lloyd" in sys.argv
m = int(args[0]) if len(args) > 0 else 50_000
n = int(args[1]) if len(args) > 1 else 68
k = int(args[2]) if len(args) > 2 else 25
rng = np.random.default_rng(0)
X = np.rint(rng.normal(size=(m, n)) * 5 + rng.integers(0, 20, (m, 1)))
C0 = X[rng.choice(m, k, replace=False)] + 0.3
if lloyd_mode:  # a c2-like chunk started from centroids converged on another chunk
    from paper_2204_07485_b200 import synthetic
    full = synthetic.generate("c2", 2 * m)
    X, n = full[m:], full.shape[1]
    warm = bm.lloyd(bm.Dataset(full[:m]), bm.Centroids(full[:k].astype(np.float64), np.zeros(k, np.uint8)))
    C0 = warm.centroids.values
d = bm.Dataset(X)
cent = bm.Centroids(C0, np.zeros(k, np.uint8))
for _ in range(3):
    if lloyd_mode:
        bm.lloyd(d, cent, bm.SearchConfig(max_iterations=1))
    else:
        bm.assign_nearest(d, cent)
buf = np.zeros(65536 + 2048 * 32, np.uint64)
lib = _capi.load()
assert lib.bm_debug_ktrace(buf.ctypes.data_as(_capi.P_u64), buf.size) == 0
ctas = (m + 127) // 128
T = buf[: min(ctas, 2048) * 32].reshape(-1, 32).astype(np.int64)
t0 = T[:, 0].min()
names = ["start", "slab0", "slab1", "slab2", "slab3", "slab4", "slab5", "bounds", "items", "recheck",
         "out", "lastwait", "fold", "fp_setup", "fp_own", "fp_fails"] + \
    [f"c{i//2}{'wait' if i % 2 == 0 else 'done'}" for i in range(10)] + ["fp_items"]
print(f"m={m} n={n} k={k} ctas={ctas}")
for i, nm in enumerate(names):
    col = T[:, i]
    v = col[col > 0] - t0
    if v.size:
        print(f"{nm:9s} n={v.size:5d}  p10={np.percentile(v,10)/1e3:8.2f}  p50={np.percentile(v,50)/1e3:8.2f}  "
              f"p90={np.percentile(v,90)/1e3:8.2f}  max={v.max()/1e3:8.2f} us")

if lloyd_mode:  # the last k_update launch (region 1)
    U = buf[65536:].reshape(-1, 32).astype(np.int64)
    U = U[U[:, 0] > 0]
    t0 = U[:, 0].min()
    print(f"k_update ctas={len(U)}")
    for i, nm in enumerate(["start", "staged", "bucketed", "prefix", "order", "folded", "merger", "totals",
                            "merged", "m0_copied", "m0_folded"]):
        col = U[:, i]
        v = col[col > 0] - t0
        if v.size:
            print(f"{nm:9s} n={v.size:5d}  p10={np.percentile(v,10)/1e3:8.2f}  p50={np.percentile(v,50)/1e3:8.2f}  "
                  f"p90={np.percentile(v,90)/1e3:8.2f}  max={v.max()/1e3:8.2f} us")
