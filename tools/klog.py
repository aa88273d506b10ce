"""Kernel log of the Lloyd graphs (debug tool; library built with -DBM_KTRACE
via `python tools/ktrace.py --build`): per kernel kind, in-graph durations and
the gaps between consecutive kernels of the chain loop.

  python tools/klog.py [chunks]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_07485_b200 import _capi  # noqa: E402
_capi.LIB_PATH = os.path.join(ROOT, "tools", "_ktrace", "libbigmeans_b200.so")
import paper_2204_07485_b200 as bm  # noqa: E402
from paper_2204_07485_b200 import synthetic  # noqa: E402

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 60
KEY = os.environ.get("KLOG_CONFIG", "c2")
w = synthetic.CONFIGS[KEY]
d = bm.Dataset(synthetic.generate(KEY))
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=chunks, seed=0)
bm.big_means(d, cfg, want_labels=False)
buf = np.zeros(540000, np.uint64)
lib = _capi.load()
lib.bm_debug_ktrace(buf.ctypes.data_as(_capi.P_u64), buf.size)
n0 = int(buf[200000])
st0 = buf[199990:199994].astype(np.int64)
bm.big_means(d, cfg, want_labels=False)
lib.bm_debug_ktrace(buf.ctypes.data_as(_capi.P_u64), buf.size)
n1 = int(buf[200000])
st1 = buf[199990:199994].astype(np.int64)
E = buf[200001:200001 + 3 * 60000].reshape(-1, 3).astype(np.int64)[n0 % 60000:n1 % 60000]
names = {0: "guard", 1: "centroids", 2: "update", 21: "begin(exit)", 22: "round(exit)", 3: "accept", 10: "assign(h0)", 11: "assign(begin)", 12: "assign(round)",
         4: "accept:folded", 5: "accept:objective", 6: "accept:record", 7: "accept:ranks"}
sub = E[(E[:, 0] >= 4) & (E[:, 0] <= 7)]
E = E[(E[:, 0] < 4) | (E[:, 0] > 7)]
acc = E[E[:, 0] == 3]
for kid in range(4, 8):  # sub-phase marks: end time relative to the enclosing accept's start
    ends = sub[sub[:, 0] == kid, 2]
    offs = [t - acc[(acc[:, 1] <= t) & (acc[:, 2] >= t), 1][0] for t in ends
            if ((acc[:, 1] <= t) & (acc[:, 2] >= t)).any()]
    if offs:
        print(f"  {names[kid]:18s} at {np.mean(offs) / 1e3:7.2f} us after the accept's start")
E = E[np.argsort(E[:, 1])]
print(f"{len(E)} kernels over {chunks} chunks; span {(E[-1, 2] - E[0, 1]) / 1e3:.1f} us "
      f"({(E[-1, 2] - E[0, 1]) / 1e3 / chunks:.1f} us per chunk)")
dur = {}
for kid, a, b in E:
    dur.setdefault(int(kid), []).append(b - a)
busy = 0
for kid in sorted(dur):
    v = np.array(dur[kid]) / 1e3
    busy += v.sum()
    print(f"{names.get(kid, kid):14s} n={len(v):5d} mean={v.mean():7.2f} p50={np.median(v):7.2f} "
          f"p90={np.percentile(v, 90):7.2f} us  total/chunk={v.sum() / chunks:7.2f} us")
gaps = (E[1:, 1] - E[:-1, 2]) / 1e3
print(f"kernel busy {busy / chunks:.1f} us per chunk; gaps between consecutive kernels: mean {gaps.mean():.2f} "
      f"p50 {np.median(gaps):.2f} p90 {np.percentile(gaps, 90):.2f} us, {gaps.sum() / chunks:.1f} us per chunk")
pairs = {}
for i in range(1, len(E)):
    key = (names.get(int(E[i - 1, 0])), names.get(int(E[i, 0])))
    pairs.setdefault(key, []).append((E[i, 1] - E[i - 1, 2]) / 1e3)
for key, v in sorted(pairs.items(), key=lambda kv: -sum(kv[1])):
    print(f"  gap {key[0]:>14s} -> {key[1]:14s} n={len(v):5d} mean={np.mean(v):6.2f} us")
ds = st1 - st0
print(f"round fast path: {ds[0]} CTAs, {ds[1]} fell back to the screen ({100 * ds[1] / max(ds[0], 1):.1f}%), "
      f"{ds[2] / max(ds[0], 1):.2f} rechecked pairs and {ds[3] / max(ds[0], 1):.2f} points with rechecks per CTA")

# per-CTA phase marks of the last begin (region 400000) and round (region 470000) launches
names_k = {14: "probe1", 0: "start", 1: "slab0", 2: "slab1", 3: "slab2", 4: "slab3", 5: "slab4", 6: "slab5", 7: "bounds",
           8: "items", 9: "recheck", 10: "out/fold", 13: "fp_setup", 15: "fp_done", 16: "c0wait", 17: "c0done",
           24: "c4wait", 25: "c4done", 26: "fp_items", 11: "acc:record", 12: "acc:ranks", 27: "lbk_written", 28: "last:arrived", 29: "last:control",
           30: "last:accept", 31: "sums_done", 18: "s:moved", 19: "s:aggregated", 20: "s:slot_fenced"}
for base, title in ((400000, "begin"), (470000, "round")):
    T = buf[base:base + 2048 * 32].reshape(-1, 32).astype(np.int64)
    T = T[T[:, 0] > 0]
    if not len(T):
        continue
    t0 = T[:, 0].min()
    print(f"--- last {title} launch: {len(T)} CTAs")
    for i in sorted(names_k):
        col = T[:, i]
        v = col[col > 0] - t0
        if v.size:
            print(f"  {names_k[i]:13s} n={v.size:5d} p10={np.percentile(v, 10) / 1e3:7.2f} p50={np.percentile(v, 50) / 1e3:7.2f} "
                  f"p90={np.percentile(v, 90) / 1e3:7.2f} max={v.max() / 1e3:7.2f} us")

# raw sequence of the last logged kernels (start / end, us from the first shown)
if os.environ.get("KLOG_RAW"):
    R = E[-int(os.environ["KLOG_RAW"]):]
    t0 = R[0, 1]
    for kid, a, b in R:
        print(f"  raw {names.get(int(kid), kid):14s} {(a - t0) / 1e3:9.2f} {(b - t0) / 1e3:9.2f}")
