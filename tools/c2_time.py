"""Device-resident c2 step time (ms, median of N runs after warm-up) — quick A/B of env toggles."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
w = synthetic.CONFIGS["c2"]
d = bm.Dataset(synthetic.generate("c2"))
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=w.chunks, seed=w.seed)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ts = []
for i in range(n + 2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out, tr = bm.big_means(d, cfg, want_labels=False)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t))
ts = np.array(ts[2:])
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("BM_"))
print(f"[{tag or 'default'}] c2 ms/step median {np.median(ts):.2f} min {ts.min():.2f} max {ts.max():.2f} obj {out.objective!r}")
