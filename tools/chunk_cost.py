"""Per-chunk cost on c2 from the difference of two chunk budgets (device-resident, median of runs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
w = synthetic.CONFIGS["c2"]
d = bm.Dataset(synthetic.generate("c2"))
res = {}
for chunks in (20, 120, 220):
    cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=chunks, seed=w.seed)
    ts = []
    for i in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        bm.big_means(d, cfg, want_labels=False)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    res[chunks] = float(np.median(ts[1:]))
    print(f"{chunks} chunks: {res[chunks]:.2f} ms")
print(f"per chunk (120->220): {1e3 * (res[220] - res[120]) / 100:.1f} us; fixed part: {res[20] - 20 * (res[220] - res[120]) / 100:.2f} ms")
