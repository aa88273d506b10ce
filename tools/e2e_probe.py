"""Time the e2e pieces on c2: dataset create (pinned host f64), big_means, destroy."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
w = synthetic.CONFIGS["c2"]
X = synthetic.generate("c2")
Xp = torch.from_numpy(np.ascontiguousarray(X)).pin_memory().numpy()
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=w.chunks, seed=0)
for i in range(4):
    t0 = time.perf_counter()
    d = bm.Dataset(Xp)
    t1 = time.perf_counter()
    out, tr = bm.big_means(d, cfg, want_labels=True)
    t2 = time.perf_counter()
    d.close() if hasattr(d, "close") else d.__exit__(None, None, None)
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  big_means {1e3*(t2-t1):.1f} ms  destroy {1e3*(t3-t2):.1f} ms")
