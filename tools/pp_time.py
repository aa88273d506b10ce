"""Time kmeanspp_fill (all-degenerate, k=25, 3 candidates) on a c2-like 50k chunk."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
X = synthetic.generate("c2", 50000)
d = bm.Dataset(X)
for rep in range(3):
    t = time.perf_counter()
    c = bm.kmeanspp_fill(d, bm.Centroids.all_degenerate(25, X.shape[1]), bm.InitConfig(), bm.Rng(1))
    print(f"{os.environ.get('BM_PP', 'device')}: {1e3 * (time.perf_counter() - t):.2f} ms")
