import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
w = synthetic.CONFIGS["c2"]
X = synthetic.generate("c2")
d = bm.Dataset(X)
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=200, seed=0)
for i in range(3):
    o, t = bm.big_means(d, cfg, want_labels=False)
