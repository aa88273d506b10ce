import sys; sys.path.insert(0, '.')
import numpy as np, time
import paper_2204_07485_b200 as bm
X = np.rint(np.random.default_rng(5).normal(size=(20000, 16)) * 4)
t = time.time()
o, tr = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=10, chunk_size=3000, max_chunks=12, seed=3))
print("ok", o.objective, len(tr.records), time.time() - t)
