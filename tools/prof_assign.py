"""Short driver for ncu: a few c2 chunks + the final pass (not a benchmark)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
key = sys.argv[1] if len(sys.argv) > 1 else "c2"
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = synthetic.CONFIGS[key]
X = synthetic.generate(key)
d = bm.Dataset(X)
out, tr = bm.big_means(d, bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=chunks, seed=w.seed),
                       want_labels=False)
print(key, out.objective, tr.chunks(), out.counter.distance_evals)
