"""Screen candidates per point of one config's big_means (profiling pass): python tools/cand_stats.py c5 [chunks]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_07485_b200 as bm  # noqa: E402
from paper_2204_07485_b200 import synthetic  # noqa: E402

key = sys.argv[1]
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = synthetic.CONFIGS[key]
X = synthetic.generate(key)
d = bm.Dataset(X)
cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=chunks, seed=w.seed)
for wide in ("1", "0"):
    os.environ["BM_WIDE"] = wide
    bm.set_profiling(True)
    out, tr = bm.big_means(d, cfg, want_labels=False)
    bm.set_profiling(False)
    p = bm.last_profile()
    print(f"{key} BM_WIDE={wide}: candidates/point {p['screen_candidates'] / max(p['screen_rows'], 1):.3f} "
          f"(rows {p['screen_rows']}), assign ms {p['phase_ms']['assign']:.2f} over {p['phase_count']['assign']} launches",
          flush=True)
