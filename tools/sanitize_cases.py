"""Small big_means runs for compute-sanitizer (memcheck / racecheck / synccheck):
every chunk-engine path once, each checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2204_07485_b200 as bm  # noqa: E402
from oracle.oracle import port  # noqa: E402
from paper_2204_07485_b200 import synthetic  # noqa: E402

P = port()
rng = np.random.default_rng(3)
cases = {
    # persistent chunk kernel, tensor-core screen (integer rows: exact in tf32), exact-sum mode
    "c2_small_tc": (synthetic.generate("c2", 40_000), 25, 1_500, 4),
    # persistent chunk kernel, packed-FFMA screen, fp32 rows, ordered mode
    "c3_small_ffma": (synthetic.generate("c3", 60_000), 20, 3_000, 4),
    # persistent chunk kernel, fp64 rows
    "c1_small_f64": (synthetic.generate("c1", 20_000), 10, 2_500, 4),
    # multi-launch chunk graphs (rows wider than the chunk kernel's instances)
    "wide_rows": (rng.normal(size=(3_000, 120)), 6, 700, 3),
    # mid-run K-means++ repairs (emptied clusters)
    "repairs": (np.rint(rng.normal(size=(3_000, 3))), 16, 40, 12),
}
only = sys.argv[1:] or list(cases)
for name in only:
    X, k, s, ch = cases[name]
    out, trace = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=ch, seed=7))
    p = P.big_means(np.asarray(X, np.float64), k, s, ch, seed=7)
    ok = out.objective == p.objective and [r.candidate_objective for r in trace.records] == [t[1] for t in p.trace]
    print(f"{name}: {'bitwise ok' if ok else 'MISMATCH'} objective {out.objective!r}", flush=True)
    assert ok
