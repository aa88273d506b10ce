"""Full-size parity: BASELINE configs at their full m, s and chunk count,
bitwise against the unmodified reference (oracle/_ref, built from the
reference sources with its own Release flags) — objective, centroid bits,
mask, final labels, the whole trace, n_d and iterations.  c1 and c5 fit the
GPU-test budget (the reference takes ~1 s and ~1 min on the box's cores);
bench.py --config cN runs the same comparison for every config
(`parity_full_size` in its JSON line)."""
import os

import numpy as np
import pytest

import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic

from conftest import bits

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("key", ["c1", "c5"])
def test_config_full_size_bitwise_vs_reference(refo, key):
    w = synthetic.CONFIGS[key]
    X = synthetic.generate(key)
    cfg = bm.BigMeansConfig(k=w.k, chunk_size=w.s, max_chunks=w.chunks, seed=w.seed,
                            search=bm.SearchConfig(w.max_iterations, w.rel_tolerance),
                            init=bm.InitConfig(w.candidates))
    out, trace = bm.big_means(bm.Dataset(X), cfg)
    refo.set_worker_count(os.cpu_count() or 1)
    r = refo.big_means(np.ascontiguousarray(X, np.float64), w.k, w.s, w.chunks, seed=w.seed,
                       max_iterations=w.max_iterations, rel_tolerance=w.rel_tolerance,
                       candidates_per_step=w.candidates)
    got = [(t.chunk_index, t.candidate_objective, t.incumbent_objective, t.accepted,
            t.degenerate_repaired) for t in trace.records]
    assert len(got) == w.chunks
    assert got == r.trace
    assert out.objective == r.objective
    assert (bits(out.centroids.values) == bits(r.centroids)).all()
    assert (out.centroids.mask == r.mask).all()
    assert (out.assignment == r.labels).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (r.evals, r.iterations)
