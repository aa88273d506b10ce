"""Device half of the ingestion path: bm_dataset_load = native parse + upload
(+ min-max normalisation on the device, io.cpp:245-264), bitwise against the
reference's io::load with the same DatasetSpec, and a big_means run on the
loaded dataset equal to the reference run on the reference-loaded matrix."""
import numpy as np
import pytest

import paper_2204_07485_b200 as bm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("normalize", [False, True])
@pytest.mark.parametrize("fmt", ["csv", "whitespace"])
def test_load_to_device_matches_reference(refo, tmp_path, normalize, fmt):
    rng = np.random.default_rng(8)
    X = rng.normal(size=(20_000, 9)) * rng.uniform(0.01, 100, (1, 9)) + rng.uniform(-50, 50, (1, 9))
    X[:, 4] = 3.0  # a constant column: normalises to 0.0
    p = tmp_path / ("d.csv" if fmt == "csv" else "d.txt")
    np.savetxt(p, X, delimiter="," if fmt == "csv" else " ", fmt="%.17g", header="h" * 3, comments="")
    d = bm.load(p, format=fmt, has_header=True, normalize=normalize, columns=[0, 4, 2, 8, 1])
    r = refo.io_load(p, format=fmt, has_header=True, normalize=normalize, columns=[0, 4, 2, 8, 1])
    assert r[0] == "ok"
    got = d.values()
    assert got.shape == r[1].shape and (got.view(np.uint64) == r[1].view(np.uint64)).all()


def test_load_then_big_means_matches_reference(refo, tmp_path):
    rng = np.random.default_rng(9)
    X = np.rint(rng.normal(size=(12_000, 5)) * 20)
    p = tmp_path / "i.csv"
    np.savetxt(p, X, delimiter=",", fmt="%.17g")
    d = bm.load(p, normalize=True)
    cfg = bm.BigMeansConfig(k=8, chunk_size=1_500, max_chunks=6, seed=4)
    out, trace = bm.big_means(d, cfg)
    Xr = refo.io_load(p, normalize=True)[1]
    r = refo.big_means(Xr, 8, 1_500, 6, seed=4)
    assert out.objective == r.objective
    assert [(t.chunk_index, t.candidate_objective, t.incumbent_objective, t.accepted, t.degenerate_repaired)
            for t in trace.records] == r.trace
