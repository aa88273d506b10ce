"""GPU parity: sampling, K-means++ repair, Lloyd (init.cpp, local_search.cpp,
big_means.cpp:39-56) — reference test_init / test_local_search /
test_big_means cases plus bitwise agreement with golden vectors."""
import numpy as np
import pytest

import paper_2204_07485_b200 as bm
from conftest import bits

pytestmark = pytest.mark.gpu


def test_rng_stream_is_mt19937_64(golden):
    r = bm.Rng(7)
    assert [r() for _ in range(16)] == golden["rng_raw_seed7"].tolist()


def test_sample_chunk_golden(golden):
    for i, (m, s, seed) in enumerate(golden["sample_cases"].tolist()):
        d = bm.Dataset(np.zeros((m, 1)))
        r = bm.Rng(seed)
        assert (bm.sample_chunk(d, s, r) == golden[f"sample_{i}"]).all()
        assert r() == int(golden[f"sample_{i}_next"][0])


@pytest.mark.parametrize("m,s", [(1, 1), (2, 1), (10, 9), (33, 32), (1000, 1), (1000, 500),
                                 (4096, 4095), (13_500, 4_000), (100_000, 10_000),
                                 (2_500_000, 50_000), (10_500_000, 100_000)])
def test_sample_chunk_vs_oracle(port, m, s):
    d = bm.Dataset(np.zeros((m, 1), np.float32))
    for seed in (0, 1, 123456789):
        r = bm.Rng(seed)
        pr = port.rng(seed)
        for _ in range(2):  # consecutive chunks share the stream
            got = bm.sample_chunk(d, s, r)
            exp = port.sample_chunk(m, s, pr)
            assert (got == exp).all()
        assert r() == port.rng_next(pr)


@pytest.mark.parametrize("m,s", [(2, 1), (33, 32), (1000, 500), (4096, 4095), (13_500, 4_000),
                                 (100_000, 10_000), (2_500_000, 50_000), (10_500_000, 100_000)])
@pytest.mark.parametrize("force_seq", [False, True])
def test_device_stream_sample_chunk_vs_oracle(port, m, s, force_seq):
    """Draws made on the device (k_mt_twist, k_mt_emit, k_mt_fix) from the device-resident stream:
    same indices and same stream position as the reference's host draws."""
    if force_seq and s > 20_000:
        pytest.skip("sequential path is a single-thread fallback; small cases suffice")
    d = bm.Dataset(np.zeros((m, 1), np.float32))
    for seed in (0, 7, 123456789):
        r, pr = bm.Rng(seed), port.rng(seed)
        for _ in range(3):
            got = bm.sample_chunk_device(d, s, r, force_sequential=force_seq)
            assert (got == port.sample_chunk(m, s, pr)).all()
        assert r() == port.rng_next(pr)


def test_sample_chunk_properties():  # test_big_means.cpp:27-54
    d = bm.Dataset(np.random.default_rng(1).uniform(0, 50, (100, 2)))
    idx = bm.sample_chunk(d, 30, bm.Rng(7))
    assert idx.size == 30 and (np.diff(idx.astype(np.int64)) > 0).all() and idx[-1] < 100
    d64 = bm.Dataset(np.zeros((64, 2)))
    r, untouched = bm.Rng(9), bm.Rng(9)
    assert (bm.sample_chunk(d64, 64, r) == np.arange(64)).all()
    assert r() == untouched()


def test_kmeanspp_golden(golden):
    P = bm.Dataset(golden["pp_P"])
    c = bm.kmeanspp_fill(P, bm.Centroids.all_degenerate(6, 3), bm.InitConfig(), bm.Rng(5))
    assert (bits(c.values) == bits(golden["pp_all_C"])).all() and c.degenerate_count() == 0
    counter = bm.EvalCounter()
    c = bm.kmeanspp_fill(P, bm.Centroids(golden["pp_part_Cin"], golden["pp_part_maskin"]),
                         bm.InitConfig(), bm.Rng(6), counter)
    assert (bits(c.values) == bits(golden["pp_part_C"])).all()
    assert c.row(2).tolist() == [100.0, 100.0, 100.0]
    assert counter.distance_evals == int(golden["pp_part_evals"][0])
    c = bm.kmeanspp_fill(bm.Dataset(golden["pp_zero_P"]), bm.Centroids.all_degenerate(3, 2),
                         bm.InitConfig(), bm.Rng(8))
    assert (bits(c.values) == bits(golden["pp_zero_C"])).all()


def test_kmeanspp_seed_overload_matches_stream():  # test_init.cpp:85-92
    d = bm.Dataset(np.random.default_rng(5).uniform(-5, 5, (60, 3)))
    a = bm.kmeanspp_fill(d, bm.Centroids.all_degenerate(4, 3), bm.InitConfig(), bm.Rng(1234))
    b = bm.kmeanspp_fill(d, bm.Centroids.all_degenerate(4, 3), bm.InitConfig(), 1234)
    assert a == b


def test_kmeanspp_law():  # acceptance.cpp:268-293 (criterion 7), reduced trials
    d = bm.Dataset([0.0, 1.0, 10.0], 3, 1)
    start = bm.Centroids.all_degenerate(2, 1)
    start.set_row(0, [0.0])
    rng = bm.Rng(bm.K_DEFAULT_SEED)
    trials, far = 1000, 0
    for _ in range(trials):
        c = bm.kmeanspp_fill(d, start, bm.InitConfig(candidates_per_step=1), rng)
        far += c.row(1)[0] == 10.0
    assert abs(far / trials - 100 / 101) <= 0.02


@pytest.mark.parametrize("tag,tol", [("tol0", 0.0), ("tol5e2", 0.05), ("tol1e4", 1e-4)])
def test_lloyd_golden(golden, tag, tol):
    d = bm.Dataset(golden["lloyd_X"])
    acc = bm.EvalCounter()
    o = bm.lloyd(d, bm.Centroids.from_rows(golden["lloyd_start"]),
                 bm.SearchConfig(rel_tolerance=tol), acc)
    assert (bits(o.centroids.values) == bits(golden[f"lloyd_{tag}_C"])).all()
    assert (o.centroids.mask == golden[f"lloyd_{tag}_mask"]).all()
    assert (o.assignment == golden[f"lloyd_{tag}_labels"]).all()
    assert (bits(o.objective_history) == bits(golden[f"lloyd_{tag}_hist"])).all()
    assert [o.counter.distance_evals, o.counter.iterations] == golden[f"lloyd_{tag}_stats"].tolist()
    assert o.objective == o.objective_history[-1]
    assert acc.distance_evals == o.counter.distance_evals and acc.iterations == o.counter.iterations
    assert o.counter.iterations == len(o.objective_history) - 1  # test_local_search.cpp:25-44


def test_lloyd_fixed_point_and_zero_objective():  # test_local_search.cpp:60-79
    d = bm.Dataset([0.0, 0.0, 2.0, 0.0, 10.0, 0.0, 12.0, 0.0], 4, 2)
    o = bm.lloyd(d, bm.Centroids.from_rows([1.0, 0.0, 11.0, 0.0], 2, 2),
                 bm.SearchConfig(rel_tolerance=0.0))
    assert o.counter.iterations == 1 and len(o.objective_history) == 2
    assert o.objective == o.objective_history[0]
    d = bm.Dataset([1.0, 1.0, 5.0, 5.0], 2, 2)
    o = bm.lloyd(d, bm.Centroids.from_rows([1.0, 1.0, 5.0, 5.0], 2, 2))
    assert o.objective == 0.0 and o.counter.iterations <= 1


def test_lloyd_iteration_cap_and_empty_cluster(golden):  # test_local_search.cpp:81-116
    X = np.random.default_rng(5).uniform(0, 100, (1000, 2))
    o = bm.lloyd(bm.Dataset(X), bm.Centroids.from_rows(X[:20]),
                 bm.SearchConfig(max_iterations=2, rel_tolerance=0.0))
    assert o.counter.iterations <= 2
    d = bm.Dataset([0.0, 0.0, 1.0, 0.0, 10.0, 0.0, 11.0, 0.0], 4, 2)
    o = bm.lloyd(d, bm.Centroids.from_rows([0.0, 0.0, 10.0, 0.0, 1000.0, 1000.0], 3, 2))
    assert o.centroids.degenerate_count() == 1 and o.centroids.degenerate(2)
    assert o.objective == golden["lloyd_empty_obj"][0] == 1.0
    with pytest.raises(bm.ConfigError):
        bm.lloyd(d, bm.Centroids.from_rows([0.0, 0.0], 1, 2), bm.SearchConfig(max_iterations=0))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lloyd_vs_oracle_random(port, dtype):
    rng = np.random.default_rng(42)
    X = (rng.normal(size=(7000, 12)) * 5).astype(dtype)
    Xd = X.astype(np.float64)
    start = Xd[rng.choice(7000, 9, replace=False)]
    o = bm.lloyd(bm.Dataset(X), bm.Centroids.from_rows(start), bm.SearchConfig(rel_tolerance=0.0))
    p = port.lloyd(Xd, start, np.zeros(9, np.uint8), 300, 0.0)
    assert (bits(o.centroids.values) == bits(p["centroids"])).all()
    assert (o.assignment == p["labels"]).all()
    assert (bits(o.objective_history) == bits(p["history"])).all()


def _blobs(rng, m, n, k, spread):
    centers = rng.normal(size=(k, n)) * spread
    return centers[rng.integers(0, k, m)] + rng.normal(size=(m, n))


@pytest.mark.parametrize("case", ["ties", "blobs", "blobs_f32", "tight", "huge", "tiny"])
def test_lloyd_bound_fast_path_vs_oracle(port, case):
    """Lloyd rounds take the certified bound test (labels kept when every point
    beats its drifted lower bound); every regime must still match the oracle's
    bits: exact ties, well separated blobs (the fast path almost always holds),
    touching blobs, values outside fp32 range (no bounds) and tiny magnitudes."""
    rng = np.random.default_rng(11)
    if case == "ties":
        X = rng.integers(0, 4, (6000, 3)).astype(np.float64)
    elif case in ("blobs", "blobs_f32"):
        X = _blobs(rng, 20000, 20, 8, 20.0)
    elif case == "tight":
        X = _blobs(rng, 20000, 9, 12, 1.5)
    elif case == "huge":
        X = _blobs(rng, 5000, 6, 5, 10.0) * 1e30
    else:
        X = _blobs(rng, 5000, 6, 5, 10.0) * 1e-30
    if case == "blobs_f32":
        X = X.astype(np.float32)
    Xd = X.astype(np.float64)
    k = 7 if case == "ties" else 10
    start = Xd[rng.choice(len(Xd), k, replace=False)]
    o = bm.lloyd(bm.Dataset(X), bm.Centroids.from_rows(start), bm.SearchConfig(rel_tolerance=0.0))
    p = port.lloyd(Xd, start, np.zeros(k, np.uint8), 300, 0.0)
    assert (bits(o.centroids.values) == bits(p["centroids"])).all()
    assert (o.centroids.mask == p["mask"]).all()
    assert (o.assignment == p["labels"]).all()
    assert (bits(o.objective_history) == bits(p["history"])).all()


@pytest.mark.parametrize("case", ["integer", "real", "huge_integer", "partial_integer", "zeros"])
def test_kmeanspp_device_steps_vs_oracle(port, case):
    """K-means++ steps run on the device while the D^2 weights are integers
    (exact prefix sums), else on the host from the same stream position."""
    rng = np.random.default_rng(21)
    k, cands = 9, 3
    mask = np.ones(k, np.uint8)
    Cn = np.zeros((k, 5))
    if case == "integer":
        X = np.rint(rng.normal(size=(7000, 5)) * 6)
    elif case == "real":
        X = rng.normal(size=(7000, 5)) * 6
    elif case == "huge_integer":  # totals beyond 2^53: host prefix sums
        X = np.rint(rng.normal(size=(7000, 5)) * 2e7)
    elif case == "partial_integer":  # active rows are data points: integer weights
        X = np.rint(rng.normal(size=(7000, 5)) * 6)
        Cn[:3] = X[:3]
        mask[:3] = 0
    else:  # many coincident points: zero weights, total <= 0 branch
        X = np.zeros((500, 5))
        X[:3] = [[1, 0, 0, 0, 0], [2, 0, 0, 0, 0], [3, 0, 0, 0, 0]]
    counter = bm.EvalCounter()
    r = bm.Rng(44)
    got = bm.kmeanspp_fill(bm.Dataset(X), bm.Centroids(Cn.copy(), mask.copy()),
                           bm.InitConfig(candidates_per_step=cands), r, counter)
    pr = port.rng(44)
    Ce, me, ev = port.kmeanspp_fill(X, Cn.copy(), mask.copy(), cands, pr)
    assert (bits(got.values) == bits(Ce)).all()
    assert (got.mask == me).all()
    assert counter.distance_evals == ev
    assert r() == port.rng_next(pr)


# kmeans with every InitMethod (local_search.cpp:62-94): forgy (init.cpp:92-115),
# kmeans_pp (:123-201), kmeans_parallel with both rounds rules (:209-347).
@pytest.mark.parametrize("meth,rule,l", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (2, 1, 0), (2, 0, 4)])
@pytest.mark.parametrize("seed", range(3))
def test_kmeans_methods_vs_oracle(port, meth, rule, l, seed):
    rng = np.random.default_rng(900 + 7 * seed + meth)
    m, n, k = int(rng.integers(300, 6000)), int(rng.integers(1, 24)), int(rng.integers(1, 28))
    X = rng.normal(size=(m, n)) * rng.uniform(0.5, 20)
    if seed == 1:
        X = np.rint(X)
    if seed == 2:
        X = X.astype(np.float32)
    init = bm.InitConfig(seed=seed, method=meth, rounds_rule=rule, oversampling_l=l)
    out = bm.kmeans(bm.Dataset(X), k, init, bm.SearchConfig())
    p = port.kmeans(X.astype(np.float64), k, meth, seed, rounds_rule=rule, oversampling_l=l)
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.centroids.mask == p.mask).all()
    assert (out.assignment == p.labels).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


def test_kmeans_golden_methods(golden):
    for i in range(6):
        X = golden[f"km{i}_X"]
        meth, rule, l, k, seed = (int(v) for v in golden[f"km{i}_cfg"])
        out = bm.kmeans(bm.Dataset(X), k, bm.InitConfig(seed=seed, method=meth, rounds_rule=rule,
                                                        oversampling_l=l), bm.SearchConfig())
        assert (bits(out.centroids.values) == bits(golden[f"km{i}_C"])).all()
        assert (out.assignment == golden[f"km{i}_labels"]).all()
        assert out.objective == golden[f"km{i}_obj"][0]
        assert [out.counter.distance_evals, out.counter.iterations] == golden[f"km{i}_stats"].tolist()


def test_kmeans_config_errors():
    X = np.random.default_rng(1).normal(size=(30, 2))
    d = bm.Dataset(X)
    for meth in (0, 1, 2):
        with pytest.raises(bm.ConfigError):
            bm.kmeans(d, 31, bm.InitConfig(method=meth), bm.SearchConfig())
    with pytest.raises(bm.ConfigError):
        bm.kmeans(d, 3, bm.InitConfig(method=2, rounds_r=0), bm.SearchConfig())
    with pytest.raises(bm.ConfigError):
        bm.kmeans(d, 3, bm.InitConfig(method=7), bm.SearchConfig())
