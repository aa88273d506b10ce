"""GPU parity: core kernels (core.cpp) — known answers from the reference's
test_core.cpp plus bitwise agreement with the golden vectors / oracle."""
import numpy as np
import pytest

import paper_2204_07485_b200 as bm
from conftest import bits

pytestmark = pytest.mark.gpu


def test_dataset_validates_shape_and_finiteness():  # test_core.cpp:27-37
    with pytest.raises(bm.ConfigError):
        bm.Dataset([1.0, 2.0, 3.0], 2, 2)
    with pytest.raises(bm.ConfigError):
        bm.Dataset([1.0, np.nan], 1, 2)
    with pytest.raises(bm.ConfigError):
        bm.Dataset([np.inf], 1, 1)
    with pytest.raises(bm.ConfigError):
        bm.Dataset(np.array([[1.0, np.inf]], np.float32))
    d = bm.Dataset([1.0, 2.0, 3.0, 4.0], 2, 2)
    assert (d.m, d.n) == (2, 2)
    v = d.values()
    assert v[1, 0] == 3.0 and v[1, 1] == 4.0


def test_gather_copies_rows_in_listed_order():  # test_core.cpp:39-45
    d = bm.Dataset([0.0, 1.0, 2.0, 3.0, 4.0, 5.0], 3, 2)
    g = d.gather([2, 0])
    assert g.m == 2
    v = g.values()
    assert v[0, 0] == 4.0 and v[1, 1] == 1.0
    with pytest.raises(bm.ConfigError):
        d.gather([3])


def test_assign_nearest_ties_low():  # test_core.cpp:72-82
    d = bm.Dataset([0.0, 0.0, 10.0, 0.0, 5.0, 0.0], 3, 2)
    c = bm.Centroids.from_rows([0.0, 0.0, 10.0, 0.0], 2, 2)
    counter = bm.EvalCounter()
    labels, dists = bm.assign_nearest(d, c, counter)
    assert labels.tolist() == [0, 1, 0]
    assert dists[0] == 0.0 and dists[2] == 25.0
    assert counter.distance_evals == 6


def test_assign_nearest_skips_degenerate():  # test_core.cpp:84-95
    d = bm.Dataset([0.0, 0.0, 10.0, 0.0], 2, 2)
    c = bm.Centroids.all_degenerate(2, 2)
    with pytest.raises(bm.StateError):
        bm.assign_nearest(d, c)
    c.set_row(1, [10.0, 0.0])
    counter = bm.EvalCounter()
    labels, _ = bm.assign_nearest(d, c, counter)
    assert labels.tolist() == [1, 1]
    assert counter.distance_evals == 2


def test_update_centroids_means_and_empty():  # test_core.cpp:97-108
    d = bm.Dataset([0.0, 0.0, 2.0, 0.0, 0.0, 4.0], 3, 2)
    c = bm.update_centroids(d, [0, 0, 2], 3)
    assert c.row(0)[0] == 1.0 and c.row(0)[1] == 0.0
    assert c.degenerate(1)
    assert c.row(2)[1] == 4.0
    with pytest.raises(bm.ConfigError):
        bm.update_centroids(d, [0, 0, 3], 3)


def test_objective_equals_summed_distances():  # test_core.cpp:110-119
    X = np.random.default_rng(7).uniform(-10, 10, (257, 3))
    d = bm.Dataset(X)
    c = bm.Centroids.from_rows(np.stack([X[0], X[9]]))
    _, dists = bm.assign_nearest(d, c)
    assert bm.objective(d, c) == pytest.approx(dists.sum(), rel=1e-12)


def test_core_golden_bitwise(golden):
    d = bm.Dataset(golden["core_X"])
    c = bm.Centroids(golden["core_C"], golden["core_mask"])
    counter = bm.EvalCounter()
    labels, dists = bm.assign_nearest(d, c, counter)
    assert (labels == golden["core_labels"]).all()
    assert (bits(dists) == bits(golden["core_dists"])).all()
    assert counter.distance_evals == int(golden["core_evals"][0])
    assert bm.objective(d, c) == golden["core_block_sum"][0]
    u = bm.update_centroids(d, labels, 4)
    assert (bits(u.values) == bits(golden["core_update_C"])).all()
    assert (u.mask == golden["core_update_mask"]).all()


def test_block_sum_golden(golden):  # test_core.cpp:121-136
    assert bm.block_sum(golden["blocksum_values"]) == golden["blocksum_total"][0]
    assert bm.block_sum(np.zeros(0)) == 0.0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n,k", [(1, 1), (2, 3), (16, 10), (28, 20), (68, 25), (70, 33), (300, 7)])
def test_assign_update_bitwise_vs_oracle(port, n, k, dtype):
    rng = np.random.default_rng(n * 100 + k)
    m = 3 * 1024 + 77
    X = (rng.normal(size=(m, n)) * 3).astype(dtype)
    Xd = X.astype(np.float64)
    C = Xd[rng.choice(m, k, replace=False)] + 0.25
    mask = (rng.random(k) < 0.2).astype(np.uint8)
    mask[0] = 0
    d = bm.Dataset(X)
    cent = bm.Centroids(C, mask)
    labels, dists = bm.assign_nearest(d, cent)
    l2, d2, _ = port.assign_nearest(Xd, cent.values, mask)
    assert (labels == l2).all()
    assert (bits(dists) == bits(d2)).all()
    u = bm.update_centroids(d, l2, k)
    uc, um = port.update_centroids(Xd, l2, k)
    assert (bits(u.values) == bits(uc)).all() and (u.mask == um).all()


def test_integer_data_exact_ties(port):
    """Integer-valued data (config 2 style) produces many exact distance ties."""
    rng = np.random.default_rng(3)
    X = rng.integers(0, 4, (5000, 3)).astype(np.float64)
    C = np.array([[1, 1, 1], [2, 2, 2], [1, 1, 1], [0, 2, 1], [2, 0, 1]], np.float64)
    mask = np.zeros(5, np.uint8)
    labels, dists = bm.assign_nearest(bm.Dataset(X), bm.Centroids(C, mask))
    l2, d2, _ = port.assign_nearest(X, C, mask)
    assert (labels == l2).all() and (bits(dists) == bits(d2)).all()


ADVERSARIAL = {
    # exact ties: duplicated centroids and points on bisectors
    "dup_centroids": lambda r: (r.integers(0, 5, (4000, 3)).astype(np.float64),
                                np.array([[1, 1, 1], [1, 1, 1], [2, 2, 2], [0, 0, 0], [2, 2, 2.0]])),
    # values far beyond fp32 range: the screen must defer to the exact path
    "beyond_fp32": lambda r: (r.normal(size=(3000, 4)) * 1e40,
                              r.normal(size=(6, 4)) * 1e40),
    # fp32-subnormal magnitudes
    "subnormal": lambda r: (r.normal(size=(3000, 5)) * 1e-41,
                            r.normal(size=(7, 5)) * 1e-41),
    # large offset, tiny spread (catastrophic for a norm-expansion screen)
    "offset": lambda r: (1e6 + r.normal(size=(5000, 8)) * 1e-3,
                         1e6 + r.normal(size=(12, 8)) * 1e-3),
    # mixed scales per dimension
    "mixed": lambda r: (r.normal(size=(5000, 30)) * np.logspace(-8, 8, 30),
                        r.normal(size=(20, 30)) * np.logspace(-8, 8, 30)),
    # near ties: centroids separated by one ulp
    "ulp_pairs": lambda r: (r.normal(size=(4000, 2)),
                            np.array([[0.5, 0.5], [np.nextafter(0.5, 1), 0.5], [-0.5, 0.1],
                                      [-0.5, np.nextafter(0.1, 1)]])),
}


@pytest.mark.parametrize("case", sorted(ADVERSARIAL))
def test_screen_adversarial_bitwise(port, case):
    X, C = ADVERSARIAL[case](np.random.default_rng(11))
    X = X.copy()
    X[:C.shape[0]] = C  # points that coincide with centroids (distance 0)
    mask = np.zeros(C.shape[0], np.uint8)
    labels, dists = bm.assign_nearest(bm.Dataset(X), bm.Centroids(C, mask))
    l2, d2, _ = port.assign_nearest(X, C, mask)
    assert (labels == l2).all()
    assert (bits(dists) == bits(d2)).all()
    assert bm.objective(bm.Dataset(X), bm.Centroids(C, mask)) == port.block_sum(d2)


_MODE_CODE = (
    "import numpy as np, sys; sys.path.insert(0, '.');"
    "import paper_2204_07485_b200 as bm;"
    "X = {X};"
    "o, t = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k={k}, chunk_size={s}, max_chunks=6, seed=3));"
    "import hashlib; print(repr(o.objective), o.counter.distance_evals, o.counter.iterations,"
    " hashlib.sha1(o.centroids.values.tobytes()).hexdigest(), repr(t.records))")


def _modes_agree(base, var, alt, X="np.rint(np.random.default_rng(5).normal(size=(20000, 16)) * 4)", k=10, s=3000):
    import subprocess, sys, os
    code = _MODE_CODE.format(X=X, k=k, s=s)
    outs = []
    for mode in (None, alt):
        env = dict(os.environ)
        env.update(base)
        env.pop(var, None)
        if mode is not None:
            env[var] = mode
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                   text=True, check=True).stdout)
    assert outs[0] == outs[1] and outs[0]


# The persistent chunk kernel (default) against the multi-launch chunk graphs
# and the host-driven loop, the screens against each other, and the
# deferred-objective / carveout switches: same bits, fresh processes.
@pytest.mark.parametrize("var,alt", [("BM_PERSIST", "0"), ("BM_GRAPHS", "0"), ("BM_STORAGE", "native"),
                                     ("BM_FORCE_EXACT_CONTROL", "1"), ("BM_TC", "0"), ("BM_CHUNK_FIX", "0"),
                                     ("BM_CARVEOUT", "0"), ("BM_PP", "host"), ("BM_CHUNK_RED", "0")])
def test_engine_modes_agree(var, alt):
    _modes_agree({}, var, alt)


@pytest.mark.parametrize("data", ["int", "real"])
def test_tc_screen_forced_agrees(data):
    """Real-valued fp32 rows are not exact in tf32: the default packed-FFMA
    screen against the tensor-core screen forced on (its loose bound)."""
    X = ("np.random.default_rng(5).normal(size=(20000, 16)).astype(np.float32)" if data == "real"
         else "np.rint(np.random.default_rng(5).normal(size=(20000, 16)) * 4)")
    _modes_agree({}, "BM_TC", "1", X=X)


# Switches of the multi-launch chunk graphs (still the path for rows wider
# than the chunk kernel's instances): each against that path's default.
@pytest.mark.parametrize("var,alt", [("BM_ASSIGN_MODE", "exact"), ("BM_HAMERLY", "0"), ("BM_SPEC", "0"),
                                     ("BM_PDL", "0"), ("BM_SUMS", "0"), ("BM_SUMS_FUSE", "0"),
                                     ("BM_FORCE_EXACT_CONTROL", "1")])
def test_multi_launch_modes_agree(var, alt):
    _modes_agree({"BM_PERSIST": "0"}, var, alt)


def test_lossless_fp32_storage():
    """fp64 input that round-trips through fp32 is stored as fp32; anything else stays fp64."""
    Xi = np.rint(np.random.default_rng(1).normal(size=(1000, 5)) * 100)
    assert bm.Dataset(Xi).storage == "f32"
    Xr = np.random.default_rng(1).normal(size=(1000, 5))
    assert bm.Dataset(Xr).storage == "f64"
    assert bm.Dataset(Xr.astype(np.float32)).storage == "f32"
    d = bm.Dataset(Xi)
    assert (d.values() == Xi).all()
    with pytest.raises(bm.ConfigError):
        bm.Dataset(np.array([[1.0, np.nan]]))


@pytest.mark.parametrize("shape,dtype", [((5000, 7), np.float64), ((3000, 300), np.float32), ((777, 1), np.float64)])
def test_min_max_normalize(shape, dtype):
    """io::min_max_normalize (io.cpp:245-264): (x - lo) / (hi - lo) per column, constant
    columns 0.0 — restated with numpy float64 (IEEE, no contraction)."""
    r = np.random.default_rng(3)
    X = (r.normal(size=shape) * r.uniform(0.1, 50, shape[1]) + r.normal(size=shape[1]) * 10).astype(dtype)
    X[:, 0] = 2.5  # a constant column
    if shape[1] > 2:
        X[:, 2] = np.rint(X[:, 2])
    Y = bm.Dataset(X).min_max_normalize().values()
    Xd = X.astype(np.float64)
    lo, hi = Xd.min(axis=0), Xd.max(axis=0)
    rng_ = hi - lo
    with np.errstate(invalid="ignore", divide="ignore"):
        ref = np.where(rng_ > 0.0, (Xd - lo) / rng_, 0.0)
    assert (bits(Y) == bits(ref)).all()


@pytest.mark.parametrize("var,alt", [("BM_SPEC", "0"), ("BM_HAMERLY", "0")])
def test_engine_modes_agree_wide_rows(var, alt):
    """Rows wider than the chunk kernel's instances (multi-launch path, 6-stage
    TMA ring): speculative begins and the bound fast path off, same bits."""
    _modes_agree({}, var, alt, X="np.random.default_rng(6).normal(size=(9000, 200)).astype(np.float32)", k=9, s=2500)


