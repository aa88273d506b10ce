"""GPU parity: the big_means driver (big_means.cpp:58-112) — reference
test_big_means.cpp / acceptance criteria 2, 3, 9 and bitwise agreement with the
golden vectors and the oracle on every BASELINE config (reduced m and s)."""
import numpy as np
import pytest

import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import synthetic
from conftest import bits

pytestmark = pytest.mark.gpu


def cfg(k, s, chunks, seed=bm.K_DEFAULT_SEED, **kw):
    return bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=chunks, seed=seed, **kw)


@pytest.mark.parametrize("i", range(4))
def test_big_means_golden(golden, i):
    X = golden[f"bm{i}_X"]
    k, s, ch, seed = golden[f"bm{i}_cfg"].tolist()
    out, trace = bm.big_means(bm.Dataset(X), cfg(k, s, ch, seed))
    assert (bits(out.centroids.values) == bits(golden[f"bm{i}_C"])).all()
    assert (out.centroids.mask == golden[f"bm{i}_mask"]).all()
    assert (out.assignment == golden[f"bm{i}_labels"]).all()
    assert out.objective == golden[f"bm{i}_obj"][0]
    assert [out.counter.distance_evals, out.counter.iterations, trace.chunks()] == \
        golden[f"bm{i}_stats"].tolist()
    tr = np.array([[r.candidate_objective, r.incumbent_objective] for r in trace.records])
    assert (bits(tr) == bits(golden[f"bm{i}_trace"])).all()
    ti = np.array([[r.chunk_index, r.accepted, r.degenerate_repaired] for r in trace.records],
                  np.uint64)
    assert ti.tolist() == golden[f"bm{i}_trace_int"].tolist()


def test_validation():  # test_big_means.cpp:56-73
    d = bm.Dataset(np.random.default_rng(3).uniform(0, 50, (50, 2)))
    with pytest.raises(bm.ConfigError):
        bm.big_means(d, bm.BigMeansConfig(k=3, chunk_size=10))
    for bad in (cfg(0, 10, 1), cfg(5, 4, 1), cfg(5, 51, 1), cfg(5, 10, 0)):
        with pytest.raises(bm.ConfigError):
            bm.big_means(d, bad)
    with pytest.raises(bm.ConfigError):
        bm.big_means(d, bm.BigMeansConfig(k=5, chunk_size=10, max_cpu_seconds=-1.0))


def test_trace_monotone_and_first_chunk_repairs_k():  # test_big_means.cpp:75-92
    d = bm.Dataset(np.random.default_rng(4).uniform(0, 50, (600, 2)))
    out, trace = bm.big_means(d, cfg(5, 100, 40))
    assert trace.chunks() == 40
    prev = trace.records[0].incumbent_objective
    for i, r in enumerate(trace.records):
        assert r.chunk_index == i and r.incumbent_objective <= prev
        prev = r.incumbent_objective
        if r.accepted:
            assert r.incumbent_objective == r.candidate_objective
        else:
            assert r.candidate_objective >= r.incumbent_objective
    assert trace.records[0].accepted and trace.records[0].degenerate_repaired == 5


def test_final_pass_and_skip():  # test_big_means.cpp:103-128
    X = np.random.default_rng(6).uniform(0, 50, (500, 2))
    d = bm.Dataset(X)
    out, _ = bm.big_means(d, cfg(4, 80, 15))
    assert out.assignment.size == 500
    assert bm.objective(d, out.centroids) == out.objective
    labels, _ = bm.assign_nearest(d, out.centroids)
    assert (labels == out.assignment).all() and out.counter.cpu_full > 0.0
    out2, tr2 = bm.big_means(d, cfg(4, 80, 15, final_assignment=False))
    assert out2.assignment.size == 0
    assert out2.objective == tr2.records[-1].incumbent_objective
    assert out.counter.distance_evals - out2.counter.distance_evals == 500 * 4


def test_budgets_and_determinism():  # test_big_means.cpp:130-158
    d = bm.Dataset(np.random.default_rng(7).uniform(0, 50, (400, 2)))
    _, tr = bm.big_means(d, cfg(3, 50, 6))
    assert tr.chunks() == 6
    out, tr = bm.big_means(d, bm.BigMeansConfig(k=3, chunk_size=50, max_cpu_seconds=0.05))
    assert tr.chunks() >= 1 and out.counter.cpu_init >= 0.0
    d = bm.Dataset(np.random.default_rng(8).uniform(0, 50, (800, 2)))
    a, ta = bm.big_means(d, cfg(5, 120, 30, seed=31337))
    b, tb = bm.big_means(d, cfg(5, 120, 30, seed=31337))
    assert a.centroids == b.centroids and (a.assignment == b.assignment).all()
    assert bits([a.objective]) == bits([b.objective])
    assert [r.candidate_objective for r in ta.records] == [r.candidate_objective for r in tb.records]


@pytest.mark.parametrize("seed", range(5))
def test_single_chunk_equals_kmeans(seed, port):  # test_big_means.cpp:177-195, criterion 3
    X = np.random.default_rng(40 + seed).uniform(0, 50, (200 + 30 * seed, 2))
    d = bm.Dataset(X)
    b, _ = bm.big_means(d, cfg(4, X.shape[0], 1, seed=900 + seed))
    km = bm.kmeans(d, 4, bm.InitConfig(seed=900 + seed), bm.SearchConfig())
    assert b.centroids == km.centroids and (b.assignment == km.assignment).all()
    assert bits([b.objective]) == bits([km.objective])
    assert b.counter.iterations == km.counter.iterations
    p = port.kmeans_pp(X, 4, 900 + seed)
    assert km.objective == p.objective and km.counter.distance_evals == p.evals


@pytest.mark.parametrize("seed", range(8))
def test_big_means_vs_oracle_random(port, seed):
    rng = np.random.default_rng(500 + seed)
    m = int(rng.integers(300, 20000))
    n = int(rng.integers(1, 40))
    k = int(rng.integers(1, 30))
    s = int(rng.integers(k, min(m, 5000) + 1))
    X = rng.normal(size=(m, n)) * rng.uniform(0.1, 30)
    if seed % 3 == 1:
        X = np.rint(X)
    if seed % 3 == 2:
        X = X.astype(np.float32)
    out, trace = bm.big_means(bm.Dataset(X), cfg(k, s, 8, seed=seed))
    p = port.big_means(X.astype(np.float64), k, s, 8, seed=seed)
    got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
            r.degenerate_repaired) for r in trace.records]
    assert got == p.trace
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.assignment == p.labels).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


CONFIG_SCALE = {"c1": (1.0, 6), "c2": (0.02, 4), "c3": (0.005, 4), "c4": (0.05, 3),
                "c5": (0.25, 3)}


@pytest.mark.parametrize("key", sorted(CONFIG_SCALE))
def test_configs_bitwise_vs_oracle(port, key):
    """Every BASELINE config's generator, reduced m/s, bitwise vs the oracle."""
    scale, chunks = CONFIG_SCALE[key]
    w = synthetic.scaled(synthetic.CONFIGS[key], scale, chunks)
    X = synthetic.generate(key, w.m)
    out, trace = bm.big_means(bm.Dataset(X), cfg(w.k, w.s, w.chunks, seed=w.seed))
    p = port.big_means(X.astype(np.float64), w.k, w.s, w.chunks, seed=w.seed)
    got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
            r.degenerate_repaired) for r in trace.records]
    assert got == p.trace
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.assignment == p.labels).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


@pytest.mark.parametrize("case", ["tiny_chunks", "duplicates"])
def test_mid_run_repairs_vs_oracle(port, case):
    """Accepted candidates with empty clusters force K-means++ repairs in later
    chunks: the pipelined loop's speculative draws and queued Lloyd graphs for
    those chunks must be discarded and redone in the reference's RNG order."""
    rng = np.random.default_rng(77)
    if case == "tiny_chunks":  # small chunks of coarse data: empty clusters are common
        X = np.rint(rng.normal(size=(4000, 5)) * 0.5)
        k, s, chunks = 8, 20, 40
    else:  # heavy duplication: many coincident points, degenerate clusters
        X = np.rint(rng.normal(size=(3000, 3)))
        k, s, chunks = 16, 40, 40
    out, trace = bm.big_means(bm.Dataset(X), cfg(k, s, chunks, seed=5))
    p = port.big_means(X.astype(np.float64), k, s, chunks, seed=5)
    got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
            r.degenerate_repaired) for r in trace.records]
    assert sum(1 for r in p.trace[1:] if r[4] > 0) >= 2  # repairs after the first chunk
    assert got == p.trace
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


def test_graphs_shared_across_datasets(port):
    """The chunk graphs are captured once per shape and read the dataset base
    from a device slot: alternating datasets of one shape (the second freed
    before the third is created, so its address can be reused) must each
    match the oracle."""
    rng = np.random.default_rng(91)
    xs = [np.rint(rng.normal(size=(6000, 12)) * (3 + i)) for i in range(3)]
    k, s, chunks = 6, 700, 6
    for i in (0, 1, 0, 2):
        d = bm.Dataset(xs[i])
        out, trace = bm.big_means(d, cfg(k, s, chunks, seed=11))
        d.close()
        p = port.big_means(xs[i], k, s, chunks, seed=11)
        assert [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
                 r.degenerate_repaired) for r in trace.records] == p.trace
        assert (bits(out.centroids.values) == bits(p.centroids)).all()
        assert (out.assignment == p.labels).all()


@pytest.mark.parametrize("case", ["f32_storage", "f64_storage", "ragged"])
def test_long_runs_vs_oracle(port, case):
    """Long runs where the incumbent settles early (most chunks rejected, the
    speculative begins of the pipeline current), fp32 and fp64 storage and
    ragged tiles, bitwise against the oracle."""
    rng = np.random.default_rng(31)
    m, n, k, s, chunks = {"f32_storage": (30000, 9, 7, 1500, 30),
                          "f64_storage": (20000, 6, 5, 1000, 30),
                          "ragged": (12345, 13, 11, 777, 25)}[case]
    centers = rng.uniform(0, 40, (k, n))
    X = centers[rng.integers(0, k, m)] + rng.normal(size=(m, n))
    if case != "f64_storage":
        X = np.rint(X * 4)  # exactly representable in fp32: fp32 storage
    out, trace = bm.big_means(bm.Dataset(X), cfg(k, s, chunks, seed=2))
    p = port.big_means(X, k, s, chunks, seed=2)
    got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
            r.degenerate_repaired) for r in trace.records]
    assert got == p.trace
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.assignment == p.labels).all()
    assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


# Exact-sum regimes (kernels.cuh §5b): the device keeps integer label sums when
# every value is a multiple of 2^e and m * max|x| < 2^52 * 2^e; the results
# must stay bitwise equal to the reference's ordered sums in every regime,
# including datasets just inside and just outside the test.
def _sum_regimes():
    r = np.random.default_rng(77)
    return {
        "small_ints": (np.rint(r.normal(size=(12000, 12)) * 40), True, 0),
        "even_ints": (np.rint(r.normal(size=(12000, 9)) * 40) * 8, True, 3),
        "quarter_steps": (np.rint(r.normal(size=(12000, 7)) * 400) / 4, True, -2),
        "fine_steps_f64": (np.rint(r.normal(size=(12000, 6)) * 2.0**36) * 2.0**-40, True, -40),
        "huge_ints": (np.rint(r.normal(size=(12000, 5)) * 2.0**36), True, 0),
        "too_wide": (np.rint(r.normal(size=(12000, 5)) * 2.0**40), False, None),
        "gaussian": (r.normal(size=(12000, 8)), False, None),
        "fp32_ints": (np.rint(r.normal(size=(12000, 10)) * 30).astype(np.float32), True, 0),
    }


@pytest.mark.parametrize("case", sorted(_sum_regimes()))
def test_exact_sum_regimes_vs_oracle(port, case):
    X, exact, e = _sum_regimes()[case]
    d = bm.Dataset(X)
    got_exact, got_e = d.exact_sums
    assert got_exact == exact
    if exact:
        # the lowest set bit over the data can only be at or above the construction's step
        assert got_e >= e
    for k, s, chunks, seed in ((7, 1500, 10, 1), (25, 3000, 6, 2)):
        out, trace = bm.big_means(d, cfg(k, s, chunks, seed=seed))
        p = port.big_means(X.astype(np.float64), k, s, chunks, seed=seed)
        got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
                r.degenerate_repaired) for r in trace.records]
        assert got == p.trace
        assert out.objective == p.objective
        assert (bits(out.centroids.values) == bits(p.centroids)).all()
        assert (out.assignment == p.labels).all()
        assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


def test_chunk_size_hint_known_answers(port):
    """test_big_means.cpp:197-215: within [k, m], deterministic, custom ladder respected;
    equal to the oracle's probe loop."""
    X = np.random.default_rng(8).uniform(0, 10, (512, 2))
    d = bm.Dataset(X)
    hint = bm.choose_chunk_size_hint(d, 4, bm.ChunkHintConfig())
    assert 4 <= hint <= 512 and hint == bm.choose_chunk_size_hint(d, 4, bm.ChunkHintConfig())
    assert hint == port.choose_chunk_size_hint(X, 4)
    h2 = bm.choose_chunk_size_hint(d, 3, bm.ChunkHintConfig(ladder=[32, 64, 128]))
    assert h2 in (32, 64, 128) and h2 == port.choose_chunk_size_hint(X, 3, (32, 64, 128))
    with pytest.raises(bm.ConfigError):
        bm.choose_chunk_size_hint(d, 600, bm.ChunkHintConfig())
    with pytest.raises(bm.ConfigError):
        bm.choose_chunk_size_hint(d, 3, bm.ChunkHintConfig(runs_per_candidate=0))


@pytest.mark.parametrize("integer", [False, True])
def test_time_budget_vs_oracle(port, integer):
    """Time-budget runs (big_means.cpp:74-77: no chunk count in advance, so no
    speculation ahead): whatever number of chunks ran, the result is the
    reference's for that chunk budget, bit for bit (ordered and exact-sum updates)."""
    r = np.random.default_rng(91)
    X = r.normal(size=(30000, 12)) * 8.0
    if integer:
        X = np.rint(X)
    out, tr = bm.big_means(bm.Dataset(X), bm.BigMeansConfig(k=9, chunk_size=2500, max_cpu_seconds=0.15, seed=4))
    c = tr.chunks()
    assert c >= 1
    p = port.big_means(X, 9, 2500, c, seed=4)
    got = [(r_.chunk_index, r_.candidate_objective, r_.incumbent_objective, r_.accepted,
            r_.degenerate_repaired) for r_ in tr.records]
    assert got == p.trace
    assert out.objective == p.objective
    assert (bits(out.centroids.values) == bits(p.centroids)).all()
    assert (out.assignment == p.labels).all()


@pytest.mark.parametrize("screen", ["tc", "ffma"])
@pytest.mark.parametrize("n", [3, 6, 13, 16, 24, 28, 37, 68, 80])
def test_chunk_kernel_screens_vs_oracle(port, monkeypatch, screen, n):
    """The persistent chunk kernel's two screens for fp32 rows — tensor core
    (tcgen05 kind::tf32, swizzled rows; forced with BM_TC=1 even for data that
    is not exact in tf32, i.e. the loose certified bound) and packed FFMA
    (BM_TC=0) — on every row-width instance, bitwise against the oracle."""
    monkeypatch.setenv("BM_TC", "1" if screen == "tc" else "0")
    rng = np.random.default_rng(1000 + n)
    m, k, s = 9000, 11, 2100
    X = (rng.normal(size=(m, n)) * 5.0 + rng.integers(0, 3, (m, 1)) * 4.0).astype(np.float32)
    for integer in (False, True):
        Xi = np.rint(X) if integer else X  # integer rows: exact-sum mode (B spread over the SMs)
        out, trace = bm.big_means(bm.Dataset(Xi), cfg(k, s, 5, seed=n))
        p = port.big_means(np.asarray(Xi, np.float64), k, s, 5, seed=n)
        got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
                r.degenerate_repaired) for r in trace.records]
        assert got == p.trace
        assert out.objective == p.objective
        assert (bits(out.centroids.values) == bits(p.centroids)).all()
        assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)


@pytest.mark.parametrize("n,k,m,s", [(89, 7, 3000, 700), (100, 3, 2000, 520), (300, 17, 2600, 900),
                                     (777, 32, 1500, 600), (2500, 10, 900, 400), (5003, 5, 600, 300),
                                     (5000, 10, 4500, 4000)])  # the last: c5's split shape (2 atoms per block)
def test_wide_rows_tensor_core_prescreen_vs_oracle(port, monkeypatch, n, k, m, s):
    """Wide fp32 rows exact in tf32 (n > 88, the c5 regime): the split-K
    tensor-core pre-screen (wide.cu, tcgen05 kind::tf32 with one TMEM block
    per 32-dim atom) feeding k_assign_tma's recheck — bitwise against the
    oracle, with the pre-screen on and off (BM_WIDE=0); ragged tiles and atoms,
    N = 16 and 32 centroid slots, 1..many splits."""
    rng = np.random.default_rng(n + 7 * k)
    grp = rng.integers(0, 3, (m, 1))
    X = np.where(rng.random((m, n)) < 0.85, 0.0, rng.integers(1, 1000, (m, n)) * (grp + 1.0)).astype(np.float64)
    chunks = 2 if s >= 4000 else 4
    p = port.big_means(X, k, s, chunks, seed=n)
    for wide in ("1", "0"):
        monkeypatch.setenv("BM_WIDE", wide)
        out, trace = bm.big_means(bm.Dataset(X), cfg(k, s, chunks, seed=n))
        got = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted,
                r.degenerate_repaired) for r in trace.records]
        assert got == p.trace, wide
        assert out.objective == p.objective
        assert (bits(out.centroids.values) == bits(p.centroids)).all()
        assert (out.assignment == p.labels).all()
        assert (out.counter.distance_evals, out.counter.iterations) == (p.evals, p.iterations)
