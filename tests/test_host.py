"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the host-side API validates like the reference, and the device sampler's
Fisher-Yates resolution identity holds (pure-numpy restatement of
kernels.cuh k_fy_pass1..3 checked against the oracle's literal shuffle)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2204_07485_b200 import _capi, synthetic


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    declared = _capi.symbols_declared_in_header()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_capi.PROTOS) <= set(declared)
    assert lib.bm_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_no_fp64_fma_contraction_in_ptx():
    """The reference's x86-64 build emits no FMA (P1): no fp64 fma may appear in
    the device code.  Checked on the PTX of the exact build flags (IEEE
    division, which ptxas later expands with DFMA, stays div.rn.f64 here)."""
    from paper_2204_07485_b200 import build as b
    out = subprocess.run([b.NVCC, *[f for f in b.FLAGS if f != "-shared"], "-ptx", "-o", "-",
                          b.SOURCES[0]], capture_output=True, text=True, check=True).stdout
    assert "fma.rn.f64" not in out
    assert "sub.rn.f64" in out and "mul.rn.f64" in out and "add.rn.f64" in out


def test_assignment_sass_has_no_fma_in_distance_kernels():
    """SASS of the pure distance kernels (no division anywhere) has no DFMA."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _capi.LIB_PATH],
                          capture_output=True, text=True, check=True).stdout
    funcs = {}
    for part in sass.split("Function : ")[1:]:
        name, _, body = part.partition("\n")
        funcs[name.strip()] = body
    names = [n for n in funcs if "k_dist_rows" in n or "k_tile_sums" in n
             or ("k_assign" in n and "tma" not in n and "screen" not in n)]
    assert len(names) >= 5
    for name in names:
        assert "DFMA" not in funcs[name], name


def test_config_defaults_match_reference():
    c = _capi.bm_config()
    _capi.load().bm_config_init(ctypes.byref(c))
    assert (c.max_iterations, c.rel_tolerance, c.candidates_per_step, c.seed,
            c.final_assignment) == (300, 1e-4, 3, 123456789, 1)


def _resolve(m, s, js):
    """numpy restatement of the device resolution (kernels.cuh section 1)."""
    LT = np.full(s, -1, np.int64)
    last = {}
    for t, j in enumerate(js):
        if j < s:
            if j > t:
                LT[j] = max(LT[j], t)
        else:
            last[j] = max(last.get(j, -1), t)
    kept = np.ones(s, bool)
    for t, j in enumerate(js):
        if j >= s and last[j] == t:
            w = t
            while LT[w] >= 0:
                w = LT[w]
            kept[w] = False
    return np.array(sorted(list(np.nonzero(kept)[0]) + list(last)), np.uint64)


@pytest.mark.parametrize("m,s", [(1, 1), (5, 3), (40, 39), (1000, 600), (13500, 4000),
                                 (100000, 10000)])
def test_fisher_yates_resolution_identity(port, m, s):
    for seed in range(3):
        r = port.rng(seed)
        js = [port.uniform_int(r, i, m - 1) for i in range(s)]
        # replay the same draws through the oracle's literal swap loop
        exp = port.sample_chunk(m, s, port.rng(seed)) if s < m else np.arange(m, dtype=np.uint64)
        if s < m:
            assert (_resolve(m, s, js) == exp).all()


def test_synthetic_generators_shapes():
    for key, w in synthetic.CONFIGS.items():
        m = min(w.m, 2000)
        X = synthetic.generate(key, m)
        assert X.shape == (m, w.n)
        assert X.dtype == (np.float32 if w.dtype == "f32" else np.float64)
        assert np.isfinite(X).all()
    X = synthetic.generate("c5", 500)
    assert 0.8 < (X == 0).mean() < 0.94 and X.max() <= 999 and (X[X > 0] >= 1).all()
    X = synthetic.generate("c2", 500)
    assert (X == np.rint(X)).all()
    X = synthetic.generate("c4", 200).astype(np.float64)
    assert np.allclose(np.linalg.norm(X, axis=1), 1.0, atol=1e-5)


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2204_07485_b200")
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("CPU oracle", ""), f


def test_product_rng_matches_oracle_stream(port):
    """The product's host engine (bm_rng: MT19937-64 + libstdc++ Lemire /
    generate_canonical) is bit-identical to the restated std:: stream."""
    from paper_2204_07485_b200 import Rng
    rng = np.random.default_rng(0)
    for seed in (0, 1, 123456789, 2**64 - 1):
        a, b = Rng(seed), port.rng(seed)
        for _ in range(200):
            assert a() == port.rng_next(b)
        for _ in range(2000):
            kind = rng.integers(0, 4)
            if kind == 0:
                lo = int(rng.integers(0, 1 << 40)); hi = lo + int(rng.integers(0, 1 << 32))
            elif kind == 1:  # ranges near 2^63..2^64: frequent Lemire rejections
                lo = 0; hi = (1 << 63) + int(rng.integers(0, 1 << 62))
            elif kind == 2:
                lo = hi = int(rng.integers(0, 1 << 20))
            else:
                lo, hi = 0, (1 << 64) - 1
            assert a.uniform_int(lo, hi) == port.uniform_int(b, lo, hi)
            t = float(rng.uniform(0, 1e6))
            assert a.uniform_real(0.0, t) == port.uniform_real(b, 0.0, t)
