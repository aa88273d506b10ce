"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two interchangeable back ends with identical signatures:

* ``port`` -- oracle/_port/libbm_oracle.so, the plain-C restatement
  (bm_oracle.c) of the reference hot path;
* ``ref``  -- oracle/_ref/libbigmeans_ref.so, the unmodified reference
  sources compiled by oracle/Makefile (present wherever it was built; the
  .so travels to the GPU box, /root/reference does not).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_port", "libbm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbigmeans_ref.so")

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class _Init(C.Structure):  # orc_init / ref_init (InitConfig init.hpp:16-27)
    _fields_ = [("method", C.c_int), ("candidates_per_step", C.c_int), ("oversampling_l", C.c_int),
                ("rounds_r", C.c_int), ("rounds_rule", C.c_int), ("seed", C.c_uint64)]


class _RefConfig(C.Structure):
    _fields_ = [("k", _u64), ("chunk_size", _u64), ("has_max_chunks", C.c_int),
                ("max_chunks", _u64), ("has_max_cpu_seconds", C.c_int),
                ("max_cpu_seconds", C.c_double), ("max_iterations", _u64),
                ("rel_tolerance", C.c_double), ("candidates_per_step", C.c_int),
                ("seed", _u64), ("final_assignment", C.c_int)]


class _PortConfig(C.Structure):
    _fields_ = [("k", _u64), ("chunk_size", _u64), ("max_chunks", _u64),
                ("max_iterations", _u64), ("rel_tolerance", C.c_double),
                ("candidates_per_step", C.c_int), ("seed", _u64),
                ("final_assignment", C.c_int)]


class _Record(C.Structure):
    _fields_ = [("chunk_index", _u64), ("candidate_objective", C.c_double),
                ("incumbent_objective", C.c_double), ("accepted", _u64),
                ("degenerate_repaired", _u64)]


class _RefOutcome(C.Structure):
    _fields_ = [("objective", C.c_double), ("evals", _u64), ("iterations", _u64),
                ("chunks", _u64), ("cpu_init", C.c_double), ("cpu_full", C.c_double)]


class _PortOutcome(C.Structure):
    _fields_ = [("objective", C.c_double), ("evals", _u64), ("iterations", _u64),
                ("chunks", _u64)]


class _LloydOut(C.Structure):
    _fields_ = [("objective", C.c_double), ("evals", _u64), ("iterations", _u64),
                ("history_len", _u64)]


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


@dataclass
class BigMeansResult:
    centroids: np.ndarray
    mask: np.ndarray
    labels: np.ndarray | None
    objective: float
    evals: int
    iterations: int
    chunks: int
    trace: list = field(default_factory=list)
    cpu_init: float = 0.0
    cpu_full: float = 0.0


class Oracle:
    """One back end (``kind`` = "port" or "ref")."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run make -f oracle/Makefile)")
        self.lib = C.CDLL(path)
        self.pre = "orc_" if kind == "port" else "ref_"
        self._rngs = []

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    # -- RNG ---------------------------------------------------------------
    def rng(self, seed: int):
        if self.kind == "port":
            buf = (C.c_uint64 * 313)()
            self._rngs.append(buf)
            h = C.c_void_p(C.addressof(buf))
            self.lib.orc_rng_seed(h, _u64(seed))
            return h
        self.lib.ref_rng_create.restype = C.c_void_p
        h = C.c_void_p(self.lib.ref_rng_create(_u64(seed)))
        self._rngs.append(h)
        return h

    def rng_next(self, r) -> int:
        f = self._fn("rng_next")
        f.restype = _u64
        return int(f(r))

    def uniform_int(self, r, a, b) -> int:
        f = self._fn("uniform_int")
        f.restype = _u64
        return int(f(r, _u64(a), _u64(b)))

    def uniform_real(self, r, a, b) -> float:
        f = self._fn("uniform_real")
        f.restype = C.c_double
        f.argtypes = [C.c_void_p, C.c_double, C.c_double]
        return float(f(r, a, b))

    # -- kernels -----------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            msg = ""
            if self.kind == "ref":
                self.lib.ref_last_error.restype = C.c_char_p
                msg = self.lib.ref_last_error().decode()
            raise OracleError(rc, msg)

    def sample_chunk(self, m, s, r):
        out = np.empty(s, np.uint64)
        self._check(self._fn("sample_chunk")(_u64(m), _u64(s), r, _p(out, _u64p)))
        return out

    def assign_nearest(self, X, Cn, mask):
        X = _f64(X)
        Cn = _f64(Cn)
        mask = np.ascontiguousarray(mask, np.uint8)
        m, n = X.shape
        k = Cn.shape[0]
        labels = np.empty(m, np.int32)
        dists = np.empty(m, np.float64)
        ev = _u64(0)
        self._check(self._fn("assign_nearest")(_p(X, _dp), _u64(m), _u64(n), _p(Cn, _dp),
                                               _p(mask, _u8p), _u64(k), _p(labels, _i32p),
                                               _p(dists, _dp), C.byref(ev)))
        return labels, dists, int(ev.value)

    def block_sum(self, v) -> float:
        v = _f64(v)
        f = self._fn("block_sum")
        f.restype = C.c_double
        return float(f(_p(v, _dp), _u64(v.size)))

    def update_centroids(self, X, labels, k):
        X = _f64(X)
        labels = np.ascontiguousarray(labels, np.int32)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        mask = np.empty(k, np.uint8)
        self._check(self._fn("update_centroids")(_p(X, _dp), _u64(m), _u64(n),
                                                 _p(labels, _i32p), _u64(k), _p(Cn, _dp),
                                                 _p(mask, _u8p)))
        return Cn, mask

    def kmeanspp_fill(self, P, Cn, mask, candidates, r):
        P = _f64(P)
        Cn = _f64(Cn).copy()
        mask = np.ascontiguousarray(mask, np.uint8).copy()
        m, n = P.shape
        ev = _u64(0)
        self._check(self._fn("kmeanspp_fill")(_p(P, _dp), _u64(m), _u64(n), _p(Cn, _dp),
                                              _p(mask, _u8p), _u64(Cn.shape[0]),
                                              C.c_int(candidates), r, C.byref(ev)))
        Cn[mask.astype(bool)] = 0.0
        return Cn, mask, int(ev.value)

    def lloyd(self, X, Cn, mask, max_iterations=300, rel_tolerance=1e-4):
        X = _f64(X)
        Cn = _f64(Cn).copy()
        mask = np.ascontiguousarray(mask, np.uint8).copy()
        m, n = X.shape
        k = Cn.shape[0]
        labels = np.empty(m, np.int32)
        cap = int(max_iterations) + 1
        hist = np.empty(cap, np.float64)
        if self.kind == "port":
            lo = _LloydOut()
            self._check(self.lib.orc_lloyd(_p(X, _dp), _u64(m), _u64(n), _p(Cn, _dp),
                                           _p(mask, _u8p), _u64(k), _u64(max_iterations),
                                           C.c_double(rel_tolerance), _p(labels, _i32p),
                                           _p(hist, _dp), _u64(cap), C.byref(lo)))
            obj, ev, it, hl = lo.objective, lo.evals, lo.iterations, lo.history_len
        else:
            obj, ev, it, hl = C.c_double(), _u64(), _u64(), _u64()
            self._check(self.lib.ref_lloyd(_p(X, _dp), _u64(m), _u64(n), _p(Cn, _dp),
                                           _p(mask, _u8p), _u64(k), _u64(max_iterations),
                                           C.c_double(rel_tolerance), _p(labels, _i32p),
                                           _p(hist, _dp), _u64(cap), C.byref(obj),
                                           C.byref(ev), C.byref(it), C.byref(hl)))
            obj, ev, it, hl = obj.value, ev.value, it.value, hl.value
        return dict(centroids=Cn, mask=mask, labels=labels, objective=float(obj),
                    evals=int(ev), iterations=int(it), history=hist[:min(int(hl), cap)].copy())

    def big_means(self, X, k, chunk_size, max_chunks, seed=123456789, max_iterations=300,
                  rel_tolerance=1e-4, candidates_per_step=3, final_assignment=True,
                  max_cpu_seconds=None) -> BigMeansResult:
        X = _f64(X)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        mask = np.empty(k, np.uint8)
        labels = np.empty(m, np.int32) if final_assignment else None
        cap = int(max_chunks) if max_chunks else 1 << 20
        trace = (_Record * cap)()
        if self.kind == "port":
            if max_cpu_seconds is not None or not max_chunks:
                raise OracleError(1, "the C restatement supports chunk budgets only")
            cfg = _PortConfig(k, chunk_size, max_chunks, max_iterations, rel_tolerance,
                              candidates_per_step, seed, int(final_assignment))
            out = _PortOutcome()
            self._check(self.lib.orc_big_means(_p(X, _dp), _u64(m), _u64(n), C.byref(cfg),
                                               _p(Cn, _dp), _p(mask, _u8p), _p(labels, _i32p),
                                               trace, C.byref(out)))
            cpu_init = cpu_full = 0.0
        else:
            cfg = _RefConfig(k, chunk_size, int(bool(max_chunks)), max_chunks or 0,
                             int(max_cpu_seconds is not None), max_cpu_seconds or 0.0,
                             max_iterations, rel_tolerance, candidates_per_step, seed,
                             int(final_assignment))
            out = _RefOutcome()
            self._check(self.lib.ref_big_means(_p(X, _dp), _u64(m), _u64(n), C.byref(cfg),
                                               _p(Cn, _dp), _p(mask, _u8p), _p(labels, _i32p),
                                               trace, _u64(cap), C.byref(out)))
            cpu_init, cpu_full = out.cpu_init, out.cpu_full
        recs = [(int(t.chunk_index), float(t.candidate_objective), float(t.incumbent_objective),
                 bool(t.accepted), int(t.degenerate_repaired)) for t in trace[:int(out.chunks)]]
        return BigMeansResult(Cn, mask, labels, float(out.objective), int(out.evals),
                              int(out.iterations), int(out.chunks), recs, cpu_init, cpu_full)

    def kmeans_pp(self, X, k, seed, candidates=3, max_iterations=300, rel_tolerance=1e-4):
        X = _f64(X)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        mask = np.empty(k, np.uint8)
        labels = np.empty(m, np.int32)
        out = _PortOutcome() if self.kind == "port" else _RefOutcome()
        self._check(self._fn("kmeans_pp")(_p(X, _dp), _u64(m), _u64(n), _u64(k),
                                          C.c_int(candidates), _u64(seed),
                                          _u64(max_iterations), C.c_double(rel_tolerance),
                                          _p(Cn, _dp), _p(mask, _u8p), _p(labels, _i32p),
                                          C.byref(out)))
        return BigMeansResult(Cn, mask, labels, float(out.objective), int(out.evals),
                              int(out.iterations), 1)

    # -- kmeans drivers with every InitMethod (init.hpp:8; local_search.cpp:62-94) --
    def _init(self, method, seed, candidates, oversampling_l, rounds_r, rounds_rule):
        return _Init(int(method), int(candidates), int(oversampling_l), int(rounds_r), int(rounds_rule),
                     _u64(seed))

    def forgy_init(self, X, k, r):
        X = _f64(X)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        self._check(self._fn("forgy_init")(_p(X, _dp), _u64(m), _u64(n), _u64(k), r, _p(Cn, _dp)))
        return Cn

    def kmeans_parallel_init(self, X, k, r, candidates=3, oversampling_l=0, rounds_r=5, rounds_rule=0):
        X = _f64(X)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        cfg = self._init(2, 0, candidates, oversampling_l, rounds_r, rounds_rule)
        ev = _u64(0)
        self._check(self._fn("kmeans_parallel_init")(_p(X, _dp), _u64(m), _u64(n), _u64(k), C.byref(cfg), r,
                                                     _p(Cn, _dp), C.byref(ev)))
        return Cn, int(ev.value)

    def kmeans(self, X, k, method, seed, candidates=3, oversampling_l=0, rounds_r=5, rounds_rule=0,
               max_iterations=300, rel_tolerance=1e-4):
        X = _f64(X)
        m, n = X.shape
        Cn = np.empty((k, n), np.float64)
        mask = np.empty(k, np.uint8)
        labels = np.empty(m, np.int32)
        cfg = self._init(method, seed, candidates, oversampling_l, rounds_r, rounds_rule)
        out = _PortOutcome() if self.kind == "port" else _RefOutcome()
        self._check(self._fn("kmeans")(_p(X, _dp), _u64(m), _u64(n), _u64(k), C.byref(cfg),
                                       _u64(max_iterations), C.c_double(rel_tolerance), _p(Cn, _dp),
                                       _p(mask, _u8p), _p(labels, _i32p), C.byref(out)))
        return BigMeansResult(Cn, mask, labels, float(out.objective), int(out.evals),
                              int(out.iterations), 1)

    def choose_chunk_size_hint(self, X, k, ladder=(), chunks_per_candidate=3, runs_per_candidate=3,
                               max_iterations=300, rel_tolerance=1e-4, candidates=3, seed=123456789):
        """big_means.cpp:114-160.  The port restates the probe loop here over its
        own big_means; the reference calls its library function."""
        X = _f64(X)
        m, n = X.shape
        if self.kind == "ref":
            lad = np.ascontiguousarray(ladder, np.uint64)
            out = _u64(0)
            self._check(self.lib.ref_choose_chunk_size_hint(
                _p(X, _dp), _u64(m), _u64(n), _u64(k), _p(lad, _u64p), _u64(lad.size),
                _u64(chunks_per_candidate), _u64(runs_per_candidate), _u64(max_iterations),
                C.c_double(rel_tolerance), C.c_int(candidates), _u64(seed), C.byref(out)))
            return int(out.value)
        if k < 1 or m < k or chunks_per_candidate < 1 or runs_per_candidate < 1:
            raise OracleError(1, "choose_chunk_size_hint: invalid arguments")  # :117-123
        lad = list(ladder)
        if not lad:  # :125-130
            div = 64
            while div >= 1:
                lad.append(max(k, m // div))
                div //= 2
        lad = sorted(set(min(max(s, k), m) for s in lad))  # clamp, sort, unique :131-135
        best_mean, best_s = float("inf"), lad[0]
        for s in lad:  # :139-157
            tot = 0.0
            for run in range(runs_per_candidate):
                tot += self.big_means(X, k, s, chunks_per_candidate, seed=seed + run,
                                      max_iterations=max_iterations, rel_tolerance=rel_tolerance,
                                      candidates_per_step=candidates).objective
            mean = tot / float(runs_per_candidate)
            if mean < best_mean:
                best_mean, best_s = mean, s
        return best_s

    def set_worker_count(self, n: int):
        if self.kind == "ref":
            self.lib.ref_set_worker_count(C.c_uint(n))

    def io_load(self, path, format="csv", has_header=False, normalize=False, columns=None):
        """The reference's io::load (io.cpp:224-243), "ref" back end only.
        Returns ("ok", values m x n) or (kind, message, line, column) for an error
        (kind: "config" / "state" / "parse" / "other")."""
        if self.kind != "ref":
            raise OracleError(1, "io_load needs the compiled reference")
        lib = self.lib
        lib.ref_io_load.restype = C.c_int
        lib.ref_io_last_error.restype = C.c_char_p
        fmt = {"csv": 0, "whitespace": 1, "tsplib": 2}[format]
        cols = None if columns is None else np.ascontiguousarray(columns, np.uint64)
        out = C.POINTER(C.c_double)()
        m, n, el, ec = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        rc = lib.ref_io_load(str(path).encode(), fmt, int(has_header), int(normalize),
                             None if cols is None else cols.ctypes.data_as(C.POINTER(C.c_uint64)),
                             C.c_uint64(0 if cols is None else cols.size), int(cols is not None),
                             C.byref(out), C.byref(m), C.byref(n), C.byref(el), C.byref(ec))
        if rc != 0:
            kind = {1: "config", 2: "state", 5: "parse"}.get(rc, "other")
            return (kind, lib.ref_io_last_error().decode(), el.value, ec.value)
        size = m.value * n.value
        vals = np.ctypeslib.as_array(out, shape=(size,)).copy() if size else np.empty(0)
        lib.ref_io_free(out)
        return ("ok", vals.reshape(m.value, n.value))


def port() -> Oracle:
    return Oracle("port")


def ref() -> Oracle | None:
    return Oracle("ref") if os.path.exists(REF_SO) else None
