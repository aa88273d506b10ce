"""Reference-mirror host API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/bigmeans/*.hpp) so that parity tests read like
the reference's own tests:

=========================  ==========================================
reference (file:line)      here
=========================  ==========================================
Dataset core.hpp:16-37     Dataset (device-resident, immutable)
Centroids core.hpp:42-74   Centroids (k x n f64 + degenerate mask)
EvalCounter core.hpp:89    EvalCounter
assign_nearest :112        assign_nearest
objective :118             objective
block_sum :122             block_sum
update_centroids :126      update_centroids
InitConfig init.hpp:14     InitConfig (candidates_per_step, seed)
kmeanspp_fill init.hpp:40  kmeanspp_fill
SearchConfig l_s.hpp:10    SearchConfig
ClusteringOutcome :24      ClusteringOutcome
lloyd l_s.hpp:38           lloyd
kmeans l_s.hpp:44          kmeans (kmeans_pp initialisation)
BigMeansConfig b_m.hpp:11  BigMeansConfig
ChunkRecord/Trace :28-40   ChunkRecord / BigMeansTrace
sample_chunk b_m.hpp:46    sample_chunk
big_means b_m.hpp:56       big_means
=========================  ==========================================

Errors raise ConfigError / StateError like the reference's exceptions.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi

K_DEFAULT_SEED = 123456789  # common.hpp:17
K_REDUCTION_BLOCK = 1024    # threading.hpp:15


class ConfigError(RuntimeError):
    """Invalid configuration (common.hpp:21-24)."""


class StateError(RuntimeError):
    """Operation on an unsupported state (common.hpp:46-49)."""


class DeviceError(RuntimeError):
    """CUDA failure or internal error."""


class ParseError(RuntimeError):
    """Failure while reading external input, with its 1-based line and column
    (common.hpp:28-42)."""

    def __init__(self, what: str, line: int, column: int):
        super().__init__(what)
        self.line = line
        self.column = column


def _check(rc: int) -> None:
    if rc == _capi.BM_OK:
        return
    lib = _capi.load()
    msg = lib.bm_last_error().decode()
    if rc == _capi.BM_CONFIG_ERROR:
        raise ConfigError(msg)
    if rc == _capi.BM_STATE_ERROR:
        raise StateError(msg)
    if rc == _capi.BM_PARSE_ERROR:
        line, col = C.c_uint64(), C.c_uint64()
        lib.bm_last_parse_location(C.byref(line), C.byref(col))
        raise ParseError(msg, line.value, col.value)
    raise DeviceError(msg)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def device_count() -> int:
    n = C.c_int(0)
    _check(_capi.load().bm_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
class Dataset:
    """Immutable m x n matrix, resident on one GPU (core.hpp:13-37).

    values: (m, n) float64 or float32 array.  float32 data is stored as
    float32 on the device and promoted exactly to float64 in every kernel.
    """

    def __init__(self, values, m: Optional[int] = None, n: Optional[int] = None,
                 device: int = 0, _handle=None):
        lib = _capi.load()
        self._lib = lib
        if _handle is not None:
            self._h = _handle
            mm, nn = C.c_uint64(), C.c_uint64()
            _check(lib.bm_dataset_shape(self._h, C.byref(mm), C.byref(nn)))
            self._m, self._n = mm.value, nn.value
            self.device = device
            return
        arr = np.asarray(values)
        if arr.dtype not in (np.float64, np.float32):
            arr = arr.astype(np.float64)
        if m is not None or n is not None:
            if arr.size != (m or 0) * (n or 0):
                raise ConfigError("dataset buffer size does not match m*n")
            arr = arr.reshape(m, n)
        if arr.ndim != 2:
            raise ConfigError("dataset values must be a 2-D array (or flat with m, n)")
        arr = np.ascontiguousarray(arr)
        self._m, self._n = arr.shape
        self.device = device
        h = C.c_void_p()
        dt = _capi.BM_F64 if arr.dtype == np.float64 else _capi.BM_F32
        _check(lib.bm_dataset_create(arr.ctypes.data_as(C.c_void_p), self._m, self._n, dt,
                                     device, C.byref(h)))
        self._h = h

    @property
    def m(self) -> int:
        return self._m

    @property
    def n(self) -> int:
        return self._n

    @property
    def handle(self):
        return self._h

    @property
    def storage(self) -> str:
        """Device storage type ("f64" or "f32"; fp64 input narrows losslessly)."""
        v = C.c_int()
        _check(self._lib.bm_dataset_storage(self._h, C.byref(v)))
        return "f64" if v.value == _capi.BM_F64 else "f32"

    @property
    def exact_sums(self):
        """(exact, exponent): whether every value is a multiple of 2^exponent with
        m * max|x| < 2^52 * 2^exponent, so update sums are exact in any order."""
        a, e = C.c_int32(), C.c_int32()
        _check(self._lib.bm_dataset_sum_mode(self._h, C.byref(a), C.byref(e)))
        return bool(a.value), int(e.value)

    def min_max_normalize(self) -> "Dataset":
        """io::min_max_normalize (io.cpp:245-264) on the device: a new dataset."""
        h = C.c_void_p()
        _check(self._lib.bm_dataset_min_max_normalize(self._h, C.byref(h)))
        return Dataset(None, device=self.device, _handle=h)

    def gather(self, rows) -> "Dataset":
        """New dataset holding the listed rows in the listed order (core.cpp:34-44)."""
        idx = np.ascontiguousarray(rows, dtype=np.uint64)
        h = C.c_void_p()
        _check(self._lib.bm_dataset_gather(self._h, _ptr(idx, _capi.P_u64), idx.size, C.byref(h)))
        return Dataset(None, device=self.device, _handle=h)

    def values(self) -> np.ndarray:
        out = np.empty((self._m, self._n), np.float64)
        _check(self._lib.bm_dataset_download(self._h, _ptr(out, _capi.P_dbl)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.bm_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Rng:
    """std::mt19937_64 (common.hpp:13), owned by the host."""

    def __init__(self, seed: int = K_DEFAULT_SEED):
        self._lib = _capi.load()
        h = C.c_void_p()
        _check(self._lib.bm_rng_create(seed, C.byref(h)))
        self._h = h

    def __call__(self) -> int:
        return int(self._lib.bm_rng_next(self._h))

    def uniform_int(self, a: int, b: int) -> int:
        """std::uniform_int_distribution<size_t>(a, b)(rng)."""
        return int(self._lib.bm_rng_uniform_int(self._h, a, b))

    def uniform_real(self, a: float, b: float) -> float:
        """std::uniform_real_distribution<double>(a, b)(rng)."""
        return float(self._lib.bm_rng_uniform_real(self._h, a, b))

    def __del__(self):
        try:
            self._lib.bm_rng_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------------------
class Centroids:
    """k x n centers + degeneracy mask (core.hpp:42-74)."""

    def __init__(self, values: np.ndarray, mask: np.ndarray):
        self.values = np.ascontiguousarray(values, np.float64)
        self.mask = np.ascontiguousarray(mask, np.uint8)
        self.values[self.mask.astype(bool)] = 0.0

    @staticmethod
    def all_degenerate(k: int, n: int) -> "Centroids":
        if k < 1 or n < 1:
            raise ConfigError("centroids must have at least one row and one column")
        return Centroids(np.zeros((k, n)), np.ones(k, np.uint8))

    @staticmethod
    def from_rows(values, k: Optional[int] = None, n: Optional[int] = None) -> "Centroids":
        v = np.asarray(values, np.float64)
        if k is not None:
            if v.size != k * n:
                raise ConfigError("centroid buffer size does not match k*n")
            v = v.reshape(k, n)
        if not np.isfinite(v).all():
            raise ConfigError("non-degenerate centroid rows must be finite")
        return Centroids(v.copy(), np.zeros(v.shape[0], np.uint8))

    @property
    def k(self) -> int:
        return self.values.shape[0]

    @property
    def n(self) -> int:
        return self.values.shape[1]

    def row(self, j: int) -> np.ndarray:
        return self.values[j]

    def set_row(self, j: int, row) -> None:
        self.values[j] = np.asarray(row, np.float64)
        self.mask[j] = 0

    def degenerate(self, j: int) -> bool:
        return bool(self.mask[j])

    def mark_degenerate(self, j: int) -> None:
        self.mask[j] = 1

    def degenerate_count(self) -> int:
        return int(self.mask.sum())

    def active_count(self) -> int:
        return self.k - self.degenerate_count()

    def copy(self) -> "Centroids":
        return Centroids(self.values.copy(), self.mask.copy())

    def __eq__(self, other) -> bool:  # operator== = default (core.hpp:67), bitwise
        return (isinstance(other, Centroids) and self.values.shape == other.values.shape
                and np.array_equal(self.values.view(np.uint64), other.values.view(np.uint64))
                and np.array_equal(self.mask, other.mask))


@dataclass
class EvalCounter:
    """core.hpp:89-101."""
    distance_evals: int = 0
    iterations: int = 0
    cpu_init: float = 0.0
    cpu_full: float = 0.0

    def merge(self, o: "EvalCounter") -> None:
        self.distance_evals += o.distance_evals
        self.iterations += o.iterations
        self.cpu_init += o.cpu_init
        self.cpu_full += o.cpu_full


class InitMethod:
    """init.hpp:8 (enum values as in the reference)."""
    forgy = 0
    kmeans_pp = 1
    kmeans_parallel = 2


class RoundsRule:
    """init.hpp:10-13."""
    fixed = 0
    log_phi = 1


@dataclass
class InitConfig:
    """init.hpp:16-27."""
    candidates_per_step: int = 3
    seed: int = K_DEFAULT_SEED
    method: int = InitMethod.kmeans_pp
    oversampling_l: int = 0
    rounds_r: int = 5
    rounds_rule: int = RoundsRule.fixed


@dataclass
class SearchConfig:
    """local_search.hpp:10-16."""
    max_iterations: int = 300
    rel_tolerance: float = 1e-4
    seed: int = K_DEFAULT_SEED


@dataclass
class ClusteringOutcome:
    """local_search.hpp:24-30."""
    centroids: Centroids
    assignment: np.ndarray
    objective: float = 0.0
    objective_history: list = field(default_factory=list)
    counter: EvalCounter = field(default_factory=EvalCounter)


@dataclass
class BigMeansConfig:
    """big_means.hpp:11-26."""
    k: int = 0
    chunk_size: int = 0
    max_cpu_seconds: Optional[float] = None
    max_chunks: Optional[int] = None
    search: SearchConfig = field(default_factory=SearchConfig)
    init: InitConfig = field(default_factory=InitConfig)
    seed: int = K_DEFAULT_SEED
    final_assignment: bool = True


@dataclass
class ChunkRecord:
    """big_means.hpp:28-34."""
    chunk_index: int
    candidate_objective: float
    incumbent_objective: float
    accepted: bool
    degenerate_repaired: int


@dataclass
class BigMeansTrace:
    """big_means.hpp:36-40."""
    records: list = field(default_factory=list)

    def chunks(self) -> int:
        return len(self.records)


# ---------------------------------------------------------------------------
def _cent_args(cent: Centroids):
    return _ptr(cent.values, _capi.P_dbl), _ptr(cent.mask, _capi.P_u8), cent.k


def assign_nearest(data: Dataset, cent: Centroids, counter: Optional[EvalCounter] = None):
    """core.hpp:112-114 -> (labels int32[m], dists f64[m])."""
    if cent.n != data.n:
        raise ConfigError("assign_nearest: dataset and centroid widths differ")
    labels = np.empty(data.m, np.int32)
    dists = np.empty(data.m, np.float64)
    ev = C.c_uint64(0)
    cv, cm, k = _cent_args(cent)
    _check(_capi.load().bm_assign_nearest(data.handle, cv, cm, k, _ptr(labels, _capi.P_i32),
                                          _ptr(dists, _capi.P_dbl), C.byref(ev)))
    if counter is not None:
        counter.distance_evals += ev.value
    return labels, dists


def objective(data: Dataset, cent: Centroids, counter: Optional[EvalCounter] = None) -> float:
    """core.hpp:118."""
    if cent.n != data.n:
        raise ConfigError("assign_nearest: dataset and centroid widths differ")
    out = C.c_double()
    ev = C.c_uint64(0)
    cv, cm, k = _cent_args(cent)
    _check(_capi.load().bm_objective(data.handle, cv, cm, k, C.byref(out), C.byref(ev)))
    if counter is not None:
        counter.distance_evals += ev.value
    return out.value


def block_sum(values, device: int = 0) -> float:
    """core.hpp:122."""
    v = np.ascontiguousarray(values, np.float64)
    out = C.c_double()
    _check(_capi.load().bm_block_sum(_ptr(v, _capi.P_dbl), v.size, device, C.byref(out)))
    return out.value


def update_centroids(data: Dataset, labels, k: int) -> Centroids:
    """core.hpp:126."""
    lab = np.ascontiguousarray(labels, np.int32)
    if lab.size != data.m:
        raise ConfigError("update_centroids: assignment length does not match dataset")
    cv = np.empty((k, data.n), np.float64)
    cm = np.empty(k, np.uint8)
    _check(_capi.load().bm_update_centroids(data.handle, _ptr(lab, _capi.P_i32), k,
                                            _ptr(cv, _capi.P_dbl), _ptr(cm, _capi.P_u8)))
    return Centroids(cv, cm)


def sample_chunk(data: Dataset, s: int, rng: Rng) -> np.ndarray:
    """big_means.hpp:46 -> s ascending distinct indices (uint64)."""
    if s < 1 or s > data.m:
        raise ConfigError("sample_chunk: chunk size must be in [1, m]")
    out = np.empty(s, np.uint64)
    _check(_capi.load().bm_sample_chunk(data.handle, s, rng._h, _ptr(out, _capi.P_u64)))
    return out


def sample_chunk_device(data: Dataset, s: int, rng: Rng, force_sequential: bool = False) -> np.ndarray:
    """sample_chunk with the draws made on the device from rng's stream (the
    path big_means takes); rng advances exactly like the host draws."""
    out = np.empty(s, np.uint64)
    _check(_capi.load().bm_sample_chunk_device(data.handle, s, rng._h, int(force_sequential),
                                               _ptr(out, _capi.P_u64)))
    return out


def kmeanspp_fill(pool: Dataset, cent: Centroids, cfg: InitConfig, rng,
                  counter: Optional[EvalCounter] = None) -> Centroids:
    """init.hpp:40-43.  rng: Rng, or an int seed (the seed overload)."""
    if pool.n != cent.n:
        raise ConfigError("kmeanspp_fill: pool and centroid widths differ")
    if not isinstance(rng, Rng):
        rng = Rng(int(rng))
    out = cent.copy()
    ev = C.c_uint64(0)
    _check(_capi.load().bm_kmeanspp_fill(pool.handle, _ptr(out.values, _capi.P_dbl),
                                         _ptr(out.mask, _capi.P_u8), out.k,
                                         cfg.candidates_per_step, rng._h, C.byref(ev)))
    if counter is not None:
        counter.distance_evals += ev.value
    return out


def lloyd(data: Dataset, start: Centroids, cfg: SearchConfig = SearchConfig(),
          accumulate: Optional[EvalCounter] = None) -> ClusteringOutcome:
    """local_search.hpp:38-39."""
    if start.n != data.n:
        raise ConfigError("assign_nearest: dataset and centroid widths differ")
    cent = start.copy()
    labels = np.empty(data.m, np.int32)
    cap = int(cfg.max_iterations) + 1
    hist = np.empty(max(cap, 1), np.float64)
    hl, obj, ev, it = C.c_uint64(), C.c_double(), C.c_uint64(), C.c_uint64()
    _check(_capi.load().bm_lloyd(data.handle, _ptr(cent.values, _capi.P_dbl),
                                 _ptr(cent.mask, _capi.P_u8), cent.k, int(cfg.max_iterations),
                                 float(cfg.rel_tolerance), _ptr(labels, _capi.P_i32),
                                 _ptr(hist, _capi.P_dbl), cap, C.byref(hl), C.byref(obj),
                                 C.byref(ev), C.byref(it)))
    counter = EvalCounter(ev.value, it.value)
    if accumulate is not None:
        accumulate.distance_evals += ev.value
        accumulate.iterations += it.value
    return ClusteringOutcome(cent, labels, obj.value, list(hist[:hl.value]), counter)


def kmeans(data: Dataset, k: int, init: InitConfig = InitConfig(),
           search: SearchConfig = SearchConfig()) -> ClusteringOutcome:
    """kmeans local_search.hpp:44 / local_search.cpp:62-94 with init.method
    (forgy, kmeans_pp or kmeans_parallel) seeded by init.seed, then lloyd."""
    cv = np.empty((k, data.n), np.float64)
    cm = np.empty(k, np.uint8)
    labels = np.empty(data.m, np.int32)
    out = _capi.bm_outcome()
    out.centroids = _ptr(cv, _capi.P_dbl)
    out.mask = _ptr(cm, _capi.P_u8)
    out.labels = _ptr(labels, _capi.P_i32)
    ic = _capi.bm_init_config(int(init.method), int(init.candidates_per_step), int(init.oversampling_l),
                              int(init.rounds_r), int(init.rounds_rule), int(init.seed))
    _check(_capi.load().bm_kmeans(data.handle, k, C.byref(ic), int(search.max_iterations),
                                  float(search.rel_tolerance), C.byref(out)))
    counter = EvalCounter(out.distance_evals, out.iterations, out.cpu_init, out.cpu_full)
    return ClusteringOutcome(Centroids(cv, cm), labels, out.objective, [], counter)


@dataclass
class ChunkHintConfig:
    """big_means.hpp:60-68."""
    ladder: list = field(default_factory=list)
    chunks_per_candidate: int = 3
    runs_per_candidate: int = 3
    search: SearchConfig = field(default_factory=SearchConfig)
    init: InitConfig = field(default_factory=InitConfig)
    seed: int = K_DEFAULT_SEED


def choose_chunk_size_hint(data: Dataset, k: int, cfg: ChunkHintConfig = ChunkHintConfig()) -> int:
    """big_means.hpp:72-73 / big_means.cpp:114-160: the ladder size with the best
    mean final objective over short big_means probes (ties: the smaller size)."""
    lad = np.ascontiguousarray(cfg.ladder, np.uint64)
    out = C.c_uint64()
    mean = C.c_double()
    _check(_capi.load().bm_choose_chunk_size_hint(
        data.handle, int(k), _ptr(lad, _capi.P_u64) if lad.size else None, lad.size,
        int(cfg.chunks_per_candidate), int(cfg.runs_per_candidate), int(cfg.search.max_iterations),
        float(cfg.search.rel_tolerance), int(cfg.init.candidates_per_step), int(cfg.seed),
        C.byref(out), C.byref(mean)))
    return int(out.value)


def _native_config(cfg: BigMeansConfig) -> _capi.bm_config:
    c = _capi.bm_config()
    _capi.load().bm_config_init(C.byref(c))
    c.k = int(cfg.k)
    c.chunk_size = int(cfg.chunk_size)
    if cfg.max_cpu_seconds is not None:
        c.has_max_cpu_seconds = 1
        c.max_cpu_seconds = float(cfg.max_cpu_seconds)
    if cfg.max_chunks is not None:
        if int(cfg.max_chunks) < 1:
            raise ConfigError("big_means: max_chunks must be at least 1")
        c.has_max_chunks = 1
        c.max_chunks = int(cfg.max_chunks)
    c.max_iterations = int(cfg.search.max_iterations)
    c.rel_tolerance = float(cfg.search.rel_tolerance)
    c.candidates_per_step = int(cfg.init.candidates_per_step)
    c.seed = int(cfg.seed)
    c.final_assignment = 1 if cfg.final_assignment else 0
    return c


def big_means(data: Dataset, cfg: BigMeansConfig, want_labels: bool = True):
    """big_means.hpp:56-57 -> (ClusteringOutcome, BigMeansTrace).

    want_labels=False keeps the final assignment on the device (the outcome's
    assignment is then empty), which is what device-resident benchmarks use.
    """
    if cfg.k < 1:
        raise ConfigError("big_means: k must be at least 1")
    c = _native_config(cfg)
    k = int(cfg.k)
    cv = np.empty((k, data.n), np.float64)
    cm = np.empty(k, np.uint8)
    labels = np.empty(data.m, np.int32) if (cfg.final_assignment and want_labels) else None
    out = _capi.bm_outcome()
    out.centroids = _ptr(cv, _capi.P_dbl)
    out.mask = _ptr(cm, _capi.P_u8)
    out.labels = _ptr(labels, _capi.P_i32)
    lib = _capi.load()
    _check(lib.bm_big_means(data.handle, C.byref(c), C.byref(out), None, 0))
    nrec = C.c_uint64(0)  # the whole trace, sized from the result (time budgets included)
    _check(lib.bm_last_trace(None, 0, C.byref(nrec)))
    recs = (_capi.bm_chunk_record * max(nrec.value, 1))()
    _check(lib.bm_last_trace(recs, nrec.value, C.byref(nrec)))
    trace = BigMeansTrace([ChunkRecord(int(r.chunk_index), float(r.candidate_objective),
                                       float(r.incumbent_objective), bool(r.accepted),
                                       int(r.degenerate_repaired))
                           for r in recs[:nrec.value]])
    counter = EvalCounter(out.distance_evals, out.iterations, out.cpu_init, out.cpu_full)
    asg = labels if labels is not None else np.empty(0, np.int32)
    return ClusteringOutcome(Centroids(cv, cm), asg, out.objective, [], counter), trace


_FORMATS = {"csv": 0, "whitespace": 1, "tsplib": 2}  # io::parse_format io.cpp:198-209


def _format_id(fmt: str) -> int:
    if fmt not in _FORMATS:
        raise ConfigError(f"unknown dataset format '{fmt}'")
    return _FORMATS[fmt]


def parse_file(path: str, format: str = "csv", has_header: bool = False, columns=None,
               threads: int = 0) -> np.ndarray:
    """The host half of io::load (io.cpp:224-243): the parsed (and column-selected)
    m x n float64 matrix, parsed natively in parallel; the reference's errors."""
    lib = _capi.load()
    cols = None if columns is None else np.ascontiguousarray(columns, np.uint64)
    out = _capi.P_dbl()
    m, n = C.c_uint64(), C.c_uint64()
    _check(lib.bm_parse_file(str(path).encode(), _format_id(format), int(has_header), _ptr(cols, _capi.P_u64),
                             0 if cols is None else cols.size, threads, C.byref(out), C.byref(m), C.byref(n)))
    try:
        arr = np.ctypeslib.as_array(out, shape=(m.value * n.value,)).copy() if m.value * n.value else np.empty(0)
    finally:
        lib.bm_free_values(out)
    return arr.reshape(m.value, n.value)


def load(path: str, format: str = "csv", has_header: bool = False, normalize: bool = False, columns=None,
         device: int = 0, threads: int = 0) -> Dataset:
    """io::load (io.hpp:31-37, DatasetSpec io.hpp:18-25) straight to a device
    Dataset: native parallel parse, upload, and the min-max normalisation
    (io.cpp:245-264) on the device."""
    lib = _capi.load()
    cols = None if columns is None else np.ascontiguousarray(columns, np.uint64)
    h = C.c_void_p()
    _check(lib.bm_dataset_load(str(path).encode(), _format_id(format), int(has_header), int(normalize),
                               _ptr(cols, _capi.P_u64), 0 if cols is None else cols.size, threads, device,
                               C.byref(h)))
    return Dataset(None, device=device, _handle=h)


def big_means_multi(datasets, cfg: BigMeansConfig, want_labels: bool = True):
    """Multi-GPU big_means in one process (bm_big_means_multi): chain g on
    datasets[g] (the same matrix, normally one handle per GPU) with seed + g and
    floor(N/G) (+1 for g < N mod G) of cfg.max_chunks = N chunks, lowest-index
    minimum f_opt wins, final pass row-sharded over the devices.
    Returns (ClusteringOutcome, BigMeansTrace, chain_chunks, winner)."""
    G = len(datasets)
    if G < 1:
        raise ConfigError("big_means_multi: at least one chain")
    c = _native_config(cfg)
    k, m, n = int(cfg.k), datasets[0].m, datasets[0].n
    cv = np.empty((k, n), np.float64)
    cm = np.empty(k, np.uint8)
    labels = np.empty(m, np.int32) if (cfg.final_assignment and want_labels) else None
    out = _capi.bm_outcome()
    out.centroids = _ptr(cv, _capi.P_dbl)
    out.mask = _ptr(cm, _capi.P_u8)
    out.labels = _ptr(labels, _capi.P_i32)
    cap = int(cfg.max_chunks) if cfg.max_chunks is not None else 1 << 16
    recs = (_capi.bm_chunk_record * max(cap, 1))()
    handles = (C.c_void_p * G)(*[d.handle for d in datasets])
    counts = np.zeros(G, np.uint64)
    winner = C.c_int32(-1)
    _check(_capi.load().bm_big_means_multi(handles, G, C.byref(c), C.byref(out), recs, cap,
                                           _ptr(counts, _capi.P_u64), C.byref(winner)))
    nrec = min(int(out.chunks), cap)
    trace = BigMeansTrace([ChunkRecord(int(r.chunk_index), float(r.candidate_objective),
                                       float(r.incumbent_objective), bool(r.accepted),
                                       int(r.degenerate_repaired)) for r in recs[:nrec]])
    counter = EvalCounter(out.distance_evals, out.iterations, out.cpu_init, out.cpu_full)
    asg = labels if labels is not None else np.empty(0, np.int32)
    return (ClusteringOutcome(Centroids(cv, cm), asg, out.objective, [], counter), trace,
            [int(x) for x in counts], int(winner.value))


def assign_rows(data: Dataset, cent: Centroids, row_begin: int, row_end: int,
                want_labels: bool = False):
    """Row-sharded final pass (multi-GPU): (labels or None, tile partials, evals)."""
    r = row_end - row_begin
    labels = np.empty(max(r, 0), np.int32) if want_labels else None
    tiles = np.empty(max((r + K_REDUCTION_BLOCK - 1) // K_REDUCTION_BLOCK, 1), np.float64)
    ev = C.c_uint64(0)
    cv, cm, k = _cent_args(cent)
    _check(_capi.load().bm_assign_rows(data.handle, cv, cm, k, row_begin, row_end,
                                       _ptr(labels, _capi.P_i32), _ptr(tiles, _capi.P_dbl),
                                       C.byref(ev)))
    return labels, tiles[:(r + K_REDUCTION_BLOCK - 1) // K_REDUCTION_BLOCK], ev.value


def set_profiling(enabled: bool) -> None:
    _check(_capi.load().bm_set_profiling(1 if enabled else 0))


def last_profile() -> dict:
    p = _capi.bm_profile()
    _check(_capi.load().bm_last_profile(C.byref(p)))
    out = {f: getattr(p, f) for f, _ in p._fields_}
    names = ["assign", "final", "update", "sample", "gather", "kmeanspp", "control"]
    out["phase_ms"] = {nm: out["phase_ms"][i] for i, nm in enumerate(names)}
    out["phase_count"] = {nm: int(out["phase_count"][i]) for i, nm in enumerate(names)}
    return out
