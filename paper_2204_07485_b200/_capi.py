"""ctypes declarations of the C-ABI in include/bigmeans_b200.h.

The shared library is the product: if it is missing the import fails loudly
(there is no CPU fallback of any kind).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BM_LIB_PATH: an alternative build of the same library (A/B diagnostics only)
LIB_PATH = os.environ.get("BM_LIB_PATH") or os.path.join(HERE, "_lib", "libbigmeans_b200.so")

u64 = C.c_uint64
i32 = C.c_int32
dbl = C.c_double
vp = C.c_void_p
P_dbl = C.POINTER(C.c_double)
P_u8 = C.POINTER(C.c_uint8)
P_i32 = C.POINTER(C.c_int32)
P_u64 = C.POINTER(C.c_uint64)

BM_OK, BM_CONFIG_ERROR, BM_STATE_ERROR, BM_CUDA_ERROR, BM_INTERNAL_ERROR, BM_PARSE_ERROR = range(6)
BM_FORMAT_CSV, BM_FORMAT_WHITESPACE, BM_FORMAT_TSPLIB = range(3)
BM_F64, BM_F32 = 0, 1


class bm_config(C.Structure):
    _fields_ = [("k", u64), ("chunk_size", u64), ("has_max_cpu_seconds", i32),
                ("max_cpu_seconds", dbl), ("has_max_chunks", i32), ("max_chunks", u64),
                ("max_iterations", u64), ("rel_tolerance", dbl),
                ("candidates_per_step", i32), ("seed", u64), ("final_assignment", i32)]


class bm_init_config(C.Structure):  # InitConfig init.hpp:16-27
    _fields_ = [("method", C.c_int32), ("candidates_per_step", C.c_int32), ("oversampling_l", C.c_int32),
                ("rounds_r", C.c_int32), ("rounds_rule", C.c_int32), ("seed", C.c_uint64)]


class bm_outcome(C.Structure):
    _fields_ = [("centroids", P_dbl), ("mask", P_u8), ("labels", P_i32), ("objective", dbl),
                ("distance_evals", u64), ("iterations", u64), ("cpu_init", dbl),
                ("cpu_full", dbl), ("chunks", u64)]


class bm_chunk_record(C.Structure):
    _fields_ = [("chunk_index", u64), ("candidate_objective", dbl),
                ("incumbent_objective", dbl), ("accepted", u64), ("degenerate_repaired", u64)]


class bm_profile(C.Structure):
    _fields_ = [("assign_ms_total", dbl), ("assign_launches", u64),
                ("assign_rows_total", u64), ("kernel_launches", u64), ("final_ms", dbl),
                ("final_rows", u64), ("screen_candidates", u64), ("screen_rows", u64),
                ("phase_ms", dbl * 8), ("phase_count", u64 * 8),
                ("chunk_ms_total", dbl), ("chunk_launches", u64), ("chunk_assign_passes", u64),
                ("chunk_update_passes", u64), ("chunk_rows", u64), ("chunk_gap_ms_total", dbl)]


# name -> (restype, argtypes)
PROTOS = {
    "bm_last_error": (C.c_char_p, []),
    "bm_abi_version": (C.c_int, []),
    "bm_config_init": (None, [C.POINTER(bm_config)]),
    "bm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "bm_dataset_create": (C.c_int, [vp, u64, u64, C.c_int, C.c_int, C.POINTER(vp)]),
    "bm_dataset_destroy": (C.c_int, [vp]),
    "bm_dataset_shape": (C.c_int, [vp, P_u64, P_u64]),
    "bm_dataset_storage": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "bm_dataset_sum_mode": (C.c_int, [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "bm_dataset_gather": (C.c_int, [vp, P_u64, u64, C.POINTER(vp)]),
    "bm_dataset_min_max_normalize": (C.c_int, [vp, C.POINTER(vp)]),
    "bm_dataset_download": (C.c_int, [vp, P_dbl]),
    "bm_rng_create": (C.c_int, [u64, C.POINTER(vp)]),
    "bm_rng_destroy": (C.c_int, [vp]),
    "bm_rng_next": (u64, [vp]),
    "bm_rng_uniform_int": (u64, [vp, u64, u64]),
    "bm_rng_uniform_real": (dbl, [vp, dbl, dbl]),
    "bm_sample_chunk_device": (C.c_int, [vp, u64, vp, C.c_int, P_u64]),
    "bm_sample_chunk": (C.c_int, [vp, u64, vp, P_u64]),
    "bm_sample_chunk_draws": (C.c_int, [u64, u64, C.POINTER(C.c_uint32), C.c_int, P_u64]),
    "bm_assign_nearest": (C.c_int, [vp, P_dbl, P_u8, u64, P_i32, P_dbl, P_u64]),
    "bm_objective": (C.c_int, [vp, P_dbl, P_u8, u64, P_dbl, P_u64]),
    "bm_block_sum": (C.c_int, [P_dbl, u64, C.c_int, P_dbl]),
    "bm_update_centroids": (C.c_int, [vp, P_i32, u64, P_dbl, P_u8]),
    "bm_kmeanspp_fill": (C.c_int, [vp, P_dbl, P_u8, u64, i32, vp, P_u64]),
    "bm_lloyd": (C.c_int, [vp, P_dbl, P_u8, u64, u64, dbl, P_i32, P_dbl, u64, P_u64, P_dbl,
                           P_u64, P_u64]),
    "bm_kmeans_pp": (C.c_int, [vp, u64, i32, u64, u64, dbl, C.POINTER(bm_outcome)]),
    "bm_kmeans": (C.c_int, [vp, u64, C.POINTER(bm_init_config), u64, dbl, C.POINTER(bm_outcome)]),
    "bm_init_centroids": (C.c_int, [vp, u64, C.POINTER(bm_init_config), P_dbl, C.POINTER(C.c_uint8), P_u64]),
    "bm_last_trace": (C.c_int, [C.POINTER(bm_chunk_record), u64, P_u64]),
    "bm_dataset_load": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, P_u64, u64, C.c_int32, C.c_int,
                                  C.POINTER(vp)]),
    "bm_parse_file": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, P_u64, u64, C.c_int32, C.POINTER(P_dbl), P_u64,
                                P_u64]),
    "bm_free_values": (None, [P_dbl]),
    "bm_last_parse_location": (C.c_int, [P_u64, P_u64]),
    "bm_big_means_multi": (C.c_int, [C.POINTER(vp), C.c_int32, C.POINTER(bm_config), C.POINTER(bm_outcome),
                                     C.POINTER(bm_chunk_record), u64, P_u64, C.POINTER(C.c_int32)]),
    "bm_choose_chunk_size_hint": (C.c_int, [vp, u64, P_u64, u64, u64, u64, u64, dbl, i32, u64, P_u64, P_dbl]),
    "bm_big_means": (C.c_int, [vp, C.POINTER(bm_config), C.POINTER(bm_outcome),
                               C.POINTER(bm_chunk_record), u64]),
    "bm_assign_rows": (C.c_int, [vp, P_dbl, P_u8, u64, u64, u64, P_i32, P_dbl, P_u64]),
    "bm_set_profiling": (C.c_int, [C.c_int]),
    "bm_debug_ktrace": (C.c_int, [P_u64, u64]),
    "bm_last_profile": (C.c_int, [C.POINTER(bm_profile)]),
    "bm_debug_chunk_phases": (C.c_int, [P_u64]),
    "bm_debug_wide_stamps": (C.c_int, [P_u64]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_2204_07485_b200.build); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOS.items():
        f = getattr(lib, name)  # AttributeError here = ABI mismatch
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def symbols_declared_in_header() -> list[str]:
    """Every function name declared in include/bigmeans_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "bigmeans_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(bm_[a-z_0-9]+)\s*\(", text)))
