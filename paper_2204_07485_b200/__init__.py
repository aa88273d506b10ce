"""B200-native Big-means hot path (arXiv 2204.07485).

Drop-in for the reference's `bigmeans::big_means` path: hand-written sm_100a
CUDA kernels behind a C-ABI (include/bigmeans_b200.h), driven from C++ host
code that owns the reference's RNG stream.  This Python package mirrors the
reference C++ API (see api.py) for tests, benchmarks and multi-GPU plumbing.
"""
from .api import (  # noqa: F401
    K_DEFAULT_SEED, K_REDUCTION_BLOCK, BigMeansConfig, BigMeansTrace, Centroids, ChunkRecord,
    ClusteringOutcome, ConfigError, Dataset, DeviceError, EvalCounter, InitConfig, InitMethod, Rng,
    RoundsRule, ChunkHintConfig, choose_chunk_size_hint,
    SearchConfig, StateError, assign_nearest, assign_rows, big_means, big_means_multi, block_sum,
    device_count, load, parse_file, ParseError,
    kmeans, kmeanspp_fill, last_profile, lloyd, objective, sample_chunk, sample_chunk_device,
    set_profiling,
    update_centroids)

__all__ = [n for n in dir() if not n.startswith("_")]
