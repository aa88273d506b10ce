"""Multi-GPU Big-means: one independent subproblem chain per rank.

This is the paper's parallel mode 2 (the reference implements
only mode 1).  The N = cfg.max_chunks subproblems are sharded over
the G ranks (strong scaling): rank g runs big_means with seed + g
and floor(N/G) (+1 for g < N mod G) chunks on the replicated dataset, then the
ranks exchange exactly three small messages:

1. all_gather of (f_opt_g): the winner is the first rank with the minimum
   (strict < scanning ranks in order -> ties go to the lowest rank);
2. broadcast of the winner's k x n f64 centroids + k mask bytes;
3. the final pass is row-sharded on 1024-row tile boundaries and the
   per-tile partial sums are all_gathered and folded left to right, which is
   bit-identical to block_sum over all m rows (core.cpp:163-175), unlike an
   all-reduce whose order is unspecified.

The exchange is written against torch.distributed (NCCL on GPUs, gloo on CPU
for tests) with injectable `chain` / `rows` callables, so the same logic is
exercised on CPU with a host-side stand-in for the device engine.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

TILE = 1024


@dataclass
class ChainResult:
    centroids: np.ndarray  # k x n f64
    mask: np.ndarray       # k u8
    f_opt: float
    evals: int
    iterations: int
    chunks: int


@dataclass
class DistributedResult:
    centroids: np.ndarray
    mask: np.ndarray
    objective: float
    winner: int
    f_opts: list
    evals: int          # all ranks: chain evals + final-pass evals
    chunks: int         # all ranks
    iterations: int     # all ranks
    local_evals: int
    local_chunks: int


def shard_rows(m: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of rank `rank`: contiguous whole 1024-row tiles."""
    tiles = (m + TILE - 1) // TILE
    per, rem = divmod(tiles, world)
    t0 = rank * per + min(rank, rem)
    t1 = t0 + per + (1 if rank < rem else 0)
    return min(m, t0 * TILE), min(m, t1 * TILE)


def chain_chunks(total: int, rank: int, world: int) -> int:
    """Chunks of chain `rank`: floor(N/G), plus one for the first N mod G chains."""
    return total // world + (1 if rank < total % world else 0)


def select_winner(f_opts) -> int:
    best, w = float("inf"), 0
    for g, f in enumerate(f_opts):
        if f < best:  # strict: lowest rank wins ties
            best, w = f, g
    return w


def fold_tiles(parts) -> float:
    total = 0.0
    for p in parts:
        for t in np.asarray(p, np.float64):
            total += float(t)  # left fold in row order (core.cpp:172)
    return total


def big_means_distributed(m: int, k: int, n: int, chain: Callable[[int, int], ChainResult],
                          rows: Callable[[np.ndarray, np.ndarray, int, int], tuple],
                          seed: int, total_chunks: int,
                          device: torch.device | str = "cpu") -> DistributedResult:
    """chain(seed_g, chunks_g) runs this rank's chain (final_assignment off);
    rows(C, mask, r0, r1) -> (tile partials f64[ceil((r1-r0)/1024)], evals)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    cg = chain_chunks(total_chunks, rank, world)
    if cg > 0:
        local = chain(seed + rank, cg)
    else:  # more ranks than chunks: this rank has no chain
        local = ChainResult(np.zeros((k, n)), np.ones(k, np.uint8), float("inf"), 0, 0, 0)
    # 1. select
    f = torch.tensor([local.f_opt], dtype=torch.float64, device=device)
    fs = [torch.empty_like(f) for _ in range(world)]
    dist.all_gather(fs, f)
    f_opts = [float(t.item()) for t in fs]
    winner = select_winner(f_opts)
    # 2. broadcast the winner's incumbent
    C = torch.from_numpy(np.ascontiguousarray(local.centroids, np.float64)).to(device)
    M = torch.from_numpy(np.ascontiguousarray(local.mask, np.uint8)).to(device)
    dist.broadcast(C, src=winner)
    dist.broadcast(M, src=winner)
    Cn = C.cpu().numpy().reshape(k, n)
    Mn = M.cpu().numpy()
    # 3. sharded final pass + ordered fold of all tile partials
    r0, r1 = shard_rows(m, rank, world)
    parts, fin_evals = rows(Cn, Mn, r0, r1) if r1 > r0 else (np.zeros(0), 0)
    max_tiles = (m + TILE - 1) // TILE // world + 1
    buf = torch.full((max_tiles + 1,), float("nan"), dtype=torch.float64, device=device)
    buf[0] = float(len(parts))
    if len(parts):
        buf[1:1 + len(parts)] = torch.from_numpy(np.asarray(parts, np.float64)).to(device)
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    ordered = []
    for b in bufs:
        b = b.cpu().numpy()
        ordered.append(b[1:1 + int(b[0])])
    objective = fold_tiles(ordered)
    # totals
    stats = torch.tensor([local.evals + fin_evals, local.chunks, local.iterations],
                         dtype=torch.float64, device=device)
    dist.all_reduce(stats)
    return DistributedResult(Cn, Mn, objective, winner, f_opts, int(stats[0].item()),
                             int(stats[1].item()), int(stats[2].item()),
                             local.evals + fin_evals, local.chunks)


# ---------------------------------------------------------------------------
# Device engine bindings (the product path on GPUs).
# ---------------------------------------------------------------------------
def gpu_chain(data, cfg):
    """chain callable over the C-ABI: big_means on this rank's device."""
    from . import api

    def run(seed_g: int, chunks_g: int) -> ChainResult:
        out, trace = api.big_means(data, replace(cfg, seed=seed_g, max_chunks=chunks_g,
                                                  final_assignment=False))
        return ChainResult(out.centroids.values, out.centroids.mask, out.objective,
                           out.counter.distance_evals, out.counter.iterations, trace.chunks())
    return run


def gpu_rows(data):
    from . import api

    def run(C, mask, r0, r1):
        _, tiles, ev = api.assign_rows(data, api.Centroids(C, mask), r0, r1)
        return tiles, ev
    return run
