"""World-size-2 gloo test of the multi-GPU exchange (paper_2204_07485_b200/multi.py)
on CPU, with the oracle standing in for each rank's device chain: the
distributed result must equal the serial G-chain oracle bit for bit
(G reference chains with seed+g, min f_opt with lowest-rank ties, then
assign_nearest + block_sum over all rows)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_07485_b200 import multi


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    X = np.random.default_rng(77).normal(size=(5000, 4)) * 4.0
    return X, dict(k=6, s=700, chunks=7, seed=11)  # 7 chunks over 2 ranks: 4 + 3


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import port as oport
    P = oport()
    X, c = _data()

    def chain(seed_g, chunks_g):
        o = P.big_means(X, c["k"], c["s"], chunks_g, seed=seed_g, final_assignment=False)
        return multi.ChainResult(o.centroids, o.mask, o.objective, o.evals, o.iterations, o.chunks)

    def rows(C, mask, r0, r1):
        lab, d, ev = P.assign_nearest(X[r0:r1], C, mask)
        parts = [P.block_sum(d[a:a + 1024]) for a in range(0, r1 - r0, 1024)]
        return np.array(parts), ev

    res = multi.big_means_distributed(X.shape[0], c["k"], X.shape[1], chain, rows, c["seed"], c["chunks"])
    q.put((rank, res.objective, res.centroids.tobytes(), res.winner, res.evals, res.chunks))
    dist.destroy_process_group()


def test_shard_rows_cover_tiles():
    for m in (1, 1023, 1024, 1025, 5000, 2_500_000):
        for world in (1, 2, 3, 8):
            spans = [multi.shard_rows(m, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            assert all(a % 1024 == 0 for a, b in spans if b > a)


def test_chain_chunks_partition():
    for total in (1, 7, 200, 512):
        for world in (1, 2, 3, 8):
            parts = [multi.chain_chunks(total, g, world) for g in range(world)]
            assert sum(parts) == total and max(parts) - min(parts) <= 1
            assert parts == sorted(parts, reverse=True)


def test_select_winner_ties_lowest_rank():
    assert multi.select_winner([3.0, 1.0, 1.0, 2.0]) == 1
    assert multi.select_winner([float("inf"), float("inf")]) == 0


def test_two_rank_exchange_equals_serial_oracle():
    from oracle.oracle import port as oport
    P = oport()
    X, c = _data()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # serial G-chain oracle
    chains = [P.big_means(X, c["k"], c["s"], multi.chain_chunks(c["chunks"], g, world),
                          seed=c["seed"] + g, final_assignment=False) for g in range(world)]
    w = multi.select_winner([o.objective for o in chains])
    lab, d, ev = P.assign_nearest(X, chains[w].centroids, chains[w].mask)
    expected = P.block_sum(d)
    total_evals = sum(o.evals for o in chains) + ev
    for rank, obj, cbytes, winner, evals, chunks in results:
        assert obj == expected
        assert cbytes == chains[w].centroids.tobytes()
        assert winner == w
        assert evals == total_evals and chunks == c["chunks"]
