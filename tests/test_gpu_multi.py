"""Multi-GPU Big-means (paper mode 2) on the device, bitwise
against the G-chain oracle: G reference chains with seed + g and
floor(N/G) (+1 for g < N mod G) of the N chunks, no final pass each; the
lowest-index minimum f_opt wins; then assign_nearest + block_sum over all
rows with the winner's centroids.

* bm_big_means_multi (one process, one host thread per device): here with
  every chain on cuda:0 (the driver's GPU tier has one GPU), which runs the
  chains of one device one after the other on that device's thread.
* multi.big_means_distributed over torch.distributed with the real device
  chain (gpu_chain / gpu_rows): two processes on cuda:0, gloo exchange."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2204_07485_b200 as bm
from paper_2204_07485_b200 import multi

from conftest import bits

pytestmark = pytest.mark.gpu


def _oracle(P, X, k, s, N, seed, G):
    chains = [P.big_means(X, k, s, multi.chain_chunks(N, g, G), seed=seed + g, final_assignment=False)
              for g in range(G)]
    w = multi.select_winner([o.objective for o in chains])
    lab, d, ev = P.assign_nearest(X, chains[w].centroids, chains[w].mask)
    return chains, w, lab, P.block_sum(d), sum(o.evals for o in chains) + ev


@pytest.mark.parametrize("G,N,case", [(2, 8, "real"), (3, 7, "int"), (4, 9, "f32")])
def test_big_means_multi_vs_g_chain_oracle(port, G, N, case):
    rng = np.random.default_rng(40 + G)
    X = rng.normal(size=(9000, 7)) * 3.0 + rng.integers(0, 4, (9000, 1)) * 6.0
    if case == "int":
        X = np.rint(X)
    if case == "f32":
        X = X.astype(np.float32)
    k, s, seed = 6, 900, 21
    ds = [bm.Dataset(X, device=0) for _ in range(G)]
    cfg = bm.BigMeansConfig(k=k, chunk_size=s, max_chunks=N, seed=seed)
    out, trace, counts, winner = bm.big_means_multi(ds, cfg)
    chains, w, lab, f, ev = _oracle(port, np.asarray(X, np.float64), k, s, N, seed, G)
    assert counts == [multi.chain_chunks(N, g, G) for g in range(G)]
    assert winner == w
    assert out.objective == f
    assert (bits(out.centroids.values) == bits(chains[w].centroids)).all()
    assert (out.centroids.mask == chains[w].mask).all()
    assert (out.assignment == lab).all()
    assert out.counter.distance_evals == ev
    assert out.counter.iterations == sum(o.iterations for o in chains)
    recs = [(r.chunk_index, r.candidate_objective, r.incumbent_objective, r.accepted, r.degenerate_repaired)
            for r in trace.records]
    assert recs == [t for o in chains for t in o.trace]


def test_big_means_multi_validation():
    X = np.random.default_rng(1).normal(size=(2000, 3))
    ds = [bm.Dataset(X), bm.Dataset(X)]
    with pytest.raises(bm.ConfigError):
        bm.big_means_multi(ds, bm.BigMeansConfig(k=3, chunk_size=100, max_chunks=1))  # fewer chunks than chains
    with pytest.raises(bm.ConfigError):
        bm.big_means_multi([bm.Dataset(X), bm.Dataset(X[:1500])], bm.BigMeansConfig(k=3, chunk_size=100, max_chunks=4))


# ---- two processes on one GPU, torch.distributed (gloo) exchange, device chains ----
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    X = np.random.default_rng(5).normal(size=(12000, 6)) * 2.0 + np.random.default_rng(6).integers(0, 5, (12000, 1)) * 5
    return X, dict(k=7, s=1500, chunks=9, seed=3)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, c = _data()
    d = bm.Dataset(X, device=0)
    cfg = bm.BigMeansConfig(k=c["k"], chunk_size=c["s"], max_chunks=c["chunks"], seed=c["seed"])
    res = multi.big_means_distributed(d.m, c["k"], d.n, multi.gpu_chain(d, cfg), multi.gpu_rows(d),
                                      c["seed"], c["chunks"])
    q.put((rank, res.objective, res.centroids.tobytes(), res.winner, res.evals, res.chunks))
    dist.destroy_process_group()


def test_two_rank_device_chains_vs_g_chain_oracle(port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    X, c = _data()
    chains, w, lab, f, ev = _oracle(port, X, c["k"], c["s"], c["chunks"], c["seed"], world)
    for rank, obj, cbytes, winner, evals, chunks in results:
        assert obj == f
        assert cbytes == np.ascontiguousarray(chains[w].centroids, np.float64).tobytes()
        assert winner == w
        assert evals == ev and chunks == c["chunks"]
