"""Generate tests/golden/golden.npz from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libbigmeans_ref.so, built
by `make -f oracle/Makefile` from /root/reference/proj/src).  The fixtures pin
both the C restatement (oracle/bm_oracle.c) and the CUDA path; the reference
itself does not travel to the GPU box, these vectors do.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    R = ref()
    if R is None:
        raise SystemExit("oracle/_ref not built; run make -f oracle/Makefile")
    g: dict[str, np.ndarray] = {}
    gen = np.random.default_rng(2204_07485)

    # -- RNG stream (common.hpp:13 + libstdc++ 13 distributions) -------------
    r = R.rng(7)
    g["rng_raw_seed7"] = np.array([R.rng_next(r) for _ in range(16)], np.uint64)
    r = R.rng(11)
    ranges = [(0, 9), (5, 100), (0, 2_500_000 - 1), (123, 10_500_000 - 1), (0, (1 << 40) + 17)]
    ints = []
    for _ in range(8):
        for a, b in ranges:
            ints.append(R.uniform_int(r, a, b))
    g["rng_int_seed11"] = np.array(ints, np.uint64)
    g["rng_int_ranges"] = np.array(ranges, np.uint64)
    r = R.rng(13)
    g["rng_real_seed13"] = np.array([R.uniform_real(r, 0.0, 123.456) for _ in range(16)])

    # -- sample_chunk (big_means.cpp:39-56) ----------------------------------
    cases = [(100, 30, 7), (64, 64, 9), (1000, 999, 3), (5000, 1500, 4), (40, 1, 5),
             (100000, 10000, 0)]
    g["sample_cases"] = np.array(cases, np.uint64)
    for i, (m, s, seed) in enumerate(cases):
        r = R.rng(seed)
        g[f"sample_{i}"] = R.sample_chunk(m, s, r)
        g[f"sample_{i}_next"] = np.array([R.rng_next(r)], np.uint64)

    # -- assign / block_sum / update (core.cpp:106-244) ----------------------
    X = gen.uniform(-10, 10, (4096 + 77, 5))
    C = X[[3, 100, 2000, 4000]].copy()
    mask = np.array([0, 1, 0, 0], np.uint8)
    C[1] = 0.0
    lab, dist, ev = R.assign_nearest(X, C, mask)
    g["core_X"], g["core_C"], g["core_mask"] = X, C, mask
    g["core_labels"], g["core_dists"], g["core_evals"] = lab, dist, np.array([ev], np.uint64)
    g["core_block_sum"] = np.array([R.block_sum(dist)])
    uc, um = R.update_centroids(X, lab, 4)
    g["core_update_C"], g["core_update_mask"] = uc, um
    adv = gen.random(5000) * (10.0 ** (np.arange(5000) % 17))  # test_core.cpp:121-136
    g["blocksum_values"] = adv
    g["blocksum_total"] = np.array([R.block_sum(adv)])

    # -- kmeanspp_fill (init.cpp:123-201) -------------------------------------
    P = gen.uniform(-5, 5, (500, 3))
    g["pp_P"] = P
    c0 = np.zeros((6, 3))
    m0 = np.ones(6, np.uint8)
    cc, cm, ev = R.kmeanspp_fill(P, c0, m0, 3, R.rng(5))
    g["pp_all_C"], g["pp_all_mask"], g["pp_all_evals"] = cc, cm, np.array([ev], np.uint64)
    c1 = np.zeros((4, 3))
    c1[2] = [100.0, 100.0, 100.0]
    m1 = np.array([1, 1, 0, 1], np.uint8)
    cc, cm, ev = R.kmeanspp_fill(P, c1, m1, 3, R.rng(6))
    g["pp_part_Cin"], g["pp_part_maskin"] = c1, m1
    g["pp_part_C"], g["pp_part_mask"], g["pp_part_evals"] = cc, cm, np.array([ev], np.uint64)
    # total <= 0 fallback: every pool point coincides with the chosen center
    Pz = np.tile(np.array([[1.0, 2.0]]), (50, 1))
    cc, cm, ev = R.kmeanspp_fill(Pz, np.zeros((3, 2)), np.ones(3, np.uint8), 3, R.rng(8))
    g["pp_zero_P"], g["pp_zero_C"], g["pp_zero_evals"] = Pz, cc, np.array([ev], np.uint64)

    # -- lloyd (local_search.cpp:16-60) ---------------------------------------
    L = gen.uniform(0, 100, (2000, 2))
    start = L[[5, 17, 400, 999, 1500, 1999, 3, 77, 1234, 1777, 42, 500, 600, 700, 800]].copy()
    g["lloyd_X"], g["lloyd_start"] = L, start
    for tag, tol in (("tol0", 0.0), ("tol5e2", 0.05), ("tol1e4", 1e-4)):
        o = R.lloyd(L, start, np.zeros(15, np.uint8), 300, tol)
        g[f"lloyd_{tag}_C"], g[f"lloyd_{tag}_mask"] = o["centroids"], o["mask"]
        g[f"lloyd_{tag}_labels"], g[f"lloyd_{tag}_hist"] = o["labels"], o["history"]
        g[f"lloyd_{tag}_stats"] = np.array([o["evals"], o["iterations"]], np.uint64)
    # emptied cluster -> degenerate (test_local_search.cpp:106-116)
    E = np.array([[0.0, 0.0], [1.0, 0.0], [10.0, 0.0], [11.0, 0.0]])
    o = R.lloyd(E, np.array([[0.0, 0.0], [10.0, 0.0], [1000.0, 1000.0]]), np.zeros(3, np.uint8))
    g["lloyd_empty_C"], g["lloyd_empty_mask"] = o["centroids"], o["mask"]
    g["lloyd_empty_obj"] = np.array([o["objective"]])

    # -- big_means (big_means.cpp:58-112) --------------------------------------
    bm_cases = [  # (m, n, k, s, chunks, seed, dtype)
        (2000, 3, 5, 300, 12, 31337, "f64"),
        (3000, 2, 6, 500, 20, 404, "f64"),
        (5000, 8, 10, 1000, 15, 0, "f32"),
        (600, 2, 5, 100, 40, 123456789, "f64"),
    ]
    for i, (m, n, k, s, ch, seed, dt) in enumerate(bm_cases):
        X = gen.uniform(0, 50, (m, n))
        if dt == "f32":
            X = X.astype(np.float32)
        o = R.big_means(X.astype(np.float64), k, s, ch, seed=seed)
        g[f"bm{i}_X"] = X
        g[f"bm{i}_cfg"] = np.array([k, s, ch, seed], np.uint64)
        g[f"bm{i}_C"], g[f"bm{i}_mask"], g[f"bm{i}_labels"] = o.centroids, o.mask, o.labels
        g[f"bm{i}_obj"] = np.array([o.objective])
        g[f"bm{i}_stats"] = np.array([o.evals, o.iterations, o.chunks], np.uint64)
        g[f"bm{i}_trace"] = np.array([[t[1], t[2]] for t in o.trace])
        g[f"bm{i}_trace_int"] = np.array([[t[0], t[3], t[4]] for t in o.trace], np.uint64)
    # s == m identity vs kmeans (test_big_means.cpp:177-195)
    X = gen.uniform(0, 50, (260, 2))
    o = R.big_means(X, 4, 260, 1, seed=901)
    km = R.kmeans_pp(X, 4, 901)
    g["ident_X"] = X
    g["ident_C"], g["ident_labels"] = o.centroids, o.labels
    g["ident_obj"] = np.array([o.objective, km.objective])
    g["ident_stats"] = np.array([o.evals, o.iterations, km.evals, km.iterations], np.uint64)

    # kmeans with every InitMethod (local_search.cpp:62-94; init.cpp:92-115, 209-347):
    # (method, rounds_rule, oversampling_l, k, seed) on integer and real data
    km_cases = [(0, 0, 0, 5, 41), (1, 0, 0, 5, 42), (2, 0, 0, 6, 43), (2, 1, 0, 6, 44), (2, 0, 3, 9, 45),
                (2, 0, 0, 1, 46)]
    for i, (meth, rule, l, k, seed) in enumerate(km_cases):
        X = gen.normal(0, 4, (700 + 50 * i, 3))
        if i % 2:
            X = np.rint(X)
        o = R.kmeans(X, k, meth, seed, rounds_rule=rule, oversampling_l=l)
        g[f"km{i}_X"] = X
        g[f"km{i}_cfg"] = np.array([meth, rule, l, k, seed], np.uint64)
        g[f"km{i}_C"], g[f"km{i}_labels"] = o.centroids, o.labels
        g[f"km{i}_obj"] = np.array([o.objective])
        g[f"km{i}_stats"] = np.array([o.evals, o.iterations], np.uint64)
    # the init functions alone on an explicit stream
    X = gen.uniform(0, 10, (400, 4))
    r = R.rng(77)
    g["init_X"] = X
    g["init_forgy"] = R.forgy_init(X, 5, r)
    g["init_kpar"], ev = R.kmeans_parallel_init(X, 7, r)
    g["init_kpar_evals"] = np.array([ev], np.uint64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
