"""The reference's own callers, UNMODIFIED, linked against the B200 drop-in
shims instead of src/big_means.cpp / src/local_search.cpp
(tools/dropin/Makefile; built by __graft_entry__.build() where
/root/reference exists, and shipped to the GPU box with the snapshot).

* acceptance_b200: the reference's acceptance gate (tests/acceptance.cpp).
  Criterion 3 checks big_means(s=m) on the GPU against the reference's CPU
  kmeans bit for bit (acceptance.cpp:167-202); 2 checks monotone traces over a
  corpus of seeded runs (:121-165); 9 checks determinism across reference
  worker counts (:334-375).
* plan_b200 vs plan_ref: the reference's experiment harness
  (bench::run_plan bench.cpp:252-424, execute_cell :25-86, metrics.cpp:21-93,
  io::load io.cpp:224 with min-max normalisation) on one plan; every cell of
  plan_b200 (big_means and the forgy / kmeans_pp / kmeans_parallel kmeans
  baselines) runs on the B200.  Objectives, E_A, n_d, iterations, n_s and the
  accuracy scores must equal the CPU reference's bit for bit (timing columns
  differ by construction).
A missing binary FAILS these tests: they run only on the GPU box, where the
snapshot must carry the binaries."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tools", "dropin", "_build")

pytestmark = pytest.mark.gpu


def _bin(name):
    p = os.path.join(BUILD, name)
    assert os.path.exists(p), f"{p} missing: run __graft_entry__.build() where /root/reference exists"
    return p


@pytest.mark.parametrize("criterion", [2, 3, 9])
def test_reference_acceptance_through_dropin(criterion):
    r = subprocess.run([_bin("acceptance_b200"), str(criterion)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


def _plan(tmp_path, case):
    rng = np.random.default_rng(11)
    if case == "blobs":
        X = np.concatenate([rng.normal(size=(1500, 6)) + c for c in (0.0, 4.0, 9.0, 15.0)])
        ds = {"chunk_size": 700, "max_chunks": 8, "normalize": True}
    else:  # integer-valued rows (exact-sum path), header line, column selection
        X = np.rint(rng.normal(size=(5000, 9)) * 12)
        ds = {"chunk_size": 1200, "max_chunks": 6, "has_header": True, "columns": [0, 2, 3, 5, 8]}
    path = tmp_path / f"{case}.csv"
    with open(path, "w") as f:
        if ds.get("has_header"):
            f.write(",".join(f"c{i}" for i in range(X.shape[1])) + "\n")
        np.savetxt(f, X, delimiter=",", fmt="%.17g")
    plan = {"n_exec": 2, "base_seed": 5, "k_values": [3, 7],
            "algorithms": ["big_means", "forgy", "kmeans_pp", "kmeans_parallel"],
            "datasets": [dict(name=case, path=str(path), format="csv", **ds)]}
    p = tmp_path / f"{case}.json"
    p.write_text(json.dumps(plan))
    return p


@pytest.mark.parametrize("case", ["blobs", "integers"])
def test_bench_plan_through_dropin(tmp_path, case):
    plan = _plan(tmp_path, case)
    out = {}
    for name in ("plan_ref", "plan_b200"):
        r = subprocess.run([_bin(name), str(plan)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        out[name] = json.loads(r.stdout)
    ref, gpu = out["plan_ref"], out["plan_b200"]
    assert len(ref["cells"]) == len(gpu["cells"]) == 8
    for cr, cg in zip(ref["cells"], gpu["cells"]):
        assert (cr["algorithm"], cr["k"], cr["failed"]) == (cg["algorithm"], cg["k"], cg["failed"])
        assert not cr["failed"]
        for rr, rg in zip(cr["runs"], cg["runs"]):
            for key in ("seed", "objective", "e_pct", "n_d", "iterations", "n_s"):
                assert rr[key] == rg[key], (cr["algorithm"], cr["k"], key, rr[key], rg[key])
    for sr, sg in zip(ref["summaries"], gpu["summaries"]):
        for key in ("e_min", "e_mean", "e_max", "nd_mean", "f_best_used"):
            assert sr[key] == sg[key], key
    for sr, sg in zip(ref["scores"], gpu["scores"]):
        assert (sr["algorithm"], sr["sum_score_accuracy"], sr["efficiency_accuracy_pct"]) == \
            (sg["algorithm"], sg["sum_score_accuracy"], sg["efficiency_accuracy_pct"])
