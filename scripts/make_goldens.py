"""Write the full-size parity goldens tests/golden/full_config{2,3,4,5}.npz.

Calls ONLY the CPU oracle (oracle/) on the seeded synthetic inputs (synth/): no value
here comes from the CUDA path.  The oracle run at BASELINE.json's full sizes takes
minutes (config 2, 3, 4) to half an hour (config 5) on one core, so its results are
stored instead of recomputed inside `pytest -m gpu`; the GPU tests
(tests/test_gpu_full.py) compare against them.

What is stored (sampled where the full array would not fit in git):
  inputs_sha   sha256 of kx|ky|kz|rhs|multipliers (the GPU test checks it first)
  per level    sweeps-to-tol, the δ history, M, nnz, the oracle's P on a seeded
               sample of rows (rowptr/cols/vals of those rows)
  A_c          config 2: every nonzero (COO); config 5: a seeded sample of rows + the
               diagonal
  solve        free-mode count k, the residual history ρ_0..ρ_k, x at k on a seeded
               sample of cells (+ ||x||_2 of the full vector)
  floors       the same solve by the ALTERNATE exact coarse solvers of oracle.coarse
               (genuine library solvers): their free-mode counts and x
               at the oracle's count, on the same sample
  config 3     the fault-split partition, and M_dyn of every iteration (oracle and
               alternates)
  config 4     per-step counts, pressure and saturation samples of the first steps

Usage: python scripts/make_goldens.py 2|3|4|5   (OMP/BLAS threads pinned to 1)
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from oracle import pipeline as opl  # noqa: E402
from oracle import transport as otr  # noqa: E402
from synth.configs import make_problem  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def inputs_sha(prob):
    h = hashlib.sha256()
    for a in (prob.kx, prob.ky, prob.kz, prob.rhs(), prob.mult_x, prob.mult_y, prob.mult_z):
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def sample(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(n, k), replace=False)).astype(np.int64)


def level_record(d, pre, li, rows):
    P = li["P"].matrix().tocsr()
    sub = P[rows]
    d[pre + "sweeps"] = np.int64(li["sweeps"])
    d[pre + "deltas"] = np.asarray(li["deltas"], dtype=np.float64)
    d[pre + "M"] = np.int64(li["M"])
    d[pre + "nnz"] = np.int64(P.nnz)
    d[pre + "P_rows"] = rows
    d[pre + "P_rowptr"] = sub.indptr.astype(np.int64)
    d[pre + "P_cols"] = sub.indices.astype(np.int32)
    d[pre + "P_vals"] = sub.data.astype(np.float64)


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def config2():
    prob = make_problem(2)
    d = dict(inputs_sha=inputs_sha(prob))
    xs = sample(prob.N, 140_000, 22)
    d["x_idx"] = xs
    log("oracle run")
    r = opl.run(prob)
    sol = r["sol"]
    level_record(d, "L0_", r["levels_info"][0], sample(prob.N, 40_000, 21))
    Ac = sp.coo_matrix(r["levels"][0].Ac)
    d.update(Ac_row=Ac.row.astype(np.int32), Ac_col=Ac.col.astype(np.int32), Ac_val=Ac.data)
    k = sol["iters"]
    d.update(k=np.int64(k), res=sol["res"], x=sol["x"][xs], x_norm=np.linalg.norm(sol["x"]),
             converged=np.bool_(sol["converged"]))
    log("k", k, "sweeps", r["levels_info"][0]["sweeps"])
    alts = []
    for coarse, assoc in (("cholesky", "right"), ("inverse", "right"),
                          ("lu_reversed", "right"), ("lu", "left")):
        name = f"{coarse}/{assoc}"
        ra = opl.run(prob, levels_info=r["levels_info"], coarse=coarse, assoc=assoc)["sol"]
        ka = ra["iters"]
        xa = ra["x"]
        if ka != k:
            xa = opl.run(prob, levels_info=r["levels_info"], coarse=coarse, assoc=assoc,
                         fixed_iters=k)["sol"]["x"]
        alts.append(name)
        d[f"alt_{len(alts) - 1}_k"] = np.int64(ka)
        d[f"alt_{len(alts) - 1}_x"] = xa[xs]
        d[f"alt_{len(alts) - 1}_res"] = ra["res"]
        log(name, "k", ka, "dx", np.linalg.norm(xa[xs] - d["x"]) / np.linalg.norm(d["x"]))
    d["alt_names"] = np.array(alts)
    return d


def config3():
    prob = make_problem(3)
    d = dict(inputs_sha=inputs_sha(prob))
    xs = sample(prob.N, 140_000, 32)
    d["x_idx"] = xs
    hashes = {}

    def rec(tag):
        def f(k, part, M):
            hashes.setdefault(tag, []).append(
                (k, M, hashlib.sha256(np.ascontiguousarray(part, dtype=np.int32)).hexdigest()))
        return f

    log("oracle run")
    r = opl.run(prob, record_dynamic=rec("lu"))
    sol = r["sol"]
    li = r["levels_info"]
    level_record(d, "L0_", li[0], sample(prob.N, 40_000, 31))
    level_record(d, "L1_", li[1], sample(prob.N, 40_000, 33))
    d["L1_part"] = li[1]["part"].astype(np.int32)
    k = sol["iters"]
    d.update(k=np.int64(k), res=sol["res"], x=sol["x"][xs], x_norm=np.linalg.norm(sol["x"]),
             converged=np.bool_(sol["converged"]), dyn_M=np.array(sol["dyn_M"], dtype=np.int64))
    d["dyn_hash"] = np.array([h for _, _, h in hashes["lu"]])
    log("k", k, "sweeps", li[0]["sweeps"], li[1]["sweeps"], "M1", li[1]["M"])
    alts = []
    for coarse in ("cholesky", "inverse", "lu_reversed"):
        ra = opl.run(prob, levels_info=li, coarse=coarse, record_dynamic=rec(coarse))["sol"]
        ka = ra["iters"]
        xa = ra["x"]
        if ka != k:
            xa = opl.run(prob, levels_info=li, coarse=coarse, fixed_iters=k)["sol"]["x"]
        alts.append(coarse)
        i = len(alts) - 1
        d[f"alt_{i}_k"] = np.int64(ka)
        d[f"alt_{i}_x"] = xa[xs]
        d[f"alt_{i}_res"] = ra["res"]
        d[f"alt_{i}_dyn_M"] = np.array(ra["dyn_M"], dtype=np.int64)
        d[f"alt_{i}_dyn_hash"] = np.array([h for _, _, h in hashes[coarse]])
        log(coarse, "k", ka, "dx", np.linalg.norm(xa[xs] - d["x"]) / np.linalg.norm(d["x"]))
    d["alt_names"] = np.array(alts)
    return d


def config4(steps=3):
    prob = make_problem(4)
    d = dict(inputs_sha=inputs_sha(prob))
    xs = sample(prob.N, 140_000, 42)
    d["x_idx"] = xs
    log("oracle run")
    r = otr.run(prob, steps=steps)
    ks = [s["iters"] for s in r["steps"]]
    d.update(steps=np.int64(steps), init_sweeps=np.int64(r["init_sweeps"]), dt=r["dt"],
             k=np.array(ks, dtype=np.int64),
             n_sub=np.array([s["n_sub"] for s in r["steps"]], dtype=np.int64),
             p=np.stack([s["p"][xs] for s in r["steps"]]),
             S=np.stack([s["S"][xs] for s in r["steps"]]),
             p_norm=np.array([np.linalg.norm(s["p"]) for s in r["steps"]]))
    log("k", ks)
    alts = []
    for coarse in ("cholesky", "inverse"):
        rf = otr.run(prob, steps=steps, coarse=coarse)
        rl = otr.run(prob, steps=steps, coarse=coarse, fixed_iters=ks)
        alts.append(coarse)
        i = len(alts) - 1
        d[f"alt_{i}_k"] = np.array([s["iters"] for s in rf["steps"]], dtype=np.int64)
        d[f"alt_{i}_p"] = np.stack([s["p"][xs] for s in rl["steps"]])
        d[f"alt_{i}_S"] = np.stack([s["S"][xs] for s in rl["steps"]])
        log(coarse, "k", d[f"alt_{i}_k"])
    d["alt_names"] = np.array(alts)
    return d


def config5():
    prob = make_problem(5)
    d = dict(inputs_sha=inputs_sha(prob))
    xs = sample(prob.N, 250_000, 52)
    d["x_idx"] = xs
    log("oracle run")
    r = opl.run(prob)
    sol = r["sol"]
    level_record(d, "L0_", r["levels_info"][0], sample(prob.N, 40_000, 51))
    Ac = r["levels"][0].Ac.tocsr()
    arows = sample(Ac.shape[0], 2_000, 53)
    sub = Ac[arows]
    d.update(Ac_rows=arows, Ac_rowptr=sub.indptr.astype(np.int64),
             Ac_cols=sub.indices.astype(np.int32), Ac_vals=sub.data, Ac_diag=Ac.diagonal(),
             Ac_nnz=np.int64(Ac.nnz), Ac_absmax=np.abs(Ac.data).max())
    k = sol["iters"]
    d.update(k=np.int64(k), res=sol["res"], x=sol["x"][xs], x_norm=np.linalg.norm(sol["x"]))
    log("k", k, "sweeps", r["levels_info"][0]["sweeps"])
    alts = []
    for coarse, assoc in (("cholesky", "right"), ("splu_natural", "right"), ("lu", "left")):
        ra = opl.run(prob, levels_info=r["levels_info"], coarse=coarse, assoc=assoc)["sol"]
        alts.append(f"{coarse}/{assoc}")
        i = len(alts) - 1
        d[f"alt_{i}_x"] = ra["x"][xs]
        d[f"alt_{i}_res"] = ra["res"]
        log(alts[-1], "dx", np.linalg.norm(ra["x"][xs] - d["x"]) / np.linalg.norm(d["x"]))
    d["alt_names"] = np.array(alts)
    return d


def main():
    cfg = int(sys.argv[1])
    t0 = time.time()
    d = {2: config2, 3: config3, 4: config4, 5: config5}[cfg]()
    d["oracle_seconds"] = time.time() - t0
    path = os.path.join(OUT, f"full_config{cfg}.npz")
    np.savez_compressed(path, **d)
    log("wrote", path, os.path.getsize(path), "bytes", f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
