"""Full-size parity (BASELINE.json configs[1..4] at their full sizes) against the CPU
oracle's stored results, tests/golden/full_config{2,3,4,5}.npz, written by
scripts/make_goldens.py — a committed script that calls only oracle/ (the oracle takes
minutes to half an hour per config on one core, so it is not re-run inside `pytest -m gpu`).

Tolerances (BASELINE.json north_star; SURVEY.md §8.c protocol):
  P      exact zeros where the oracle has zeros, else |ΔP|/P <= 1e-10, after the same
         sweeps-to-tol count (on a seeded sample of rows: the oracle's P has 6.96M / 68.1M
         entries)
  A_c    entrywise <= 1e-12 max|A_c|
  x      ||Δx|| / ||x|| <= max(1e-9, 2 * floor) at an equal iteration count, on a seeded
         sample of cells; floor = the largest distance of the GENUINE alternate exact
         coarse solvers (oracle.coarse) from the oracle, stored with the golden
  counts |k_gpu - k_oracle| <= max(1, 2 * the alternates' count spread) in free mode
Every comparison is logged (conftest.record_parity -> parity_r02.json).
"""
import hashlib
import os

import numpy as np
import pytest

from synth.configs import make_problem

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
P_RTOL = 1e-10
X_RTOL = 1e-9


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2001_01624_b200 import Context
    return Context(0)


def _gold(cfg):
    path = os.path.join(GOLD, f"full_config{cfg}.npz")
    assert os.path.exists(path), f"missing golden {path} (scripts/make_goldens.py {cfg})"
    with np.load(path, allow_pickle=False) as z:  # decompress every array once
        return {k: z[k] for k in z.files}


def _inputs_sha(prob):
    h = hashlib.sha256()
    for a in (prob.kx, prob.ky, prob.kz, prob.rhs(), prob.mult_x, prob.mult_y, prob.mult_z):
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def _check_P(lev, g, pre):
    """GPU P on the golden's sampled rows: exact zeros and 1e-10 relative."""
    rowptr, cols, vals, _ = lev.export()
    rows = g[pre + "P_rows"]
    rp = g[pre + "P_rowptr"]
    worst = 0.0
    for t, r in enumerate(rows):
        a, b = rowptr[r], rowptr[r + 1]
        gc, gv = cols[a:b], vals[a:b]
        oc, ov = g[pre + "P_cols"][rp[t]:rp[t + 1]], g[pre + "P_vals"][rp[t]:rp[t + 1]]
        assert np.array_equal(gc, oc), (pre, r)
        z = ov == 0.0
        assert np.all(gv[z] == 0.0), (pre, r)
        if np.any(~z):
            worst = max(worst, float(np.max(np.abs(gv[~z] - ov[~z]) / ov[~z])))
    assert worst <= P_RTOL, (pre, worst)
    return worst


def _floors(g, k_key="k"):
    names = [str(n) for n in g["alt_names"]]
    xo = g["x"]
    fl = [float(np.linalg.norm(g[f"alt_{i}_x"] - xo) / np.linalg.norm(xo)) for i in range(len(names))]
    ks = [int(g[f"alt_{i}_k"]) for i in range(len(names))] if f"alt_0_k" in g else []
    return names, fl, ks


def test_full_config2_free_mode_parity(ctx):
    """Config 2 (1.122M cells, M = 3,400): sweeps-to-tol and δ history, P, A_c, the
    free-mode Richardson count and the iterate at an equal count."""
    import torch
    from conftest import record_parity
    from paper_2001_01624_b200 import pipeline as gp
    g = _gold(2)
    prob = make_problem(2)
    assert _inputs_sha(prob) == str(g["inputs_sha"])
    op = gp.build_operator(ctx, prob)
    levels, info = gp.build_levels(ctx, op, prob)
    n, last, deltas, _ = info[0]
    assert n == int(g["L0_sweeps"]), (n, int(g["L0_sweeps"]))
    assert np.allclose(deltas, g["L0_deltas"], rtol=1e-9, atol=1e-15)
    p_err = _check_P(levels[0], g, "L0_")
    _, _, _, Ac = levels[0].export(with_Ac=True)
    r, c, v = g["Ac_row"], g["Ac_col"], g["Ac_val"]
    scale = np.abs(v).max()
    ac_err = float(np.max(np.abs(Ac[r, c] - v)) / scale)
    mask = np.zeros_like(Ac, dtype=bool)
    mask[r, c] = True
    ac_out = float(np.max(np.abs(Ac[~mask])) / scale)
    s = gp.make_solver(ctx, op, levels, prob)
    x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    free = s.iterate(x, None, prob.cycle_tol, prob.max_iter)
    k_or = int(g["k"])
    names, fl, ks = _floors(g)
    k_tol = max(1, 2 * max(abs(k - k_or) for k in ks))
    x.zero_()
    fixed = s.iterate(x, None, prob.cycle_tol, prob.max_iter, k_or)
    xs = x.cpu().numpy()[g["x_idx"]]
    err = float(np.linalg.norm(xs - g["x"]) / np.linalg.norm(g["x"]))
    x_tol = max(X_RTOL, 2.0 * max(fl))
    record_parity("full/config2", sweeps=n, p_err=p_err, ac_err=ac_err, ac_outside=ac_out,
                  k_gpu=free["iters"], k_oracle=k_or, k_alternates=ks, k_tol=k_tol, err=err,
                  floor=max(fl), alternates=dict(zip(names, fl)), x_tol=x_tol)
    assert ac_err <= 1e-12 and ac_out <= 1e-12, (ac_err, ac_out)
    assert abs(free["iters"] - k_or) <= k_tol, (free["iters"], k_or, ks)
    assert err <= x_tol, (err, fl)
    assert np.allclose(fixed["res"], g["res"][:k_or + 1], rtol=1e-6, atol=1e-12)


def test_full_config3_free_mode_parity(ctx):
    """Config 3 (faults; Cartesian + fault-split M = 4,284 levels, the dynamic stage every
    iteration, post-smoothing): both levels' sweeps and P, the split partition bit-exact
    (its restriction is the column gather with W > 1 slot planes), M_dyn per iteration
    until the genuine alternates themselves diverge, the free-mode count and the iterate
    at an equal count."""
    import torch
    from conftest import record_parity
    from paper_2001_01624_b200 import pipeline as gp
    g = _gold(3)
    prob = make_problem(3)
    assert _inputs_sha(prob) == str(g["inputs_sha"])
    op = gp.build_operator(ctx, prob)
    levels, info = gp.build_levels(ctx, op, prob)
    for li, pre in zip(info, ("L0_", "L1_")):
        assert li[0] == int(g[pre + "sweeps"]), (pre, li[0])
        assert np.allclose(li[2], g[pre + "deltas"], rtol=1e-9, atol=1e-15)
    sp_info = levels[1].info(with_part=True)
    assert sp_info["M"] == int(g["L1_M"]) and sp_info["W"] > 1
    assert np.array_equal(sp_info["part"], g["L1_part"])
    p0 = _check_P(levels[0], g, "L0_")
    p1 = _check_P(levels[1], g, "L1_")
    s = gp.make_solver(ctx, op, levels, prob)
    x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    free = s.iterate(x, None, prob.cycle_tol, prob.max_iter)
    k_or = int(g["k"])
    names, fl, ks = _floors(g)
    k_tol = max(1, 2 * max(abs(k - k_or) for k in ks))
    # M_dyn per iteration: equal up to the first iteration where a genuine alternate's
    # Δp partitions (label hashes) leave the oracle's
    h_or = [str(h) for h in g["dyn_hash"]]
    div = len(h_or)
    for i in range(len(names)):
        ha = [str(h) for h in g[f"alt_{i}_dyn_hash"]]
        j = next((t for t, (a, b) in enumerate(zip(ha, h_or)) if a != b), min(len(ha), len(h_or)))
        div = min(div, j)
    m_or = g["dyn_M"]
    m_gpu = np.asarray(free["dyn_M"])[1:]  # iteration 1 has no dynamic stage
    n_eq = min(div, len(m_or), len(m_gpu))
    x.zero_()
    s.iterate(x, None, prob.cycle_tol, prob.max_iter, k_or)
    xs = x.cpu().numpy()[g["x_idx"]]
    err = float(np.linalg.norm(xs - g["x"]) / np.linalg.norm(g["x"]))
    x_tol = max(X_RTOL, 2.0 * max(fl))
    record_parity("full/config3", p_err=max(p0, p1), k_gpu=free["iters"], k_oracle=k_or,
                  k_alternates=ks, k_tol=k_tol, dyn_equal_until=int(n_eq),
                  dyn_first_mismatch=int(next((t for t in range(min(len(m_or), len(m_gpu)))
                                               if m_or[t] != m_gpu[t]), -1)),
                  err=err, floor=max(fl), alternates=dict(zip(names, fl)), x_tol=x_tol)
    assert np.array_equal(m_gpu[:n_eq], m_or[:n_eq]), (m_gpu[:n_eq], m_or[:n_eq])
    assert abs(free["iters"] - k_or) <= k_tol, (free["iters"], k_or, ks)
    assert err <= x_tol, (err, fl)


def test_full_config3_dynamic_labels(ctx):
    """The dynamic-partition rebuild at full size: the same Δp in gives the same integer
    partition out, bit-exact (a smooth seeded Δp with features at every scale)."""
    from oracle import partition as opart
    from paper_2001_01624_b200 import pipeline as gp
    prob = make_problem(3, dynamic=True)
    op = gp.build_operator(ctx, prob)
    levels, _ = gp.build_levels(ctx, op, prob, sweeps=2, fixed=True)
    rng = np.random.default_rng(11)
    c = np.arange(prob.N)
    i, j, k = c % prob.nx, (c // prob.nx) % prob.ny, c // (prob.nx * prob.ny)
    dp = np.zeros(prob.N)
    for _ in range(12):  # Gaussian bumps of random width and sign
        ci, cj, ck = rng.uniform(0, prob.nx), rng.uniform(0, prob.ny), rng.uniform(0, prob.nz)
        w = rng.uniform(3, 40)
        dp += rng.choice([-1, 1]) * np.exp(-((i - ci) ** 2 + (j - cj) ** 2 + (k - ck) ** 2) / w ** 2)
    dp += 1e-3 * rng.standard_normal(prob.N)
    for mb in (1024, 64):
        prob.dyn_max_blocks = mb
        s2 = gp.make_solver(ctx, op, levels, prob)
        part_o, M_o = opart.dynamic_partition(dp, prob.nx, prob.ny, prob.nz, max_blocks=mb)
        part_g = np.zeros(prob.N, dtype=np.int32)
        M_g = s2.add_dynamic_basis(np.ascontiguousarray(dp), part_g)
        assert M_g == M_o, (mb, M_g, M_o)
        assert np.array_equal(part_g, part_o.astype(np.int32)), mb


def test_full_config4_first_steps(ctx):
    """Config 4 (two-phase, 1.122M cells): the first steps' free-mode counts, then pressure
    and saturation in lockstep (the oracle's per-step counts)."""
    from conftest import record_parity
    from paper_2001_01624_b200 import pipeline as gp
    g = _gold(4)
    prob = make_problem(4)
    assert _inputs_sha(prob) == str(g["inputs_sha"])
    steps = int(g["steps"])
    free = gp.run_sequential(ctx, prob, steps=steps)
    assert free["init_sweeps"] == int(g["init_sweeps"])
    # dt = pv Σφ|Ω| / Σq⁺ (reading A18): a device sum of 1.12M terms in another order than
    # numpy's pairwise sum — the rounding bound of the longest addition chain (~330 adds)
    assert abs(free["dt"] - float(g["dt"])) <= 1e-12 * float(g["dt"])
    k_or = [int(k) for k in g["k"]]
    names = [str(n) for n in g["alt_names"]]
    spread = max(abs(int(a) - b) for i in range(len(names)) for a, b in zip(g[f"alt_{i}_k"], k_or))
    k_tol = max(1, 2 * spread)
    k_gpu = [r["iters"] for r in free["steps"]]
    lock = gp.run_sequential(ctx, prob, steps=steps, fixed_iters=k_or, keep_states=True)
    idx = g["x_idx"]
    recs = []
    for n, r in enumerate(lock["steps"]):
        assert r["n_sub"] == int(g["n_sub"][n])
        pn, Sn = g["p"][n], g["S"][n]
        ep = float(np.linalg.norm(r["p"][idx] - pn) / np.linalg.norm(pn))
        eS = float(np.max(np.abs(r["S"][idx] - Sn)))
        fp = max(float(np.linalg.norm(g[f"alt_{i}_p"][n] - pn) / np.linalg.norm(pn))
                 for i in range(len(names)))
        fS = max(float(np.max(np.abs(g[f"alt_{i}_S"][n] - Sn))) for i in range(len(names)))
        recs.append((ep, fp, eS, fS))
    record_parity("full/config4", k_gpu=k_gpu, k_oracle=k_or, k_tol=k_tol,
                  p_err=[r[0] for r in recs], p_floor=[r[1] for r in recs],
                  S_err=[r[2] for r in recs], S_floor=[r[3] for r in recs])
    for kg, ko in zip(k_gpu, k_or):
        assert abs(kg - ko) <= k_tol, (k_gpu, k_or)
    for ep, fp, eS, fS in recs:
        assert ep <= max(X_RTOL, 2.0 * fp), (ep, fp)
        assert eS <= max(1e-9, 2.0 * fS), (eS, fS)


def test_full_config5_fixed_iterations(ctx):
    """Config 5 (10M cells, M = 20,000, anisotropic K): sweeps-to-tol, P, the exact A_c
    (box stencil) on sampled rows, and 20 fixed iterations with the Schur-complement
    coarse solver."""
    import torch
    from conftest import record_parity
    from paper_2001_01624_b200 import pipeline as gp
    g = _gold(5)
    prob = make_problem(5)
    assert _inputs_sha(prob) == str(g["inputs_sha"])
    op = gp.build_operator(ctx, prob)
    levels, info = gp.build_levels(ctx, op, prob)
    n = info[0][0]
    assert n == int(g["L0_sweeps"]), (n, int(g["L0_sweeps"]))
    assert np.allclose(info[0][2], g["L0_deltas"], rtol=1e-9, atol=1e-15)
    p_err = _check_P(levels[0], g, "L0_")
    r, c, v = levels[0].export_coarse()
    M = 20000
    rows = g["Ac_rows"]
    rp = g["Ac_rowptr"]
    scale = float(g["Ac_absmax"])
    order = np.argsort(r, kind="stable")
    rs = np.searchsorted(r[order], np.arange(M + 1))
    ac_err = 0.0
    for t, a in enumerate(rows):
        sel = order[rs[a]:rs[a + 1]]
        got = dict(zip(c[sel].tolist(), v[sel].tolist()))
        oc, ov = g["Ac_cols"][rp[t]:rp[t + 1]], g["Ac_vals"][rp[t]:rp[t + 1]]
        for cc, vv in zip(oc.tolist(), ov.tolist()):
            ac_err = max(ac_err, abs(got.get(cc, 0.0) - vv) / scale)
        ref = dict(zip(oc.tolist(), ov.tolist()))
        for cc, vv in got.items():
            if cc not in ref:
                ac_err = max(ac_err, abs(vv) / scale)
    diag = np.zeros(M)
    dm = r == c
    diag[r[dm]] = v[dm]
    ac_err = max(ac_err, float(np.max(np.abs(diag - g["Ac_diag"])) / scale))
    s = gp.make_solver(ctx, op, levels, prob)
    x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    out = s.iterate(x, None, prob.cycle_tol, 100, int(g["k"]))
    xs = x.cpu().numpy()[g["x_idx"]]
    err = float(np.linalg.norm(xs - g["x"]) / np.linalg.norm(g["x"]))
    names, fl, _ = _floors(g)
    x_tol = max(X_RTOL, 2.0 * max(fl))
    record_parity("full/config5", sweeps=n, p_err=p_err, ac_err=ac_err, k=int(g["k"]), err=err,
                  floor=max(fl), alternates=dict(zip(names, fl)), x_tol=x_tol)
    assert ac_err <= 1e-12, ac_err
    assert err <= x_tol, (err, fl)
    assert np.allclose(out["res"], g["res"], rtol=1e-6, atol=1e-13)
