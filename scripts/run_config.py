"""Run one BASELINE config at full size on cuda:0 and report phase timings, iteration
counts and HBM fractions (CUDA events on the library stream).  Not the bench (bench.py
is config 2); this is the config-5 / config-4 measurement harness.

usage: python scripts/run_config.py 5 [--iters 20] [--sweeps 300]
       python scripts/run_config.py 4 [--steps 100]
       python scripts/run_config.py 1|3          (full pipeline incl. split/dynamic stages)
       python scripts/run_config.py 2 --static   (NEXT-2/-3 variants)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2001_01624_b200 import Context, Level, Solver  # noqa: E402
from paper_2001_01624_b200 import pipeline as gp  # noqa: E402
from synth.configs import make_problem  # noqa: E402


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def config_single(cfg, args):
    prob = make_problem(cfg)
    ctx = Context(0)
    st = torch.cuda.current_stream()
    t0 = time.perf_counter()
    e0 = ev(st)
    op = gp.build_operator(ctx, prob)
    lev = Level.cartesian(ctx, op, prob.block)
    e1 = ev(st)
    n, last, deltas, _ = lev.smooth(op, args.sweeps or prob.max_sweeps, prob.omega,
                                   -1.0 if prob.fixed_sweeps else prob.sweep_tol)
    e2 = ev(st)
    lev.assemble(op)
    e3c = ev(st)
    s = Solver(ctx, op, [lev], prob.omega_s, prob.nu, prob.post_smooth)
    x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    fi = args.iters if args.iters else prob.fixed_iters
    # warm-up solve (graph capture/instantiation, first-touch), then the timed solve
    s.iterate(x, None, prob.cycle_tol, prob.max_iter, fi)
    x.zero_()
    e3 = ev(st)
    out = s.iterate(x, None, prob.cycle_tol, prob.max_iter, fi)
    e4 = ev(st)
    torch.cuda.synchronize()
    info = lev.info()
    nnz, M, N, nf = info["nnz"], info["M"], prob.N, prob.n_faces
    t = [e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3c), e3.elapsed_time(e4)]
    b_sweep = 16 * nnz + 8 * nf
    b_iter = 16 * nnz + 8 * nf + 40 * N + 4 * M * (M + 1)  # symmetric inverse: lower triangle
    ms_sweep = t[1] / max(1, n)
    ms_iter = t[3] / max(1, out["iters"])
    pk = peak()
    rec = dict(config=cfg, N=N, M=M, nnz=nnz, sweeps=n, last_delta=last, iters=out["iters"],
               final_res=float(out["res"][-1]), phase_ms=dict(setup=t[0], smooth=t[1], coarse=t[2],
                                                               cycle=t[3]),
               ms_per_sweep=ms_sweep, sweeps_per_s=1e3 / ms_sweep, ms_per_iteration=ms_iter,
               sweep_gbs=b_sweep / ms_sweep / 1e6, iter_gbs=b_iter / ms_iter / 1e6,
               sweep_frac=b_sweep / ms_sweep / 1e6 / pk, iter_frac=b_iter / ms_iter / 1e6 / pk,
               wall_s=time.perf_counter() - t0)
    print(json.dumps(rec), flush=True)


def config_static(cfg, args):
    """Config `cfg` solved with and without the NEXT-3 static levels (wells, MsRSB halo 2;
    log-permeability indicator, constant basis) and with the Jacobi or the NEXT-2 ILU(0)
    smoother: iterations and solve time."""
    ctx = Context(0)
    st = torch.cuda.current_stream()
    W = {"kind": "wells", "radius": 2, "halo": 2}
    I = {"kind": "indicator", "edges": (1.0, 2.5), "halo": 0, "max_blocks": 1024}
    recs = []
    for name, sl, sm in (("cartesian", (), "jacobi"), ("cartesian+wells+logk", (W, I), "jacobi"),
                         ("cartesian / ilu0", (), "ilu0"),
                         ("cartesian+wells+logk / ilu0", (W, I), "ilu0")):
        prob = make_problem(cfg, static_levels=sl, smoother=sm)
        e0 = ev(st)
        op = gp.build_operator(ctx, prob)
        levels, info = gp.build_levels(ctx, op, prob)
        e1 = ev(st)
        s = gp.make_solver(ctx, op, levels, prob)
        x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
        s.iterate(x, None, prob.cycle_tol, prob.max_iter, 0)  # warm-up (graph capture)
        x.zero_()
        e2 = ev(st)
        out = s.iterate(x, None, prob.cycle_tol, prob.max_iter, 0)
        e3 = ev(st)
        torch.cuda.synchronize()
        x.zero_()
        s.fgmres(x, None, tol=prob.cycle_tol, restart=20, max_iter=2000)  # warm-up
        x.zero_()
        e4 = ev(st)
        fg = s.fgmres(x, None, tol=prob.cycle_tol, restart=20, max_iter=2000)
        e5 = ev(st)
        torch.cuda.synchronize()
        recs.append(dict(levels=name, M=[lv.info()["M"] for lv in levels],
                         sweeps=[i[0] for i in info], iters=out["iters"],
                         converged=out["converged"], setup_ms=e0.elapsed_time(e1),
                         solve_ms=e2.elapsed_time(e3),
                         ms_per_iteration=e2.elapsed_time(e3) / max(1, out["iters"]),
                         fgmres_steps=fg["iters"], fgmres_converged=fg["converged"],
                         fgmres_ms=e4.elapsed_time(e5),
                         fgmres_ms_per_step=e4.elapsed_time(e5) / max(1, fg["iters"])))
    print(json.dumps(dict(config=cfg, static_levels=recs)), flush=True)


def config_pipeline(cfg, args):
    """Configs 1 and 3 (and any config) through the full pipeline: all of the config's
    levels (config 3: Cartesian + fault-split, dynamic stage, post-smoothing), phases timed
    with CUDA events; the solve is timed after a warm-up solve."""
    prob = make_problem(cfg)
    ctx = Context(0)
    st = torch.cuda.current_stream()
    e0 = ev(st)
    op = gp.build_operator(ctx, prob)
    levels, info = gp.build_levels(ctx, op, prob)
    e1 = ev(st)
    s = gp.make_solver(ctx, op, levels, prob)
    x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
    s.iterate(x, None, prob.cycle_tol, prob.max_iter, prob.fixed_iters)
    x.zero_()
    e2 = ev(st)
    out = s.iterate(x, None, prob.cycle_tol, prob.max_iter, prob.fixed_iters)
    e3 = ev(st)
    torch.cuda.synchronize()
    dyn = out.get("dyn_M")
    rec = dict(config=cfg, N=prob.N, M=[lv.info()["M"] for lv in levels],
               sweeps=[i[0] for i in info], iters=out["iters"], converged=out["converged"],
               final_res=float(out["res"][-1]), setup_levels_ms=e0.elapsed_time(e1),
               solve_ms=e2.elapsed_time(e3),
               ms_per_iteration=e2.elapsed_time(e3) / max(1, out["iters"]),
               dyn_M_median=float(np.median(dyn[dyn > 0])) if dyn is not None and np.any(dyn > 0) else 0,
               dyn_M_pct=[float(np.percentile(dyn[dyn > 0], q)) for q in (10, 25, 75, 90, 100)]
               if dyn is not None and np.any(dyn > 0) else [])
    print(json.dumps(rec), flush=True)


def config4(args):
    prob = make_problem(4)
    ctx = Context(0)
    t0 = time.perf_counter()
    out = gp.run_sequential(ctx, prob, steps=args.steps)
    torch.cuda.synchronize()
    its = [r["iters"] for r in out["steps"]]
    rec = dict(config=4, steps=args.steps, init_sweeps=out["init_sweeps"], total_iters=int(sum(its)),
               per_step_iters=its, substeps=[r["n_sub"] for r in out["steps"]],
               wall_s=time.perf_counter() - t0,
               S_max=float(out["S"].max()), S_mean=float(out["S"].mean()))
    print(json.dumps(rec), flush=True)


def config_cpr(cfg, args):
    """§8 NEXT-4 on config `cfg`'s grid (default the 1.122M-cell config-2 grid): the
    compressible two-phase Newton system at a synthetic state (synth.configs.cpr_state),
    linearize, quasi-IMPES decoupling + predictor/corrector setup, one CPR application,
    FGMRES(40) to 1e-8 with CPR and with ILU(0) alone; CUDA events on the library stream."""
    from paper_2001_01624_b200 import Cpr
    from synth.configs import cpr_state
    prob = make_problem(cfg)
    st_ = cpr_state(prob)
    ctx = Context(0)
    st = torch.cuda.current_stream()
    op = gp.build_operator(ctx, prob)
    lev = Level.cartesian(ctx, op, prob.block)
    lev.smooth(op, prob.max_sweeps, prob.omega, prob.sweep_tol)
    fl = dict(mu_w=1.0, mu_o=5.0, rho_w=1000.0, rho_o=800.0, c_w=4e-5, c_o=1e-4, c_r=3e-5,
              phi=0.2, p_ref=100.0, dt=0.05, nrel=2)
    c = Cpr(ctx, op, lev, fl, n_cycles=args.cycles)
    N = prob.N
    q = np.zeros(N)
    np.add.at(q, st_.well_cells, st_.well_rates)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    p, S, pn, Sn, qd = dev(st_.p), dev(st_.S), dev(st_.p_n), dev(st_.S_n), dev(q)
    c.linearize(p, S, pn, Sn, qd)
    c.decouple("quasi")  # warm-up
    torch.cuda.synchronize()
    e0 = ev(st)
    c.linearize(p, S, pn, Sn, qd)
    e1 = ev(st)
    c.decouple("quasi")
    e2 = ev(st)
    r = torch.randn(2 * N, dtype=torch.float64, device="cuda")
    dx = torch.empty_like(r)
    c.apply(r, dx)
    torch.cuda.synchronize()
    e3 = ev(st)
    for _ in range(10):
        c.apply(r, dx)
    e4 = ev(st)
    torch.cuda.synchronize()
    out = {}
    for pre in ("cpr", "ilu0"):
        x = torch.zeros(2 * N, dtype=torch.float64, device="cuda")
        a = ev(st)
        g = c.fgmres(x, None, tol=1e-8, restart=40, max_iter=args.max_iter or 400, precond=pre)
        b = ev(st)
        torch.cuda.synchronize()
        out[pre] = dict(iters=g["iters"], converged=g["converged"], ms=a.elapsed_time(b),
                        final=float(g["res"][-1]))
    rec = dict(workload=f"cpr on config{cfg} grid", N=N, M=lev.info()["M"], n_cycles=args.cycles,
               linearize_ms=e0.elapsed_time(e1), decouple_setup_ms=e1.elapsed_time(e2),
               apply_ms=e3.elapsed_time(e4) / 10, fgmres=out)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--sweeps", type=int, default=0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--static", action="store_true", help="NEXT-3 static levels vs none")
    ap.add_argument("--cpr", action="store_true", help="NEXT-4 CPR on the config's grid")
    ap.add_argument("--cycles", type=int, default=1)
    ap.add_argument("--max-iter", type=int, default=0)
    a = ap.parse_args()
    if a.cpr:
        config_cpr(a.config, a)
    elif a.static:
        config_static(a.config, a)
    elif a.config in (1, 3):
        config_pipeline(a.config, a)
    elif a.config == 4:
        config4(a)
    else:
        config_single(a.config, a)
