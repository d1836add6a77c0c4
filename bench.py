#!/usr/bin/env python
"""bench.py — MsRSB basis smoothing + iterative multiscale cycle on one B200.

Workload (BASELINE.json configs[1], "config2"): 60x220x85 = 1,122,000 cells, fp64
TPFA, synthetic SPE10-shaped K (synth/, seed 2), 5-spot source columns, 6x11x5
coarse blocks (M = 3,400), ω = 2/3, smoothing to δ <= 1e-3 or 300 sweeps, then the
Richardson multiscale cycle (pre-Jacobi ν = 1, ω_s = 2/3) to ||r|| <= 1e-6 ||b||.

One timed STEP = the whole hot path on HBM-resident inputs: build_tpfa ->
Cartesian partition/supports -> smooth_basis -> coarse_assemble (RAP + Cholesky +
inverse) -> ms_iterate.  Phases are timed with CUDA events on the library stream.
value = basis smoothing sweeps/s (smoothing phase); ms_per_iteration = cycle phase /
iterations.  e2e = the same metric with the whole step driven from pinned host
buffers through the C ABI (K in, pressure out, copies inside the timed region).

--impl reference runs the CPU oracle (oracle/) as it stands on a bounded sample of
the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "basis smoothing sweeps/s & ms per multiscale iteration; achieved HBM GB/s vs peak"
WORKLOAD = "config2: 60x220x85 (1.122M cells) fp64 TPFA, channelized synthetic K, 6x11x5 blocks"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def max_over_ranks(vals, dist=None, device=None):
    """Element-wise max of per-rank timings (the slowest rank defines the job time)."""
    if dist is None:
        return list(vals)
    import torch
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


CYCLE_KERNELS = ("k_jacobi", "k_residual", "k_restrict_cart", "k_symv_tiles", "k_symv_reduce",
                 "k_prolong_cart",
                 "k_finalize")


def _traffic():
    """Per-launch DRAM bytes of the timed kernels from the committed ncu capture
    (profiles/roofline_traffic.json, written by scripts/traffic_from_ncu.py), or None."""
    try:
        doc = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
    except Exception:
        return None, None
    k = doc.get("kernels", {})

    def find(prefix):
        for name, v in k.items():
            if name.startswith(prefix):
                return v
        return None
    sw = find("k_sweep_ws")
    sw_bytes = None
    if sw:  # the persistent sweep kernel runs a chunk of sweeps per launch: per sweep
        sw_bytes = sw.get("per_unit", sw)["dram_bytes"]
    parts = [find(n) for n in CYCLE_KERNELS]
    cyc = None
    if all(p is not None for p in parts):
        cyc = sum(p["dram_bytes"] for p in parts)
    return sw_bytes, cyc


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_info():
    cores = os.cpu_count()
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


# ----------------------------------------------------------------------------- oracle arm
def oracle_sample(prob, sweeps=10, iters=5):
    """Time the CPU oracle as it stands (single thread) on a bounded sample."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import basis as ob
    from oracle import partition as opart
    from oracle import support as osup
    from oracle import tpfa as otpfa
    from oracle.cycle import Level, stage

    A_T, A, q, _ = otpfa.build(prob)
    part, M, _ = opart.cartesian(prob.nx, prob.ny, prob.nz, prob.block)
    pat = osup.box_pattern(prob.nx, prob.ny, prob.nz, prob.block)
    P = ob.indicator(part, pat)
    t0 = time.perf_counter()
    for _ in range(sweeps):
        P, _ = ob.sweep(P, A_T, prob.omega)
    t_sw = time.perf_counter() - t0
    out = dict(sweeps=sweeps, sweep_s=t_sw, sweeps_per_s=sweeps / t_sw)
    if iters > 0:
        import numpy as np
        lev = Level(P.matrix(), A)
        x = np.zeros(prob.N)
        DA = A.diagonal()
        t0 = time.perf_counter()
        for _ in range(iters):
            x = stage(A, DA, q, x, lev, prob.omega_s, prob.nu, prob.post_smooth)
            np.linalg.norm(q - A @ x)
        t_it = time.perf_counter() - t0
        out.update(iters=iters, ms_per_iteration=1e3 * t_it / iters)
    return out


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from synth.configs import make_problem
    prob = make_problem(2)
    cores, model = _cpu_info()
    for _ in range(args.warmup):
        oracle_sample(prob, sweeps=1, iters=0)
    times, sweeps = [], 0
    res = None
    for _ in range(args.steps):
        res = oracle_sample(prob, sweeps=args.ref_sweeps, iters=0)
        times.append(res["sweep_s"])
        sweeps += res["sweeps"]
    tot = sum(times)
    value = sweeps / tot
    it = oracle_sample(prob, sweeps=1, iters=3)
    sample = (f"{args.ref_sweeps} oracle MsRSB sweeps per step on the full config2 grid "
              f"(SciPy SpGEMM, 1 thread); ms/iteration from 3 oracle cycles")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sweeps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "l2": "n/a (CPU)"},
        "ms_per_iteration": it["ms_per_iteration"],
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": model, "host_cores": cores},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
class Clocks:
    def __init__(self, idx):
        self.idx = idx
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{idx}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
            return
        # nvidia-smi takes a while to produce its first sample: wait for it, so that the
        # (short) timed region is sampled; only lines written after mark() count
        t0 = time.time()
        while time.time() - t0 < 10 and self.p.poll() is None:
            self.f.flush()
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.05)
        self.skip = 0

    def mark(self):
        """Start of the timed region: samples written so far are not counted."""
        try:
            with open(self.path) as f:
                self.skip = sum(1 for _ in f)
        except OSError:
            self.skip = 0

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in list(open(self.path))[getattr(self, "skip", 0):]:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def run_gpu(args):
    import numpy as np
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    from paper_2001_01624_b200 import Context, Level, Operator, Solver
    from paper_2001_01624_b200 import pipeline as gp
    from synth.configs import make_problem

    prob = make_problem(2)
    if args.max_iter:
        prob.max_iter = args.max_iter
    N = prob.N
    stream = torch.cuda.current_stream()
    ctx = Context(local, stream)
    K_host = torch.from_numpy(gp.problem_K(prob)).pin_memory()
    K_dev = K_host.to(f"cuda:{local}")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2

    level_facts = {}

    def step(K, x_out=None, timers=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        op = Operator(ctx, prob.nx, prob.ny, prob.nz, K, prob.src_cells, prob.src_rates)
        lev = Level.cartesian(ctx, op, prob.block)
        ev[1].record(stream)
        n, last, deltas, _ = lev.smooth(op, prob.max_sweeps, prob.omega, prob.sweep_tol)
        ev[2].record(stream)
        lev.assemble(op)
        if not level_facts:
            level_facts.update(lev.info())
        solver = Solver(ctx, op, [lev], prob.omega_s, prob.nu, prob.post_smooth)
        x = torch.zeros(N, dtype=torch.float64, device=f"cuda:{local}")
        ev[3].record(stream)
        sol = solver.iterate(x, None, prob.cycle_tol, prob.max_iter, 0, history=True)
        ev[4].record(stream)
        if x_out is not None:
            x_out.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        info = dict(sweeps=n, iters=sol["iters"], t_setup=t[0], t_smooth=t[1], t_coarse=t[2],
                    t_cycle=t[3], t_step=sum(t), res=float(sol["res"][-1]))
        solver.close(); lev.close(); op.close()
        return info

    for _ in range(args.warmup):
        step(K_dev)
    clocks = Clocks(local)
    clocks.start()
    flush.zero_()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks.mark()
    launches0 = ctx.launch_count()
    infos = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between steps (256 MB write)
        infos.append(step(K_dev))
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    if dist:
        dist.barrier()

    # e2e: pinned host K in, pressure out, through the C ABI (copies inside the region)
    x_host = torch.empty(N, dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(0 if args.no_e2e else max(1, min(args.steps, 3))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        inf = step(K_host, x_out=x_host)
        e2e.append((time.perf_counter() - t0, inf["sweeps"]))

    t_smooth = sum(i["t_smooth"] for i in infos) / 1e3
    t_cycle = sum(i["t_cycle"] for i in infos) / 1e3
    t_step = sum(i["t_step"] for i in infos) / 1e3
    sweeps = sum(i["sweeps"] for i in infos)
    iters = sum(i["iters"] for i in infos)
    t_smooth, t_cycle, t_step = max_over_ranks([t_smooth, t_cycle, t_step], dist,
                                               f"cuda:{local}")
    if rank != 0:
        return 0

    # algorithmic bytes: sweep = 16 nnz + 8 faces; cycle stage =
    # 16 nnz + 8 faces + 40 N + coarse solve, the coarse solve reading the lower
    # triangle of the symmetric A_c^{-1}: 8 M (M + 1) / 2
    nnz, faces, M = level_facts["nnz"], prob.n_faces, level_facts["M"]
    b_sweep = 16 * nnz + 8 * faces
    b_iter = 16 * nnz + 8 * faces + 40 * N + 4 * M * (M + 1)
    peaks = _peaks()
    peak = peaks["hbm_gbs"]
    per_sweep = t_smooth / sweeps
    per_iter = t_cycle / max(1, iters)
    gbs_sweep = b_sweep / per_sweep / 1e9
    gbs_iter = b_iter / per_iter / 1e9
    # roofline of the dominant phase of the step (the cycle on config 2): one multiscale
    # iteration is one CUDA-graph launch unit (k_jacobi, k_finalize, k_residual,
    # k_restrict_cart, k_gemv, k_prolong_cart), timed with CUDA events on the library
    # stream around the whole phase and divided by the iteration count
    tr_sweep, tr_iter = _traffic()
    src = "measured (MEASURED_PEAKS.json hbm_gbs, copy)" if not peaks.get("_fallback") \
        else "fallback 6650 GB/s (B200_PROFILING.md)"
    roof_cycle = {"bound": "hbm", "kernel": "cycle iteration: " + " + ".join(CYCLE_KERNELS),
                  "achieved": gbs_iter, "peak": peak, "unit": "GB/s", "frac": gbs_iter / peak,
                  "traffic": tr_iter, "algorithmic_bytes_per_launch": b_iter,
                  "launch_us": 1e6 * per_iter, "peak_source": src,
                  "traffic_source": "profiles/roofline_traffic.json (ncu --set full, cold cache)"}
    roof_sweep = {"bound": "hbm", "kernel": "k_sweep_ws (one sweep; launched in chunks of 32)",
                  "achieved": gbs_sweep, "peak": peak,
                  "unit": "GB/s", "frac": gbs_sweep / peak, "traffic": tr_sweep,
                  "algorithmic_bytes_per_launch": b_sweep, "launch_us": 1e6 * per_sweep,
                  "peak_source": src}
    dominant = roof_cycle if t_cycle >= t_smooth else roof_sweep
    value = ws * sweeps / t_smooth
    cores, model = _cpu_info()
    cpu = None
    if not args.no_cpu_baseline:
        s = oracle_sample(prob, sweeps=args.cpu_sweeps, iters=args.cpu_iters)
        cpu = {"value": s["sweeps_per_s"], "unit": "sweeps/s", "cores": 1, "kind": "oracle",
               "sample": f"{args.cpu_sweeps} oracle sweeps + {args.cpu_iters} oracle cycles on "
                         f"the full config2 grid, single thread",
               "ms_per_iteration": s.get("ms_per_iteration"), "cpu": model, "host_cores": cores}
    c5 = None if args.no_config5 else config5_measure(ctx, stream, local, peak, src)
    cpr = None if args.no_cpr else cpr_measure(ctx, stream, local)
    e2e_t = sum(t for t, _ in e2e) or float("nan")
    e2e_sw = sum(n for _, n in e2e)
    line = {
        "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_step / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "grid": [60, 220, 85], "coarse_blocks": [6, 11, 5],
                   "l2": "flushed between steps (256 MB write)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "ms_per_iteration": 1e3 * per_iter,
        "ms_per_sweep": 1e3 * per_sweep,
        "sweeps_per_step": sweeps / args.steps, "iterations_per_step": iters / args.steps,
        "final_rel_residual": infos[-1]["res"],
        "phase_ms": {k: sum(i[k] for i in infos) / args.steps
                     for k in ("t_setup", "t_smooth", "t_coarse", "t_cycle")},
        "hbm": {"sweep_gbs": gbs_sweep, "cycle_gbs": gbs_iter, "peak_gbs": peak,
                "sweep_frac": gbs_sweep / peak, "cycle_frac": gbs_iter / peak,
                "sweep_frac_nominal_8tbs": gbs_sweep / 8000.0,
                "cycle_frac_nominal_8tbs": gbs_iter / 8000.0},
        "roofline": dominant,
        "roofline_sweep": roof_sweep,
        "roofline_cycle": roof_cycle,
        "config5": c5,
        "next4_cpr": cpr,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_sw / e2e_t, "unit": "sweeps/s",
                "ms_per_step": 1e3 * e2e_t / max(1, len(e2e)),
                "h2d_bytes_per_step": 3 * N * 8, "d2h_bytes_per_step": N * 8},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def config5_measure(ctx, stream, local, peak, src):
    """BASELINE.json configs[4] (200x400x125 = 10M cells, M = 20,000): the whole path once
    untimed, then timed with CUDA events on the library stream — the smoothing phase to
    δ <= 1e-3 (or 300 sweeps), the coarse setup, and the 20 fixed multiscale iterations
    (after one untimed pass that captures the iteration graph).  The half-bandwidth of
    the band-factor bytes is that of A_c's nonzeros in natural order (841).
    Fractions use SURVEY.md §8.d's algorithmic bytes: sweep 16 nnz + 8 faces; iteration
    16 nnz + 8 faces + 40 N + the band factor's two sweeps 2 * 8 M (bw + 1)."""
    import numpy as np
    import torch
    from paper_2001_01624_b200 import Level, Operator, Solver
    from paper_2001_01624_b200 import pipeline as gp
    from synth.configs import make_problem

    prob = make_problem(5)
    K = torch.from_numpy(gp.problem_K(prob)).to(f"cuda:{local}")
    res = {}
    for rep in range(2):  # rep 0 warms up (allocator, graph instantiation)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        op = Operator(ctx, prob.nx, prob.ny, prob.nz, K, prob.src_cells, prob.src_rates)
        lev = Level.cartesian(ctx, op, prob.block)
        ev[1].record(stream)
        n, _, _, _ = lev.smooth(op, prob.max_sweeps, prob.omega, prob.sweep_tol)
        ev[2].record(stream)
        lev.assemble(op)
        solver = Solver(ctx, op, [lev], prob.omega_s, prob.nu, prob.post_smooth)
        x = torch.zeros(prob.N, dtype=torch.float64, device=f"cuda:{local}")
        # the 20 iterations are too few to amortise the one-time CUDA-graph capture of the
        # solver's iteration chunk: capture it untimed, then time the 20 iterations
        solver.iterate(x, None, prob.cycle_tol, 100, prob.fixed_iters, history=True)
        x.zero_()
        ev[3].record(stream)
        sol = solver.iterate(x, None, prob.cycle_tol, 100, prob.fixed_iters, history=True)
        ev[4].record(stream)
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        info = lev.info()
        if rep == 1:
            r, c, v = lev.export_coarse()
            nzm = v != 0.0
            bw = int(np.max(np.abs(r[nzm].astype(np.int64) - c[nzm])))
            N, nnz, M, faces = prob.N, info["nnz"], info["M"], prob.n_faces
            b_sweep = 16 * nnz + 8 * faces
            b_band = 2 * 8 * M * (bw + 1)
            b_iter = 16 * nnz + 8 * faces + 40 * N + b_band
            per_sweep = t[1] / 1e3 / n
            per_iter = t[3] / 1e3 / sol["iters"]
            res = {"workload": "config5: 200x400x125 (10M cells), log-normal K sigma=2, "
                               "Kz/Kx in [0.01, 0.1], 10x10x5 blocks (M = 20,000)",
                   "sweeps": n, "iterations": sol["iters"], "ms_per_sweep": 1e3 * per_sweep,
                   "ms_per_iteration": 1e3 * per_iter, "setup_ms": t[0], "coarse_setup_ms": t[2],
                   "final_rel_residual": float(sol["res"][-1]),
                   "bytes": {"sweep": b_sweep, "iteration": b_iter, "coarse_band": b_band,
                             "coarse_half_bandwidth": bw},
                   "roofline_sweep": {"bound": "hbm", "achieved": b_sweep / per_sweep / 1e9,
                                      "peak": peak, "unit": "GB/s",
                                      "frac": b_sweep / per_sweep / 1e9 / peak,
                                      "peak_source": src},
                   "roofline_cycle": {"bound": "hbm", "achieved": b_iter / per_iter / 1e9,
                                      "peak": peak, "unit": "GB/s",
                                      "frac": b_iter / per_iter / 1e9 / peak,
                                      "peak_source": src,
                                      "coarse_solver": "Schur complement (one-level nested "
                                                       "dissection), own fp64 kernels"}}
        solver.close(); lev.close(); op.close()
    return res


def cpr_measure(ctx, stream, local):
    """SURVEY §8.f NEXT-4 on the config-2 grid (1.122M cells, M = 3,400): the compressible
    two-phase Newton system at a seeded synthetic state (synth.configs.cpr_state), timed with
    CUDA events on the library stream after one untimed pass — linearize (F, J), quasi-IMPES
    decoupling + predictor (A_c = P^T J*_pp P, Gauss–Jordan inverse) + corrector (ILU(0))
    setup, one CPR application, and FGMRES(40) to 1e-8 with the CPR preconditioner."""
    import numpy as np
    import torch
    from paper_2001_01624_b200 import Cpr, Level
    from paper_2001_01624_b200 import pipeline as gp
    from synth.configs import cpr_state, make_problem

    prob = make_problem(2)
    stt = cpr_state(prob)
    op = gp.build_operator(ctx, prob)
    lev = Level.cartesian(ctx, op, prob.block)
    lev.smooth(op, prob.max_sweeps, prob.omega, prob.sweep_tol)
    fl = dict(mu_w=1.0, mu_o=5.0, rho_w=1000.0, rho_o=800.0, c_w=4e-5, c_o=1e-4, c_r=3e-5,
              phi=0.2, p_ref=100.0, dt=0.05, nrel=2)
    c = Cpr(ctx, op, lev, fl)
    N = prob.N
    q = np.zeros(N)
    np.add.at(q, stt.well_cells, stt.well_rates)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{local}")
    p, S, pn, Sn, qd = dev(stt.p), dev(stt.S), dev(stt.p_n), dev(stt.S_n), dev(q)
    r = torch.from_numpy(np.random.default_rng(0).standard_normal(2 * N)).to(f"cuda:{local}")
    dx = torch.empty_like(r)
    out = {}
    for rep in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(stream)
        c.linearize(p, S, pn, Sn, qd)
        ev[1].record(stream)
        c.decouple("quasi")
        ev[2].record(stream)
        c.apply(r, dx)
        ev[3].record(stream)
        x = torch.zeros(2 * N, dtype=torch.float64, device=f"cuda:{local}")
        ev[4].record(stream)
        g = c.fgmres(x, None, tol=1e-8, restart=40, max_iter=400, precond="cpr")
        ev[5].record(stream)
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
        out = {"workload": "config-2 grid (1.122M cells), compressible two-phase Newton system "
                           "at a seeded synthetic state, quasi-IMPES, M = 3,400",
               "linearize_ms": t[0], "decouple_setup_ms": t[1], "cpr_apply_ms": t[2],
               "fgmres_iterations": g["iters"], "fgmres_converged": bool(g["converged"]),
               "fgmres_ms": t[4], "fgmres_final_rel_residual": float(g["res"][-1])}
    c.close(); lev.close(); op.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--max-iter", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e steps "
                    "(ncu launch-list runs)")
    ap.add_argument("--no-cpr", action="store_true", help="skip the NEXT-4 CPR block")
    ap.add_argument("--no-config5", action="store_true", help="skip the 10M-cell config-5 "
                    "sweep / cycle measurement")
    ap.add_argument("--cpu-sweeps", type=int, default=20)
    ap.add_argument("--cpu-iters", type=int, default=10)
    ap.add_argument("--ref-sweeps", type=int, default=5)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
