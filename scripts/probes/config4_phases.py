import os, sys, time, json
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2001_01624_b200 import Context, Level, Solver
from paper_2001_01624_b200 import pipeline as gp
from synth.configs import make_problem
prob = make_problem(4); ctx = Context(0); st = torch.cuda.current_stream()
N = prob.N; q = prob.rhs(); dt = 0.005 * prob.phi * N / float(q[q > 0].sum())
phi = torch.full((N,), float(prob.phi), dtype=torch.float64, device="cuda")
mob = torch.as_tensor(gp.initial_mobility(prob, 1.0, 5.0), device="cuda")
op = gp.build_operator(ctx, prob); cart = Level.cartesian(ctx, op, prob.block)
cart.smooth(op, 300, prob.omega, prob.sweep_tol); op.set_mobility(mob)
S = torch.zeros(N, dtype=torch.float64, device="cuda"); x = torch.zeros(N, dtype=torch.float64, device="cuda")
acc = np.zeros(5); wall = np.zeros(5); its = 0
for n in range(20):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]; t = [time.perf_counter()]
    ev[0].record(st); cart.smooth(op, 5, prob.omega, -1.0); ev[1].record(st); t.append(time.perf_counter())
    cart.assemble(op); ev[2].record(st); t.append(time.perf_counter())
    solver = Solver(ctx, op, [cart], omega_s=prob.omega_s, nu=prob.nu, post_smooth=prob.post_smooth)
    sol = solver.iterate(x, None, prob.cycle_tol, prob.max_iter, 0, history=False); solver.close(); ev[3].record(st); t.append(time.perf_counter())
    nsub = op.transport_upwind(x, S, phi, 1.0, 5.0, dt, mob_out=mob); ev[4].record(st); t.append(time.perf_counter())
    op.set_mobility(mob); ev[5].record(st); torch.cuda.synchronize(); t.append(time.perf_counter())
    acc += [ev[i].elapsed_time(ev[i+1]) for i in range(5)]; wall += np.diff(t); its += sol["iters"]
print(json.dumps(dict(steps=20, iters=its, gpu_ms=dict(zip(["smooth","assemble","solve","transport","mobility"], acc.round(1).tolist())), wall_ms=dict(zip(["smooth","assemble","solve","transport","mobility"], (wall*1e3).round(1).tolist())), nsub_last=nsub)))
