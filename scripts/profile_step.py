"""Reduced step for ncu: config2 full grid, fixed 12 sweeps, assemble, fixed 12 cycles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_01624_b200 import Context, Level, Operator, Solver
from paper_2001_01624_b200 import pipeline as gp
from synth.configs import make_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = make_problem(cfg)
ctx = Context(0)
op = gp.build_operator(ctx, prob)
lev = Level.cartesian(ctx, op, prob.block)
lev.smooth(op, 12, prob.omega, -1.0)
lev.assemble(op)
s = Solver(ctx, op, [lev], prob.omega_s, prob.nu, prob.post_smooth)
x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
its = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = s.iterate(x, None, 1e-6, max(100, its), its)
torch.cuda.synchronize()
print("ok", out["iters"], out["res"][-1])
