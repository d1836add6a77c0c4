"""ncu launch-list target: config 3 at full size, levels built with 20 sweeps, 6 cycles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2001_01624_b200 import Context
from paper_2001_01624_b200 import pipeline as gp
from synth.configs import make_problem
prob = make_problem(3)
ctx = Context(0)
op = gp.build_operator(ctx, prob)
levels, _ = gp.build_levels(ctx, op, prob, sweeps=20, fixed=True)
s = gp.make_solver(ctx, op, levels, prob)
x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
out = s.iterate(x, None, 1e-6, 100, 6)
torch.cuda.synchronize()
print("ok", out["iters"])
