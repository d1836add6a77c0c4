"""ncu target: a few config-2 ILU(0) iterations and one config-4 transport call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2001_01624_b200 import Context, Level, Solver
from paper_2001_01624_b200 import pipeline as gp
from synth.configs import make_problem
prob = make_problem(2, smoother="ilu0")
ctx = Context(0)
op = gp.build_operator(ctx, prob)
lev = Level.cartesian(ctx, op, prob.block)
lev.smooth(op, 12, prob.omega, -1.0)
lev.assemble(op)
s = Solver(ctx, op, [lev], prob.omega_s, prob.nu, prob.post_smooth, smoother="ilu0")
x = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
s.iterate(x, None, 1e-6, 100, 4)
phi = torch.full((prob.N,), 0.2, dtype=torch.float64, device="cuda")
S = torch.zeros(prob.N, dtype=torch.float64, device="cuda")
n = op.transport_upwind(x, S, phi, 1.0, 5.0, 1e-3)
torch.cuda.synchronize()
print("ok", n)
