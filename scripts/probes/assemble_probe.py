"""Host wall time of one constant-basis coarse assembly (exact RAP + factor + inverse) on
the config-3 grid, the dynamic stage's per-iteration rebuild, at several M."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2001_01624_b200 import Context, Level
from paper_2001_01624_b200 import pipeline as gp
from synth.configs import make_problem

prob = make_problem(3)
ctx = Context(0)
op = gp.build_operator(ctx, prob)
N = prob.N
Ms = [int(a) for a in sys.argv[1:]] or [40, 165, 168, 200, 400]
for M in Ms:
    part = (np.arange(N, dtype=np.int64) * M // N).astype(np.int32)  # M contiguous slabs
    lev = Level.constant(ctx, op, part, M)
    for _ in range(3):
        lev.assemble(op)
    torch.cuda.synchronize()
    reps = 30
    t0 = time.perf_counter()
    for _ in range(reps):
        lev.assemble(op)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps * 1e6
    print(f"M={M:4d} assemble {dt:8.1f} us/call", flush=True)
