import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import make_problem
from oracle import pipeline as opl
from paper_2001_01624_b200 import Context
from paper_2001_01624_b200 import pipeline as gp
p = make_problem(1, dynamic=True)
orc = opl.run(p, record_dynamic=True)
k = orc["sol"]["iters"]
ctx = Context(0)
for fi in [5, 20, 50, k]:
    o = opl.run(p, fixed_iters=fi)
    g = gp.run(ctx, p, fixed_iters=fi)
    x = g["x"].cpu().numpy()
    err = np.linalg.norm(x - o["sol"]["x"]) / np.linalg.norm(o["sol"]["x"])
    dm_o = np.array(o["sol"]["dyn_M"]); dm_g = g["sol"]["dyn_M"][1:]
    print(fi, "err", err, "dynM equal", np.array_equal(dm_o, dm_g[:len(dm_o)]), dm_o[:8], dm_g[:8])
    rr = np.abs(g["sol"]["res"] - o["sol"]["res"]) / o["sol"]["res"]
    print("   res rel diff max", rr.max(), "first >1e-8 at", np.argmax(rr > 1e-8) if (rr > 1e-8).any() else None)
