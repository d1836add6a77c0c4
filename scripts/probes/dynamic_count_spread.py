import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from synth.configs import make_problem
from oracle import pipeline as opl, cycle as ocy
from paper_2001_01624_b200 import Context
from paper_2001_01624_b200 import pipeline as gp
import scipy.linalg as la
prob = make_problem(1, dynamic=True)
ctx = Context(0)
print("gpu", [gp.run(ctx, prob)["sol"]["iters"] for _ in range(6)])
class PLU:
    seed = 0
    def __init__(self, Ac):
        self._lu = la.lu_factor(Ac); PLU.seed += 1; self._rng = np.random.default_rng(PLU.seed)
    def solve(self, rc):
        x = la.lu_solve(self._lu, rc)
        return x * (1.0 + 4 * np.finfo(float).eps * self._rng.uniform(-1.0, 1.0, x.shape))
saved = ocy.CoarseSolver
ks = []
for s0 in range(6):
    PLU.seed = 1000 * s0
    ocy.CoarseSolver = PLU
    ks.append(opl.run(prob)["sol"]["iters"])
ocy.CoarseSolver = saved
print("oracle", opl.run(prob)["sol"]["iters"], "perturbed seeds", ks)
