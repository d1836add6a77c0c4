import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.configs import make_problem
from oracle import pipeline as opl, partition as opart, cycle as ocyc, coarse as oco, tpfa
from paper_2001_01624_b200 import Context, Level
from paper_2001_01624_b200 import pipeline as gp
p = make_problem(1, shape=(32, 32), block=(8, 8, 1), max_sweeps=60, dynamic=True)
orc = opl.run(p, fixed_iters=1)
dp = orc["sol"]["x"].copy()
part_o, M_o = opart.dynamic_partition(dp, p.nx, p.ny, p.nz)
A_T, A, q, _ = tpfa.build(p)
ref = oco.galerkin(ocyc.constant_basis(part_o, M_o), A)
print("oracle M", M_o, ref, np.linalg.eigvalsh(ref))
ctx = Context(0)
op = gp.build_operator(ctx, p)
levels, _ = gp.build_levels(ctx, op, p)
s = gp.make_solver(ctx, op, levels, p)
part_g = np.zeros(p.N, dtype=np.int32)
try:
    M_g = s.add_dynamic_basis(dp, part_g)
    print("M", M_g, np.array_equal(part_g, part_o))
except Exception as e:
    print("add_dynamic failed", e, np.array_equal(part_g, part_o), part_g.max(), np.bincount(part_g))
cl = Level.constant(ctx, op, part_o.astype(np.int32), M_o)
try:
    cl.assemble(op)
    print("const assemble ok")
except Exception as e:
    print("const assemble failed", e)
    _, _, _, Ac = cl.export(with_Ac=True)
    print(Ac)
