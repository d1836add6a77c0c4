import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.configs import make_problem
from oracle import pipeline as opl, partition as opart, cycle as ocyc, coarse as oco
from paper_2001_01624_b200 import Context, Level
from paper_2001_01624_b200 import pipeline as gp
p = make_problem(1, shape=(32, 32), block=(8, 8, 1), max_sweeps=60, dynamic=True)
rng = np.random.default_rng(0)
dp = rng.standard_normal(p.N) ** 3
part_o, M_o = opart.dynamic_partition(dp, p.nx, p.ny, p.nz)
ctx = Context(0)
op = gp.build_operator(ctx, p)
levels, _ = gp.build_levels(ctx, op, p)
s = gp.make_solver(ctx, op, levels, p)
part_g = np.zeros(p.N, dtype=np.int32)
M_g = s.add_dynamic_basis(dp, part_g)
print("M", M_o, M_g, "labels equal", np.array_equal(part_o, part_g))
if not np.array_equal(part_o, part_g):
    print(part_o[:64]); print(part_g[:64])
cl = Level.constant(ctx, op, part_g, M_g)
try:
    cl.assemble(op)
    _, _, _, Ac = cl.export(with_Ac=True)
    from oracle import tpfa
    A_T, A, q, _ = tpfa.build(p)
    ref = oco.galerkin(ocyc.constant_basis(part_g.astype(np.int64), M_g), A)
    print("Ac err", np.abs(Ac - ref).max(), np.abs(ref).max())
except Exception as e:
    print("assemble failed", e)
    from oracle import tpfa
    A_T, A, q, _ = tpfa.build(p)
    ref = oco.galerkin(ocyc.constant_basis(part_g.astype(np.int64), M_g), A)
    print(ref[:5,:5], np.linalg.eigvalsh(ref)[:3])
