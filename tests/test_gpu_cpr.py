"""GPU parity of §8 NEXT-4 (the CPR two-stage preconditioner)
through the C ABI against oracle/cpr.py on the same seeded inputs:
  F, J (analytic on the device vs the oracle's complex step)   <= 1e-11 of each block's max
  weights, J*, F*                                                <= 1e-12 relative
  A_c = P^T J*_pp P                                              <= 1e-12 max|A_c|
  cpr_apply(r)                                                   <= 1e-9 relative (the coarse
        inverse is explicit Gauss–Jordan on the device, LU in the oracle: cond(A_c) eps)
  FGMRES counts                                                  within ±1 of the oracle's
"""
import numpy as np
import pytest

from synth.configs import cpr_state, make_problem

from conftest import record_parity

pytestmark = pytest.mark.gpu

SWEEPS = 40


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2001_01624_b200 import Context
    return Context(0)


CASES = {
    "small": dict(shape=(12, 10, 4), block=(4, 5, 2), seed=3),
    "ragged": dict(shape=(17, 13, 5), block=(5, 4, 3), seed=4),
    "linear_rp": dict(shape=(12, 10, 4), block=(4, 5, 2), seed=5, nrel=1),
}


def _fluid(nrel=2):
    from oracle import cpr as ocpr
    return ocpr.Fluid(nrel=nrel)


def _setup(ctx, case):
    from oracle import cpr as ocpr
    from oracle import pipeline as opl
    from oracle import tpfa
    from paper_2001_01624_b200 import Cpr, Level
    from paper_2001_01624_b200.pipeline import build_operator
    c = CASES[case]
    prob = make_problem(2, shape=c["shape"], block=c["block"])
    st = cpr_state(prob, seed=c["seed"])
    fl = _fluid(c.get("nrel", 2))
    tr = tpfa.transmissibilities(prob)
    N = prob.N
    J = ocpr.jacobian(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells, st.well_rates)
    F = np.concatenate(ocpr.residual(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells,
                                     st.well_rates))
    A_T = tpfa.flux_matrix(N, tr)
    cart = opl.cartesian_level(prob, A_T, SWEEPS, True)
    op = build_operator(ctx, prob)
    lev = Level.cartesian(ctx, op, prob.block)
    lev.smooth(op, SWEEPS, prob.omega, -1.0)
    cpr = Cpr(ctx, op, lev, vars(fl))
    q = np.zeros(N)
    np.add.at(q, st.well_cells, st.well_rates)
    cpr.linearize(st.p, st.S, st.p_n, st.S_n, q)
    return dict(prob=prob, st=st, fl=fl, J=J, F=F, cart=cart, op=op, lev=lev, cpr=cpr)


def _planes(J, nx, ny, nz):
    """oracle CSR -> the library's 28 planes [(2b+v)][d][c]"""
    from oracle.cpr import _neighbours
    N = nx * ny * nz
    nb = _neighbours(nx, ny, nz)
    out = np.zeros((2, 2, 7, N))
    Jc = J.tocsr()
    for b in range(2):
        for v in range(2):
            for d in range(7):
                ok = nb[d] >= 0
                rows = b * N + np.nonzero(ok)[0]
                cols = v * N + nb[d][ok]
                out[b, v, d, ok] = np.asarray(Jc[rows, cols]).ravel()
    return out


@pytest.mark.parametrize("case", list(CASES))
def test_linearize_parity(ctx, case):
    s = _setup(ctx, case)
    prob = s["prob"]
    g = s["cpr"].export(decoupled=False)
    errF = np.max(np.abs(g["F"] - s["F"])) / np.max(np.abs(s["F"]))
    ref = _planes(s["J"], prob.nx, prob.ny, prob.nz)
    errJ = 0.0
    for b in range(2):
        for v in range(2):
            scale = np.max(np.abs(ref[b, v]))
            errJ = max(errJ, np.max(np.abs(g["J"][b, v] - ref[b, v])) / scale)
    record_parity(f"cpr/linearize/{case}", errF=errF, errJ=errJ, tol=1e-11)
    assert errF <= 1e-11, errF
    assert errJ <= 1e-11, errJ


@pytest.mark.parametrize("method", ["impes", "quasi"])
@pytest.mark.parametrize("case", ["small", "ragged"])
def test_decouple_and_coarse_parity(ctx, case, method):
    from oracle import cpr as ocpr
    from oracle.cycle import Level as OLevel
    s = _setup(ctx, case)
    prob, st, fl = s["prob"], s["st"], s["fl"]
    N = prob.N
    w = (ocpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n) if method == "impes"
         else ocpr.quasi_impes_weights(s["J"], N))
    Js, Fs = ocpr.premultiply(s["J"], s["F"], w)
    cpr = s["cpr"]
    cpr.decouple(method)
    g = cpr.export()
    errw = np.max(np.abs(g["w"] - w))
    assert errw <= 1e-12, errw
    refp = _planes(Js, prob.nx, prob.ny, prob.nz)
    errJs = max(np.max(np.abs(g["Js"][v] - refp[0, v])) / np.max(np.abs(refp[0, v]))
                for v in range(2))
    errFs = np.max(np.abs(g["Fs"] - Fs)) / np.max(np.abs(Fs))
    Ac_ref = OLevel(s["cart"]["P"].matrix(), Js[:N, :N]).Ac
    Ac_ref = Ac_ref.toarray() if hasattr(Ac_ref, "toarray") else np.asarray(Ac_ref)
    Ac = cpr.export_coarse()
    errAc = np.max(np.abs(Ac - Ac_ref)) / np.max(np.abs(Ac_ref))
    record_parity(f"cpr/decouple/{case}/{method}", errw=errw, errJs=errJs, errFs=errFs,
                  errAc=errAc, tol=1e-12)
    assert errJs <= 1e-11, errJs
    assert errFs <= 1e-11, errFs
    assert errAc <= 1e-12, errAc


def _oracle_cpr(s, method):
    from oracle import cpr as ocpr
    from oracle.cycle import Level as OLevel
    prob, st, fl = s["prob"], s["st"], s["fl"]
    N = prob.N
    w = (ocpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n) if method == "impes"
         else ocpr.quasi_impes_weights(s["J"], N))
    Js, Fs = ocpr.premultiply(s["J"], s["F"], w)
    lev = OLevel(s["cart"]["P"].matrix(), Js[:N, :N])
    return ocpr.CPR(Js, N, [lev], prob.nx, prob.ny, prob.nz), Js, Fs


@pytest.mark.parametrize("method", ["impes", "quasi"])
@pytest.mark.parametrize("case", ["small", "ragged", "linear_rp"])
def test_apply_parity(ctx, case, method):
    import torch
    s = _setup(ctx, case)
    N = s["prob"].N
    C, Js, Fs = _oracle_cpr(s, method)
    cpr = s["cpr"]
    cpr.decouple(method)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(2 * N)
    ref = C.apply(r)
    rd = torch.from_numpy(r).cuda()
    dx = torch.empty_like(rd)
    cpr.apply(rd, dx)
    err = np.max(np.abs(dx.cpu().numpy() - ref)) / np.max(np.abs(ref))
    # corrector alone (the ILU(0) of the full J*)
    refi = C.corrector(r)
    y = torch.empty_like(rd)
    cpr.apply_system(rd, y)
    erry = np.max(np.abs(y.cpu().numpy() - Js @ r)) / np.max(np.abs(Js @ r))
    record_parity(f"cpr/apply/{case}/{method}", err=err, err_system=erry, tol=1e-9)
    assert erry <= 1e-12, erry
    assert err <= 1e-9, err
    assert np.all(np.isfinite(refi))


@pytest.mark.parametrize("method", ["impes", "quasi"])
def test_fgmres_counts(ctx, method):
    from oracle import fgmres as ofg
    s = _setup(ctx, "small")
    N = s["prob"].N
    C, Js, Fs = _oracle_cpr(s, method)
    cpr = s["cpr"]
    cpr.decouple(method)
    out = {}
    for pre, M in (("cpr", C.apply), ("ilu0", C.corrector)):
        o = ofg.fgmres(Js, -Fs, np.zeros(2 * N), [], tol=1e-8, restart=30, max_iter=150,
                       precond=M)
        x = np.zeros(2 * N)
        g = cpr.fgmres(x, None, tol=1e-8, restart=30, max_iter=150, precond=pre)
        out[pre] = (g["iters"], o["iters"])
        if o["converged"]:
            assert abs(g["iters"] - o["iters"]) <= 1, (pre, g["iters"], o["iters"])
            rel = np.linalg.norm(x - o["x"]) / np.linalg.norm(o["x"])
            assert rel <= 1e-6, rel
        record_parity(f"cpr/fgmres/{method}/{pre}", k_gpu=g["iters"], k_oracle=o["iters"],
                      tol="±1")
    assert out["cpr"][0] < out["ilu0"][0]


def test_errors(ctx):
    from paper_2001_01624_b200 import Cpr, Level, MsbError
    from paper_2001_01624_b200.pipeline import build_operator
    prob = make_problem(2, shape=(8, 6, 3), block=(4, 3, 3))
    op = build_operator(ctx, prob)
    lev = Level.cartesian(ctx, op, prob.block)
    fl = vars(_fluid())
    with pytest.raises(MsbError):
        Cpr(ctx, op, lev, dict(fl, nrel=3))
    c = Cpr(ctx, op, lev, fl)
    with pytest.raises(MsbError):
        c.decouple("impes")  # before linearize
