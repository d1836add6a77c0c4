"""Eq. (9) — the paper's operation-count model.

Per-stage counts: smooth 2Nd (ILU(0)), residual Nd+N,
update N; restrict Nd+N + b_ℓN; coarse M^p; prolong b_ℓN + N.  Cycle total
≈ (4d+2b+4) N_p N.  Garbled macros read per A21:
\\noverlapN = b·N, \\npartN = N_p·N, \\nsparseN_c = d·N_c, \\ncompN = N_c·N, giving
    c(N_p) = N [N_p(4d + 2b + 4) + N_c(d + 1) + N_c(2 d N_c + 1)].
TEST INFRASTRUCTURE ONLY (the bench derives its own byte counts).
"""


def cost_per_iteration(N, Np, d, b, Nc):
    return N * (Np * (4 * d + 2 * b + 4) + Nc * (d + 1) + Nc * (2 * d * Nc + 1))


def cost_breakdown(N, d, b, M, p=2):
    smooth = 2 * N * d + (N * d + N) + N
    restrict = (N * d + N) + b * N
    coarse = M ** p
    prolong = b * N + N
    return dict(smooth=smooth, restrict=restrict, coarse=coarse, prolong=prolong)
