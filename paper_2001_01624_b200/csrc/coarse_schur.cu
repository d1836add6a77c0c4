// Row a5 for large Cartesian coarse grids (config 5: M = 20,000): a direct solver that
// is a one-level nested dissection of the coarse grid.
//
// The paper inverts the coarse matrix by "direct Gaussian elimination" at O(M^p) cost,
// p ~ 2 for the sparse A_c; SURVEY §8.a5 names a band factor for config 5
// (half-bandwidth 841), whose two triangular solves are 2 M dependent steps — on a GPU a
// chain of ~600 latency-bound block steps.  Instead the coarse grid (nb0 x nb1 x nb2 blocks,
// A_c a box stencil of reach r_a <= 2 per axis, coarse.cu) is cut by separator slabs of
// thickness r_a into independent domains d and one separator set S:
//     A_c = [A_DD  A_DS]      A_DD = diag(A_dd) (domains do not couple),
//           [A_SD  A_SS],     Schur complement  C = A_SS - sum_d A_Sd A_dd^{-1} A_dS,
// and every solve x_c = A_c^{-1} r_c is
//     y_d = A_dd^{-1} r_d                   (batched packed SYMV, all domains at once)
//     t   = r_S - sum_d A_Sd y_d           (sparse, one thread per separator node)
//     x_S = C^{-1} t                        (packed SYMV)
//     u_d = r_d - A_dS x_S                  (sparse, one thread per domain node)
//     x_d = A_dd^{-1} u_d                   (batched packed SYMV)
// — block Gaussian elimination of A_c in the order (domains, separator), exact up to
// rounding (the same matrix, a different elimination order than the band LU).  The
// explicit inverses A_dd^{-1} and C^{-1} come from the dense recursive Cholesky + inverse
// of coarse_factor.cu (reading B1), so each phase is a fully parallel HBM stream:
// 8 sum_d |d|(|d|+64) + 4 |S|(|S|+64) bytes per solve (config 5: ~210 MB, against 1.6 GB
// for the packed dense inverse and 270 MB for the band factor's two sweeps).
// Setup: C is formed with two fp64 tensor-core GEMMs per domain, Z_d = A_dd^{-1} B_d and
// B_d^T Z_d (B_d = A_dS_d, dense over the separator nodes S_d coupled to d), subtracted
// into C one domain after another (fixed order: deterministic).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"
#include "symv.cuh"

namespace msb {

constexpr int SW = 125, SC = 62;  // box-stencil slots per row, centre slot (coarse.cu)

struct Schur {
  int M = 0, nd = 0, nD = 0, nS = 0;  // nodes, domains, domain nodes, separator nodes
  int32_t* node_pos = nullptr;   // [M] p >= 0: domain-order position; -(q+1): separator q
  int32_t* dom_nodes = nullptr;  // [nD] coarse node of domain position p
  int32_t* sep_nodes = nullptr;  // [nS]
  double* Xd = nullptr;          // packed tiles of every A_dd^{-1}
  double* partd = nullptr;
  SymvTile* td = nullptr;        // domain tile / row descriptors
  SymvRow* rd = nullptr;
  int ntd = 0, nrd = 0;
  Coarse C;                      // Schur complement: dense factor, packed inverse C.Xp
  SymvTile* tc = nullptr;
  SymvRow* rcd = nullptr;
  int ntc = 0, nrc = 0;
  double* y = nullptr;           // [nD]
  double* u = nullptr;           // [nD]
  double* t = nullptr;           // [nS]
  double* xs = nullptr;          // [nS]
  int64_t solve_bytes = 0;
};

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ int box_nb(int a, int d, int n0, int n1, int n2) {
  const int ax = a % n0, ay = (a / n0) % n1, az = a / (n0 * n1);
  const int bx = ax + d % 5 - 2, by = ay + (d / 5) % 5 - 2, bz = az + d / 25 - 2;
  if (bx < 0 || bx >= n0 || by < 0 || by >= n1 || bz < 0 || bz >= n2) return -1;
  return bx + n0 * (by + n1 * bz);
}

// out (nr x ncol, row-major, zero-filled) += the entries A_c(rows[i], K) with
// colmap[K] >= 0, at column colmap[K]
__global__ void k_extract(const double* __restrict__ Aell, int n0, int n1, int n2,
                          const int32_t* __restrict__ rows, int nr,
                          const int32_t* __restrict__ colmap, int ncol, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nr * SW) return;
  const int i = (int)(e / SW), d = (int)(e - (int64_t)i * SW);
  const int a = rows[i];
  const int b = d == SC ? a : box_nb(a, d, n0, n1, n2);
  if (b < 0) return;
  const int j = colmap[b];
  if (j >= 0) out[(int64_t)i * ncol + j] = Aell[(int64_t)a * SW + d];
}

__global__ void k_fill_map(int32_t* __restrict__ p, int64_t n, int32_t v) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}

__global__ void k_set_map(int32_t* __restrict__ map, const int32_t* __restrict__ list, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) map[list[i]] = i;
}

// C[idx[i], idx[j]] -= G[i, j]   (G: n x n row-major)
__global__ void k_scatter_sub(double* __restrict__ C, int ldc, const int32_t* __restrict__ idx,
                              int n, const double* __restrict__ G) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
  C[(int64_t)idx[i] * ldc + idx[j]] -= G[e];
}

// t_q = r_c[s_q] - sum over s_q's domain neighbours K of A_c(s_q, K) y[pos(K)]: one warp
// per separator node, lanes over the 125 stencil slots (coalesced row of A_c, the
// neighbour loads of all slots in flight together), then a fixed shuffle tree
__global__ void __launch_bounds__(256) k_schur_t(const double* __restrict__ Aell, int n0, int n1,
                                                 int n2, const int32_t* __restrict__ sep_nodes,
                                                 int nS, const int32_t* __restrict__ node_pos,
                                                 const double* __restrict__ rc,
                                                 const double* __restrict__ y,
                                                 double* __restrict__ t) {
  pdl_wait();  // y comes from the domain solve
  pdl_trigger();
  const int q = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nS) return;  // warp-uniform
  const int s = sep_nodes[q];
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int d = lane + 32 * u;
    const int K = d < SW ? box_nb(s, d, n0, n1, n2) : -1;
    const int p = K >= 0 ? node_pos[K] : -1;
    if (p >= 0) v = fma(Aell[(int64_t)s * SW + d], y[p], v);
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) t[q] = rc[s] - v;
}

// u_p = r_c[J_p] - sum over J_p's separator neighbours K of A_c(J_p, K) x_S[q(K)] (one warp
// per domain node, as k_schur_t); warps past nD write the separator part of x_c (x_S
// scattered), done-guarded
__global__ void __launch_bounds__(256) k_schur_u(const double* __restrict__ Aell, int n0, int n1,
                                                 int n2, const int32_t* __restrict__ dom_nodes,
                                                 int nD, const int32_t* __restrict__ sep_nodes,
                                                 int nS, const int32_t* __restrict__ node_pos,
                                                 const double* __restrict__ rc,
                                                 const double* __restrict__ xs,
                                                 double* __restrict__ u, double* __restrict__ xc,
                                                 const int* done) {
  pdl_wait();  // x_S comes from the separator solve
  pdl_trigger();
  const int w = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w < nD) {
    const int J = dom_nodes[w];
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int d = lane + 32 * k;
      const int K = d < SW ? box_nb(J, d, n0, n1, n2) : -1;
      const int q = K >= 0 ? node_pos[K] : 0;
      if (q < 0) v = fma(Aell[(int64_t)J * SW + d], xs[-q - 1], v);
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) u[w] = rc[J] - v;
  } else {
    const bool skip = done && *(volatile const int*)done;
    const int q = (w - nD) * 32 + lane;  // 32 separator entries per trailing warp
    if (q < nS && !skip) xc[sep_nodes[q]] = xs[q];
  }
}

// ---------------------------------------------------------------- planning (host)
// Open-box support range of block J along one axis (reading A3; cycle.cu support_range).
static void support_range_h(int J, int b, int n, int nb, int& x0, int& x1) {
  x0 = 0;
  x1 = n;
  if (J > 0) {
    const int lo = (J - 1) * b;
    x0 = (lo + std::min(lo + b, n) + 1) >> 1;
  }
  if (J < nb - 1) {
    const int lo = (J + 1) * b;
    x1 = (lo + std::min(lo + b, n)) >> 1;
  }
}

// coupling reach along one axis: the largest block distance whose supports touch
static int axis_reach(int b, int n, int nb) {
  int r = 0;
  for (int J = 0; J < nb; ++J)
    for (int K = J + 1; K < nb && K <= J + 2; ++K) {
      int a0, a1, c0, c1;
      support_range_h(J, b, n, nb, a0, a1);
      support_range_h(K, b, n, nb, c0, c1);
      if (c0 <= a1) r = std::max(r, K - J);  // overlapping or face-adjacent supports
    }
  return std::max(r, 1);
}

struct AxisSplit {
  std::vector<int> seg;   // coordinate -> domain slab index, or -1 in a separator slab
  std::vector<int> lo, hi;  // domain slab ranges
};

static AxisSplit split_axis(int c, int s, int r) {
  AxisSplit A;
  A.seg.assign(c, -1);
  const int w = c - s * r;
  int x = 0;
  for (int k = 0; k <= s; ++k) {
    const int wk = w / (s + 1) + (k < w % (s + 1) ? 1 : 0);
    A.lo.push_back(x);
    for (int t = 0; t < wk; ++t) A.seg[x++] = k;
    A.hi.push_back(x);
    if (k < s) x += r;
  }
  return A;
}

struct Plan {
  int s[3] = {0, 0, 0};
  double bytes = 0;
  int nS = 0, maxd = 0, nd = 0;
};

static bool plan_split(const int c[3], const int r[3], Plan& best) {
  bool found = false;
  for (int sx = 0; sx <= 8; ++sx)
    for (int sy = 0; sy <= 8; ++sy)
      for (int sz = 0; sz <= 8; ++sz) {
        const int s[3] = {sx, sy, sz};
        bool ok = true;
        std::vector<int> ws[3];
        for (int a = 0; a < 3 && ok; ++a) {
          const int w = c[a] - s[a] * r[a];
          if (w < s[a] + 1) {
            ok = false;
            break;
          }
          for (int k = 0; k <= s[a]; ++k) ws[a].push_back(w / (s[a] + 1) + (k < w % (s[a] + 1) ? 1 : 0));
        }
        if (!ok) continue;
        const int M = c[0] * c[1] * c[2];
        double bytes = 0;
        int nD = 0, maxd = 0, nd = 0;
        for (int x : ws[0])
          for (int y : ws[1])
            for (int z : ws[2]) {
              const int d = x * y * z;
              bytes += 8.0 * d * (d + 64);
              nD += d;
              maxd = std::max(maxd, d);
              ++nd;
            }
        const int nS = M - nD;
        if (nd < 2 || nS > 8192 || maxd > 4096 || nd > 512) continue;
        bytes += 4.0 * nS * (nS + 64);
        if (!found || bytes < best.bytes) {
          found = true;
          best.bytes = bytes;
          for (int a = 0; a < 3; ++a) best.s[a] = s[a];
          best.nS = nS;
          best.maxd = maxd;
          best.nd = nd;
        }
      }
  return found;
}

// packed-tile descriptors of one matrix of order m (tiles from tile_base, rows from roff)
static void describe(int m, int64_t tile_base, int roff, std::vector<SymvTile>& td,
                     std::vector<SymvRow>& rd) {
  const int ntb = (m + ST - 1) / ST;
  const int64_t nt = (int64_t)ntb * (ntb + 1) / 2;
  for (int64_t t = 0; t < nt; ++t) td.push_back(SymvTile{tile_base, m, roff, (int)t});
  for (int b = 0; b < ntb; ++b) rd.push_back(SymvRow{tile_base, m, ntb, b, roff});
}

template <class T>
static T* upload(msb_ctx ctx, const std::vector<T>& h) {
  T* d = dalloc_n<T>(ctx, h.size() + 1);
  if (d && !h.empty() &&
      cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream) !=
          cudaSuccess) {
    dfree(ctx, d);
    return nullptr;
  }
  return d;
}

void coarse_schur_free(msb_ctx ctx, Coarse& co) {
  Schur* S = co.sch;
  if (!S) return;
  for (void* p : {(void*)S->node_pos, (void*)S->dom_nodes, (void*)S->sep_nodes, (void*)S->Xd,
                  (void*)S->partd, (void*)S->td, (void*)S->rd, (void*)S->tc, (void*)S->rcd,
                  (void*)S->y, (void*)S->u, (void*)S->t, (void*)S->xs})
    dfree(ctx, p);
  coarse_free(ctx, S->C);
  delete S;
  co.sch = nullptr;
}

msb_status coarse_schur_setup(msb_ctx ctx, Coarse& co, const msb_level_s& L) {
  const int c[3] = {L.nb[0], L.nb[1], L.nb[2]};
  const int dims[3] = {L.nx, L.ny, L.nz};
  int r[3];
  for (int a = 0; a < 3; ++a) r[a] = axis_reach(L.bs[a], dims[a], c[a]);
  Plan pl;
  if (!plan_split(c, r, pl)) return set_error(ctx, MSB_EINVAL, "no separator split of the coarse grid");
  const int M = c[0] * c[1] * c[2];
  AxisSplit ax[3];
  for (int a = 0; a < 3; ++a) ax[a] = split_axis(c[a], pl.s[a], r[a]);
  const int ndx = pl.s[0] + 1, ndy = pl.s[1] + 1;
  // classify nodes (natural order: domain lists and the separator stay in natural order)
  std::vector<std::vector<int32_t>> dl(pl.nd);
  std::vector<int32_t> sep;
  std::vector<int32_t> dom_of(M);
  for (int J = 0; J < M; ++J) {
    const int x = J % c[0], y = (J / c[0]) % c[1], z = J / (c[0] * c[1]);
    const int gx = ax[0].seg[x], gy = ax[1].seg[y], gz = ax[2].seg[z];
    if (gx < 0 || gy < 0 || gz < 0) {
      dom_of[J] = -1;
      sep.push_back(J);
    } else {
      const int d = gx + ndx * (gy + ndy * gz);
      dom_of[J] = d;
      dl[d].push_back(J);
    }
  }
  Schur* S = new Schur();
  co.sch = S;
  S->M = M;
  S->nd = pl.nd;
  S->nS = (int)sep.size();
  std::vector<int32_t> node_pos(M), dom_nodes, dom_off(pl.nd + 1, 0);
  for (int d = 0; d < pl.nd; ++d) {
    dom_off[d + 1] = dom_off[d] + (int)dl[d].size();
    for (int32_t J : dl[d]) {
      node_pos[J] = (int32_t)dom_nodes.size();
      dom_nodes.push_back(J);
    }
  }
  for (int q = 0; q < S->nS; ++q) node_pos[sep[q]] = -(q + 1);
  S->nD = (int)dom_nodes.size();
  // separator nodes coupled to each domain: within the reach box of the domain's box
  std::vector<std::vector<int32_t>> sd(pl.nd);  // separator indices q
  for (int q = 0; q < S->nS; ++q) {
    const int J = sep[q];
    const int x[3] = {J % c[0], (J / c[0]) % c[1], J / (c[0] * c[1])};
    for (int d = 0; d < pl.nd; ++d) {
      const int g[3] = {d % ndx, (d / ndx) % ndy, d / (ndx * ndy)};
      bool near = true;
      for (int a = 0; a < 3 && near; ++a) {
        const int lo = ax[a].lo[g[a]], hi = ax[a].hi[g[a]] - 1;
        const int dist = x[a] < lo ? lo - x[a] : (x[a] > hi ? x[a] - hi : 0);
        near = dist <= r[a];
      }
      if (near) sd[d].push_back(q);
    }
  }
  cudaStream_t st = ctx->stream;
  S->node_pos = upload(ctx, node_pos);
  S->dom_nodes = upload(ctx, dom_nodes);
  S->sep_nodes = upload(ctx, sep);
  MSB_ALLOC(ctx, S->y, double, S->nD);
  MSB_ALLOC(ctx, S->u, double, S->nD);
  MSB_ALLOC(ctx, S->t, double, S->nS);
  MSB_ALLOC(ctx, S->xs, double, S->nS);
  if (!S->node_pos || !S->dom_nodes || !S->sep_nodes) return set_error(ctx, MSB_ENOMEM, "schur maps");
  // domain tile layout
  std::vector<SymvTile> td;
  std::vector<SymvRow> rd;
  std::vector<int64_t> tbase(pl.nd + 1, 0);
  for (int d = 0; d < pl.nd; ++d) {
    const int m = (int)dl[d].size();
    const int ntb = (m + ST - 1) / ST;
    tbase[d + 1] = tbase[d] + (int64_t)ntb * (ntb + 1) / 2;
    describe(m, tbase[d], dom_off[d], td, rd);
  }
  MSB_ALLOC(ctx, S->Xd, double, tbase[pl.nd] * ST * ST);
  S->td = upload(ctx, td);
  S->rd = upload(ctx, rd);
  S->ntd = (int)td.size();
  S->nrd = (int)rd.size();
  MSB_ALLOC(ctx, S->partd, double, tbase[pl.nd] * 2 * ST);
  if (!S->td || !S->rd) return set_error(ctx, MSB_ENOMEM, "schur descriptors");
  // the Schur complement starts as A_SS
  Coarse& C = S->C;
  C.M = S->nS;
  MSB_ALLOC(ctx, C.Ac, double, (int64_t)S->nS * S->nS);
  C.cap = S->nS;
  int32_t* colmap = nullptr;
  MSB_ALLOC(ctx, colmap, int32_t, M);
  auto fill_map = [&](const int32_t* list_dev, int n) -> msb_status {
    k_fill_map<<<grid_for(M, 256), 256, 0, st>>>(colmap, M, -1);
    MSB_LAUNCH_CHECK(ctx);
    if (n > 0) {
      k_set_map<<<grid_for(n, 256), 256, 0, st>>>(colmap, list_dev, n);
      MSB_LAUNCH_CHECK(ctx);
    }
    return MSB_OK;
  };
  msb_status rc = fill_map(S->sep_nodes, S->nS);
  if (rc) return rc;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(C.Ac, 0, (size_t)S->nS * S->nS * sizeof(double), st));
  k_extract<<<grid_for((int64_t)S->nS * SW, 256), 256, 0, st>>>(co.Aell, c[0], c[1], c[2],
                                                                S->sep_nodes, S->nS, colmap, S->nS,
                                                                C.Ac);
  MSB_LAUNCH_CHECK(ctx);
  // per domain: factor + inverse A_dd, then C -= B_d^T A_dd^{-1} B_d
  int maxd = 0, maxs = 0;
  for (int d = 0; d < pl.nd; ++d) {
    maxd = std::max(maxd, (int)dl[d].size());
    maxs = std::max(maxs, (int)sd[d].size());
  }
  double *B = nullptr, *Z = nullptr, *G = nullptr;
  int32_t* sidx = nullptr;
  int32_t* snodes = nullptr;
  MSB_ALLOC(ctx, B, double, (int64_t)maxd * std::max(maxs, 1));
  MSB_ALLOC(ctx, Z, double, (int64_t)maxd * std::max(maxs, 1));
  MSB_ALLOC(ctx, G, double, (int64_t)std::max(maxs, 1) * std::max(maxs, 1));
  MSB_ALLOC(ctx, sidx, int32_t, std::max(maxs, 1));
  MSB_ALLOC(ctx, snodes, int32_t, std::max(maxs, 1));
  Coarse D;  // one domain's dense factor (reused)
  std::vector<int32_t> hn;
  for (int d = 0; d < pl.nd && !rc; ++d) {
    const int m = (int)dl[d].size(), ns = (int)sd[d].size();
    D.M = m;
    if (D.cap < m) {
      coarse_free(ctx, D);
      MSB_ALLOC(ctx, D.Ac, double, (int64_t)maxd * maxd);
      MSB_ALLOC(ctx, D.L, double, (int64_t)maxd * maxd);
      MSB_ALLOC(ctx, D.Ainv, double, (int64_t)maxd * maxd);
      D.cap = maxd;
    }
    const int32_t* rows = S->dom_nodes + dom_off[d];
    if ((rc = fill_map(rows, m))) break;
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(D.Ac, 0, (size_t)m * m * sizeof(double), st));
    k_extract<<<grid_for((int64_t)m * SW, 256), 256, 0, st>>>(co.Aell, c[0], c[1], c[2], rows, m,
                                                             colmap, m, D.Ac);
    MSB_LAUNCH_CHECK(ctx);
    if ((rc = coarse_factor_dense(ctx, D))) break;  // D.Ainv = A_dd^{-1}, D.Xp packed
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(S->Xd + tbase[d] * ST * ST, D.Xp,
                                      (size_t)(tbase[d + 1] - tbase[d]) * ST * ST * sizeof(double),
                                      cudaMemcpyDeviceToDevice, st));
    if (ns == 0) continue;
    hn.resize(ns);
    for (int k = 0; k < ns; ++k) hn[k] = sep[sd[d][k]];
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(snodes, hn.data(), ns * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(sidx, sd[d].data(), ns * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    if ((rc = fill_map(snodes, ns))) break;
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(B, 0, (size_t)m * ns * sizeof(double), st));
    k_extract<<<grid_for((int64_t)m * SW, 256), 256, 0, st>>>(co.Aell, c[0], c[1], c[2], rows, m,
                                                             colmap, ns, B);
    MSB_LAUNCH_CHECK(ctx);
    if ((rc = dgemm(ctx, false, false, m, ns, m, 1.0, D.Ainv, m, B, ns, 0.0, Z, ns))) break;
    if ((rc = dgemm(ctx, true, false, ns, ns, m, 1.0, B, ns, Z, ns, 0.0, G, ns))) break;
    k_scatter_sub<<<grid_for((int64_t)ns * ns, 256), 256, 0, st>>>(C.Ac, S->nS, sidx, ns, G);
    MSB_LAUNCH_CHECK(ctx);
    // hn / sd[d] host buffers are read by the async copies above: drain before reuse
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  cudaStreamSynchronize(st);
  coarse_free(ctx, D);
  for (void* p : {(void*)B, (void*)Z, (void*)G, (void*)sidx, (void*)snodes, (void*)colmap}) dfree(ctx, p);
  if (rc) return rc;
  if ((rc = coarse_factor_dense(ctx, C))) return rc;
  std::vector<SymvTile> tc;
  std::vector<SymvRow> rcd;
  describe(S->nS, 0, 0, tc, rcd);
  S->tc = upload(ctx, tc);
  S->rcd = upload(ctx, rcd);
  S->ntc = (int)tc.size();
  S->nrc = (int)rcd.size();
  if (!S->tc || !S->rcd) return set_error(ctx, MSB_ENOMEM, "schur descriptors");
  S->solve_bytes = (int64_t)(2 * 8 * tbase[pl.nd] * ST * ST / 2 + 8 * (int64_t)S->ntc * ST * ST);
  // the separator factor's dense buffers are setup-only
  dfree(ctx, C.Ac);
  dfree(ctx, C.L);
  dfree(ctx, C.Ainv);
  C.Ac = C.L = C.Ainv = nullptr;
  C.cap = 0;
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MSB_OK;
}

void coarse_schur_solve(msb_ctx ctx, const Coarse& co, const double* rc, double* xc, const int* done) {
  const Schur* S = co.sch;
  cudaStream_t st = ctx->stream;
  const int n0 = co.nb[0], n1 = co.nb[1], n2 = co.nb[2];
  // y_d = A_dd^{-1} r_d (r_c read through the domain node map)
  symv_batched(ctx, S->td, S->ntd, S->rd, S->nrd, S->Xd, rc, S->dom_nodes, S->partd, S->y, nullptr,
               nullptr);
  launch_ex(k_schur_t, dim3(grid_for((int64_t)S->nS * 32, 256)), dim3(256), 0, st, kPDL, 1, co.Aell,
            n0, n1, n2, S->sep_nodes, S->nS, S->node_pos, rc, S->y, S->t);
  count_launch();
  symv_batched(ctx, S->tc, S->ntc, S->rcd, S->nrc, S->C.Xp, S->t, nullptr, S->C.part, S->xs,
               nullptr, nullptr);
  const int64_t wu = (int64_t)S->nD + (S->nS + 31) / 32;  // warps
  launch_ex(k_schur_u, dim3(grid_for(wu * 32, 256)), dim3(256), 0, st, kPDL, 1, co.Aell, n0, n1, n2,
            S->dom_nodes, S->nD, S->sep_nodes, S->nS, S->node_pos, rc, S->xs, S->u, xc, done);
  count_launch();
  symv_batched(ctx, S->td, S->ntd, S->rd, S->nrd, S->Xd, S->u, nullptr, S->partd, xc, S->dom_nodes,
               done);
}

}  // namespace msb
