// Rows a6–a11: the multibasis Richardson cycle (Eq. 8) and the
// dynamic Δp stage.
//
// Kernels (all HBM-bound, fp64, one thread per cell, coalesced SoA loads):
//   k_jacobi        x_out = x + ω_s D_A^{-1}(b - A x)           (a7; first kernel of an
//                   iteration also reduces ||b - A x||^2 -> stop test, a11)
//   k_res_restrict  r = b - A x, rc += P^T r                      (a6 + a8; warp-segmented
//                   sums over runs of equal columns, one fp64 atomic per run)
//   k_gemv          xc = A_c^{-1} rc                              (a5, coarse.cu)
//   k_prolong       x += P xc                                     (a9; row gather)
// Stop test on the device: the iteration's first kernel stores per-warp partial sums
// of r^2 (no barrier, no fence); a one-CTA k_finalize sums them in a fixed order
// (deterministic), records ρ_k and sets `done`; every later kernel of the enqueued
// chunk sees `done` and returns at once, so the host synchronises once per chunk.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include <chrono>
#include <cstdio>

#include "internal.cuh"
#include "symv.cuh"

struct IterState {
  int done;
  int k;          // completed iterations
  int converged;
  int diverged;
  int max_iter;
  int fixed;
  double tol;
  double bscale;  // ||b|| (1 if b = 0)
  double r0;
};

namespace msb {

constexpr int CT = 256;  // cycle kernel block size

struct StencilT {
  const double* Tx;
  const double* Ty;
  const double* Tz;
  Grid3 g;
};

// r = b - A x at cell c (gauge: A_00 doubled); returns r and D_A.
__device__ __forceinline__ double residual_at(const StencilT& S, const double* __restrict__ x,
                                              const double* __restrict__ b, int c, int i, int j,
                                              int k, double* DA) {
  const int nx = S.g.nx, sxy = S.g.nxy;
  double txp = S.Tx[c], typ = S.Ty[c], tzp = S.Tz[c];
  double txm = i > 0 ? S.Tx[c - 1] : 0.0;
  double tym = j > 0 ? S.Ty[c - nx] : 0.0;
  double tzm = k > 0 ? S.Tz[c - sxy] : 0.0;
  double D = txp + txm + typ + tym + tzp + tzm;
  double off = 0.0;
  if (k > 0) off += tzm * x[c - sxy];
  if (j > 0) off += tym * x[c - nx];
  if (i > 0) off += txm * x[c - 1];
  if (i < nx - 1) off += txp * x[c + 1];
  if (j < S.g.ny - 1) off += typ * x[c + nx];
  if (k < S.g.nz - 1) off += tzp * x[c + sxy];
  double dA = (c == 0) ? 2.0 * D : D;
  *DA = dA;
  return b[c] - (dA * x[c] - off);
}

// per-block partial sum -> partials[blockIdx] (one barrier, no fence, no atomics)
__device__ __forceinline__ void warp_partial(double v, double* __restrict__ partials) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (threadIdx.x == 0) partials[blockIdx.x] = w;
  }
}

__device__ __forceinline__ bool is_done(const IterState* st) {
  return *(volatile const int*)&st->done != 0;
}
// The streaming kernels read the flag at entry but test it only before their stores,
// so its L2 round trip overlaps the data loads instead of serialising every CTA.

// Stop test (a11): one CTA sums the per-warp partials in a fixed order (deterministic),
// records ρ_k and decides.  mode 1: store ||b||.
__global__ void __launch_bounds__(1024) k_finalize(const double* __restrict__ partials, int np,
                                                   int mode, IterState* st,
                                                   double* __restrict__ res) {
  if (mode == 0 && is_done(st)) return;
  __shared__ double sh[32];
  double s = 0.0;
  for (int t = threadIdx.x; t < np; t += blockDim.x) s += partials[t];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if (threadIdx.x != 0) return;
  double nrm = sqrt(w);
  if (mode == 1) {
    st->bscale = nrm > 0.0 ? nrm : 1.0;
    return;
  }
  int k = st->k;
  double rho = nrm / st->bscale;
  res[k] = rho;
  if (k == 0) st->r0 = nrm;
  int done = 0;
  if (st->fixed > 0) {
    if (k >= st->fixed) {
      done = 1;
      st->converged = rho <= st->tol;
    }
  } else if (rho <= st->tol) {
    done = 1;
    st->converged = 1;
  } else if (k >= st->max_iter) {
    done = 1;
  }
  if (!(nrm <= 1e6 * st->r0) && st->r0 > 0.0) {  // also catches NaN
    done = 1;
    st->diverged = 1;
  }
  if (done) st->done = 1;
  else st->k = k + 1;
}

__global__ void __launch_bounds__(CT) k_norm(StencilT S, const double* __restrict__ x,
                                             const double* __restrict__ b, int mode,
                                             double* __restrict__ partials, const IterState* st) {
  if (mode == 0 && is_done(st)) return;
  const int N = S.g.nxy * S.g.nz;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (c < N) {
    if (mode == 1) {
      v = b[c] * b[c];
    } else {
      int i, j, k;
      g3_coords(S.g, c, i, j, k);
      double dA;
      double r = residual_at(S, x, b, c, i, j, k, &dA);
      v = r * r;
    }
  }
  warp_partial(v, partials);
}

// a7: x_out = x + ω_s D_A^{-1}(b - A x); `first` also emits the ||r||^2 partials.
// CPT cells per thread (strided by the block size, so every load instruction stays
// coalesced): the loads of all CPT cells are in flight together and the grid is CPT
// times shorter, which is what a short stencil pass needs to approach HBM bandwidth.
constexpr int CPT = 4;
// On grids whose stencil working set (5 N doubles) is beyond L2 every load of a pass goes to
// HBM and the passes gain from more, shorter CTAs instead: CPT_BIG cells per thread (config 5:
// 527 -> 507 us per iteration with 2; 8 measured 556; on config 2 4 stays best: 63.5 us against
// 64.5 with 2 and 67.4 with 8; profiles/r02i/cells_per_thread_ab.txt)
constexpr int CPT_BIG = 2;
constexpr int CPT_WAVE = 6;  // residual pass of the single-level iteration: see enqueue_stage
constexpr int64_t CPT_BIG_MIN_N = 3200000;  // 5 N doubles > 128 MB

// Stencil passes launched as programmatic dependents: the inputs they do not write (the
// transmissibility planes incl. the -y/-z face planes, and b) are bulk-prefetched into L2
// for this CTA's cells, then the pass waits for its predecessor (which wrote x).
template <int CPT>
__device__ __forceinline__ void stencil_prologue(const StencilT& S, const double* b) {
  const int N = S.g.nxy * S.g.nz;
  const int cb = blockIdx.x * (CT * CPT);
  const int ce = min(cb + CT * CPT, N);
  const size_t n = (size_t)(ce - cb) * sizeof(double);
  switch (threadIdx.x) {
    case 0: prefetch_l2(S.Tx + max(cb - 1, 0), n + 8); break;
    case 32: prefetch_l2(S.Ty + cb, n); break;
    case 64: prefetch_l2(S.Tz + cb, n); break;
    case 96: prefetch_l2(b + cb, n); break;
    case 128: if (cb >= S.g.nx) prefetch_l2(S.Ty + cb - S.g.nx, n); break;
    case 160: if (cb >= S.g.nxy) prefetch_l2(S.Tz + cb - S.g.nxy, n); break;
    default: break;
  }
  pdl_wait();
  pdl_trigger();
}

template <int CPT>
__global__ void __launch_bounds__(CT) k_jacobi(StencilT S, const double* __restrict__ x,
                                               double* __restrict__ xo,
                                               const double* __restrict__ b, double omega,
                                               int first, double* __restrict__ partials,
                                               const IterState* st) {
  stencil_prologue<CPT>(S, b);
  const bool done = is_done(st);
  const int N = S.g.nxy * S.g.nz;
  const int c0 = blockIdx.x * (CT * CPT) + threadIdx.x;
  double r[CPT], dA[CPT], xv[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = min(c0 + u * CT, N - 1);
    int i, j, k;
    g3_coords(S.g, c, i, j, k);
    r[u] = residual_at(S, x, b, c, i, j, k, &dA[u]);
    xv[u] = x[c];
  }
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = c0 + u * CT;
    if (c < N) {
      if (!done) xo[c] = xv[u] + omega * div_rn(r[u], dA[u], rcp_fast(dA[u]));
      v += r[u] * r[u];
    }
  }
  if (first) warp_partial(v, partials);
}

struct LevelView {
  int kind, W, nb0, nb1, nb2, b0, b1, b2;
  Grid3 g;
  const int32_t* tab;
  const int32_t* col;
  const double* P;
  int unit;  // W = 1 with rows summing to one: every P entry is exactly 1, not read
};

__device__ __forceinline__ int lv_col(const LevelView& L, int c, int i, int j, int k, int s) {
  if (L.kind == 1) return L.col[(size_t)s * (L.g.nxy * L.g.nz) + c];
  int jx = L.tab[2 * i + (s & 1)], jy = L.tab[2 * (L.g.nx + j) + ((s >> 1) & 1)],
      jz = L.tab[2 * (L.g.nx + L.g.ny + k) + (s >> 2)];
  if (jx < 0 || jy < 0 || jz < 0) return -1;
  return jx + L.nb0 * (jy + L.nb1 * jz);
}

// Sum val over runs of equal key in consecutive lanes; the last lane of each run
// with key >= 0 adds the run total to out[key].
__device__ __forceinline__ void warp_segmented_add(int key, double val, double* __restrict__ out) {
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31;
  int prev = __shfl_up_sync(full, key, 1);
  int head = (lane == 0) || (prev != key);
  unsigned heads = __ballot_sync(full, head);
  int start = 31 - __clz(heads & ((2u << lane) - 1u));
  double s = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(full, s, o);
    if (lane - o >= start) s += y;
  }
  int next = __shfl_down_sync(full, key, 1);
  int tail = (lane == 31) || (next != key);
  if (tail && key >= 0) atomicAdd(out + key, s);
}

// a6 + a8: r = b - A x, rc += P^T r.
__global__ void __launch_bounds__(CT) k_res_restrict(StencilT S, LevelView L,
                                                     const double* __restrict__ x,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ rc, int first,
                                                     double* __restrict__ partials,
                                                     const IterState* st) {
  if (is_done(st)) return;
  const int N = S.g.nxy * S.g.nz;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  bool in = c < N;
  int cc = in ? c : N - 1;
  int i, j, k;
  g3_coords(S.g, cc, i, j, k);
  double r = 0.0;
  if (in) {
    double dA;
    r = residual_at(S, x, b, c, i, j, k, &dA);
  }
  if (L.kind == 0) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      int key = in ? lv_col(L, cc, i, j, k, s) : -1;
      double v = key >= 0 ? L.P[(size_t)s * N + c] * r : 0.0;
      warp_segmented_add(key, v, rc);
    }
  } else {
    for (int s = 0; s < L.W; ++s) {
      int key = in ? L.col[(size_t)s * N + c] : -1;
      double v = key >= 0 ? L.P[(size_t)s * N + c] * r : 0.0;
      warp_segmented_add(key, v, rc);
    }
  }
  if (first) warp_partial(r * r, partials);
}

// ---------------------------------------------------------------- NEXT-2: red-black ILU(0)
// ILU(0) of A in red-black ordering (red: i + j + k even; reading B12; oracle/ilu.py).
// With the 7-point stencil red cells couple only to black cells, so the factors keep A's
// off-diagonal entries: L = [I 0; A_br D_r^-1 I], U = [D_r A_rb; 0 D~_b] with
// D~_b = a_bb - sum_r a_br a_rb / a_rr over the red neighbours (the fill between black
// cells is dropped), and one smoothing step x += (LU)^{-1} r is three parallel passes:
// r = b - A x (k_residual), then black cells e_b = (r_b - sum a_br r_r / a_rr) / D~_b,
// then red cells e_r = (r_r - sum a_rb e_b) / a_rr.  Sums in ascending neighbour index
// (-z, -y, -x, +x, +y, +z), the order of the oracle's row-wise elimination and solves;
// the solves multiply by stored reciprocal pivots (one division per cell per solve
// instead of seven per step) and each colour pass runs one thread per cell of its colour.
__device__ __forceinline__ double diag_at(const StencilT& S, int c, int i, int j, int k) {
  const int nx = S.g.nx, sxy = S.g.nxy;
  const double txp = S.Tx[c], typ = S.Ty[c], tzp = S.Tz[c];
  const double txm = i > 0 ? S.Tx[c - 1] : 0.0;
  const double tym = j > 0 ? S.Ty[c - nx] : 0.0;
  const double tzm = k > 0 ? S.Tz[c - sxy] : 0.0;
  const double D = txp + txm + typ + tym + tzp + tzm;
  return c == 0 ? 2.0 * D : D;
}

// face transmissibilities of cell c in ascending neighbour order and the neighbours
__device__ __forceinline__ void faces_at(const StencilT& S, int c, int i, int j, int k,
                                         double t[6], int nb[6]) {
  const int nx = S.g.nx, ny = S.g.ny, nz = S.g.nz, sxy = S.g.nxy;
  t[0] = k > 0 ? S.Tz[c - sxy] : 0.0;      nb[0] = c - sxy;
  t[1] = j > 0 ? S.Ty[c - nx] : 0.0;       nb[1] = c - nx;
  t[2] = i > 0 ? S.Tx[c - 1] : 0.0;        nb[2] = c - 1;
  t[3] = i < nx - 1 ? S.Tx[c] : 0.0;       nb[3] = c + 1;
  t[4] = j < ny - 1 ? S.Ty[c] : 0.0;       nb[4] = c + nx;
  t[5] = k < nz - 1 ? S.Tz[c] : 0.0;       nb[5] = c + sxy;
}

// dinv[c] = 1 / pivot: 1 / a_rr on red cells, 1 / D~_b on black cells
__global__ void __launch_bounds__(CT) k_ilu_diag(StencilT S, double* __restrict__ dinv) {
  const int N = S.g.nxy * S.g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(S.g, c, i, j, k);
  double a = diag_at(S, c, i, j, k);
  if ((i + j + k) & 1) {  // black: subtract l_bk u_kb = (a_bk / a_kk) a_kb over red neighbours
    double t[6];
    int nb[6];
    faces_at(S, c, i, j, k, t, nb);
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (t[f] == 0.0) continue;
      int ii, jj, kk;
      g3_coords(S.g, nb[f], ii, jj, kk);
      const double l = -t[f] / diag_at(S, nb[f], ii, jj, kk);
      a = a - l * -t[f];
    }
  }
  dinv[c] = 1.0 / a;
}

// colour-compact thread map: thread t -> the q-th cell of colour `col` in grid row
// rho = t / hx (hx = ceil(nx / 2)), i = 2 q + ((j + k + col) & 1); false past the row end
__device__ __forceinline__ bool colour_cell(const Grid3& g, int t, int col, int& c, int& i,
                                            int& j, int& k) {
  const int hx = (g.nx + 1) >> 1;
  const int rho = t / hx, q = t - rho * hx;
  k = rho / g.ny;
  j = rho - k * g.ny;
  if (k >= g.nz) return false;
  i = 2 * q + ((j + k + col) & 1);
  if (i >= g.nx) return false;
  c = i + g.nx * j + g.nxy * k;
  return true;
}

// black cells: e_b = (r_b + sum_k T_bk r_k / a_kk) / D~_b, stored over r_b; x_b += e_b
__global__ void __launch_bounds__(CT) k_ilu_black(StencilT S, const double* __restrict__ dinv,
                                                  double* __restrict__ r, double* __restrict__ x,
                                                  const IterState* st) {
  if (is_done(st)) return;
  int c, i, j, k;
  if (!colour_cell(S.g, blockIdx.x * blockDim.x + threadIdx.x, 1, c, i, j, k)) return;
  double t[6];
  int nb[6];
  faces_at(S, c, i, j, k, t, nb);
  double y = r[c];
#pragma unroll
  for (int f = 0; f < 6; ++f)
    if (t[f] != 0.0) y += t[f] * (r[nb[f]] * dinv[nb[f]]);
  const double e = y * dinv[c];
  r[c] = e;
  x[c] += e;
}

// red cells: e_r = (r_r + sum_b T_rb e_b) / a_rr; x_r += e_r
__global__ void __launch_bounds__(CT) k_ilu_red(StencilT S, const double* __restrict__ dinv,
                                                const double* __restrict__ r,
                                                double* __restrict__ x, const IterState* st) {
  if (is_done(st)) return;
  int c, i, j, k;
  if (!colour_cell(S.g, blockIdx.x * blockDim.x + threadIdx.x, 0, c, i, j, k)) return;
  double t[6];
  int nb[6];
  faces_at(S, c, i, j, k, t, nb);
  double y = r[c];
#pragma unroll
  for (int f = 0; f < 6; ++f)
    if (t[f] != 0.0) y += t[f] * r[nb[f]];
  x[c] += y * dinv[c];
}

// Deterministic form for M <= RRD_MAX_M (the dynamic, well and indicator levels): no
// atomics anywhere.  Each warp reduces runs of equal columns with shuffles and its run
// tails add into the warp's own shared row one lane at a time (ascending lane), the CTA
// sums its eight rows in order into rc_part[cta][.], and k_rc_combine sums the CTAs in
// order.  The same inputs give the same r_c bits on every run, so the chaotic
// dynamic-stage iteration (its Δp bins) cannot drift with atomics order.
constexpr int RRD_MAX_M = 1536;
constexpr int RRD_WARPS = CT / 32;
__global__ void __launch_bounds__(CT) k_res_restrict_det(StencilT S, LevelView L, int M,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ rc_part, int first,
                                                         double* __restrict__ partials,
                                                         const IterState* st, const int* Md) {
  if (is_done(st)) return;
  if (Md) M = *Md;  // M from the device (graph-captured small dynamic path)
  extern __shared__ double acc[];  // [RRD_WARPS][M]
  for (int m = threadIdx.x; m < RRD_WARPS * M; m += blockDim.x) acc[m] = 0.0;
  __syncthreads();
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* row = acc + warp * M;
  const int N = S.g.nxy * S.g.nz;
  const int stride = gridDim.x * blockDim.x;
  double v2 = 0.0;
  for (int base = blockIdx.x * blockDim.x; base < N; base += stride) {  // warp-uniform
    const int c = base + threadIdx.x;
    const bool in = c < N;
    const int cc = in ? c : N - 1;
    int i, j, k;
    g3_coords(S.g, cc, i, j, k);
    double r = 0.0;
    if (in) {
      double dA;
      r = residual_at(S, x, b, c, i, j, k, &dA);
    }
    v2 += r * r;
    for (int s2 = 0; s2 < L.W; ++s2) {
      const int key = in ? L.col[(size_t)s2 * N + c] : -1;
      double v = key >= 0 ? (L.unit ? r : L.P[(size_t)s2 * N + c] * r) : 0.0;
      // inclusive segmented scan over runs of equal keys (fixed shuffle order)
      const int prev = __shfl_up_sync(full, key, 1);
      const unsigned heads = __ballot_sync(full, lane == 0 || prev != key);
      const int start = 31 - __clz(heads & ((2u << lane) - 1u));
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(full, v, o);
        if (lane - o >= start) v += y;
      }
      const int next = __shfl_down_sync(full, key, 1);
      unsigned tails = __ballot_sync(full, key >= 0 && (lane == 31 || next != key));
      while (tails) {  // one run tail at a time, ascending lane
        const int t = __ffs(tails) - 1;
        if (lane == t) row[key] += v;
        __syncwarp();
        tails &= tails - 1;
      }
    }
  }
  __syncthreads();
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double t = 0.0;
    for (int w = 0; w < RRD_WARPS; ++w) t += acc[w * M + m];
    rc_part[(size_t)blockIdx.x * M + m] = t;
  }
  if (first) warp_partial(v2, partials);
}

// one CTA per column: strided partial sums then a shuffle/shared tree, all fixed-order
__global__ void __launch_bounds__(256) k_rc_combine(const double* __restrict__ rc_part, int G,
                                                    int M, double* __restrict__ rc,
                                                    const IterState* st, const int* Md) {
  if (is_done(st)) return;
  if (Md) M = *Md;
  const int m = blockIdx.x;
  if (m >= M) return;
  double t = 0.0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) t += rc_part[(size_t)g * M + m];
  __shared__ double sh[8];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < 8; ++w) u += sh[w];
    rc[m] = u;
  }
}

// a8 for explicit levels with many columns (M > RRD_MAX_M: the fault-split level): one warp
// per column gathers its entries from the column-major index (positions ascending) —
// r_c[J] = sum_k P[pos_k] r[cell_k], lane-strided then a fixed shuffle tree: no atomics,
// so r_c is the same bits on every run (the atomic scatter it replaces spent ~100 us per
// config-3 iteration in contended fp64 atomics and made the dynamic stage's bins drift).
__global__ void __launch_bounds__(256) k_restrict_csc(const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ pos,
                                                      const double* __restrict__ P,
                                                      const double* __restrict__ r, int N, int M,
                                                      double* __restrict__ rc, const IterState* st) {
  if (is_done(st)) return;
  const int w = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= M) return;  // warp-uniform
  const int k1 = ptr[w + 1];
  // four independent chains per lane (positions k, k+32, k+64, k+96): the dependent
  // index -> value loads of one column overlap; partial sums combined in a fixed order
  double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
  int k = ptr[w] + lane;
  for (; k + 96 < k1; k += 128) {
    // the index and P are streamed (ld.cs, evict-first: see restrict_row_body), r is re-read
    const int p0 = __ldcs(pos + k), p1 = __ldcs(pos + k + 32), p2 = __ldcs(pos + k + 64),
              p3 = __ldcs(pos + k + 96);
    const double a0 = __ldcs(P + p0), a1 = __ldcs(P + p1), a2 = __ldcs(P + p2), a3 = __ldcs(P + p3);
    const double b0 = r[p0 - (p0 / N) * N], b1 = r[p1 - (p1 / N) * N], b2 = r[p2 - (p2 / N) * N],
                 b3 = r[p3 - (p3 / N) * N];
    t0 = fma(a0, b0, t0);
    t1 = fma(a1, b1, t1);
    t2 = fma(a2, b2, t2);
    t3 = fma(a3, b3, t3);
  }
  for (; k < k1; k += 32) {
    const int p = __ldcs(pos + k);
    t0 = fma(__ldcs(P + p), r[p - (p / N) * N], t0);
  }
  double t = (t0 + t1) + (t2 + t3);
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) rc[w] = t;
}

// Column-major index build: keys (column << 32 | position) of the valid entries, radix
// sorted (CUB), column counts scanned into csc_ptr.
__global__ void k_csc_keys(const int32_t* __restrict__ col, int64_t n, int32_t* __restrict__ cnt,
                           unsigned long long* __restrict__ keys, int* __restrict__ fill) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int J = col[e];
  if (J < 0) return;
  atomicAdd(cnt + J, 1);
  keys[atomicAdd(fill, 1)] = ((unsigned long long)J << 32) | (unsigned)e;
}

__global__ void k_csc_pos(const unsigned long long* __restrict__ keys, int64_t n,
                          int32_t* __restrict__ pos) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) pos[e] = (int32_t)(unsigned)(keys[e] & 0xffffffffull);
}

// a9: x += P xc (row gather).// a9: x += P xc (row gather).
__global__ void __launch_bounds__(CT) k_prolong(LevelView L, double* __restrict__ x,
                                                const double* __restrict__ xc,
                                                const IterState* st) {
  if (is_done(st)) return;
  const int N = L.g.nxy * L.g.nz;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double acc = 0.0;
  if (L.kind == 0) {
    int i, j, k;
    g3_coords(L.g, c, i, j, k);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      int key = lv_col(L, c, i, j, k, s);
      if (key >= 0) acc += L.P[(size_t)s * N + c] * xc[key];
    }
  } else {
    // four slots at a time: their column and value loads, then the x_c gathers, are
    // independent and overlap; the sum is still taken in slot order
    int s = 0;
    for (; s + 4 <= L.W; s += 4) {
      int key[4];
      double p[4], v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        key[u] = __ldcs(L.col + (size_t)(s + u) * N + c);  // streamed, like the Cartesian P
        p[u] = __ldcs(L.P + (size_t)(s + u) * N + c);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = key[u] >= 0 ? p[u] * xc[key[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (key[u] >= 0) acc += v[u];
    }
    for (; s < L.W; ++s) {
      int key = L.col[(size_t)s * N + c];
      if (key >= 0) acc += L.unit ? xc[key] : L.P[(size_t)s * N + c] * xc[key];
    }
  }
  x[c] += acc;
}

// a6: r = b - A x (materialised for the gather restriction); `first` also emits the
// ||r||^2 partials of the stop test (post-smoothing order starts a cycle here).
template <int CPT>
__global__ void __launch_bounds__(CT) k_residual(StencilT S, const double* __restrict__ x,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ r, int first,
                                                 double* __restrict__ partials,
                                                 const IterState* st) {
  stencil_prologue<CPT>(S, b);
  const bool done = is_done(st);
  const int N = S.g.nxy * S.g.nz;
  const int c0 = blockIdx.x * (CT * CPT) + threadIdx.x;
  double rv[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = min(c0 + u * CT, N - 1);
    int i, j, k;
    g3_coords(S.g, c, i, j, k);
    double dA;
    rv[u] = residual_at(S, x, b, c, i, j, k, &dA);
  }
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = c0 + u * CT;
    if (c < N) {
      if (!done) r[c] = rv[u];
      v += rv[u] * rv[u];
    }
  }
  if (first) warp_partial(v, partials);
}

// Open-box support range of block J along one axis (reading A3): cells x with
// C(J-1) < 2x+1 < C(J+1), C(J) = lo_J + hi_J, limits dropped at the boundary.
__device__ __forceinline__ void support_range(int J, int b, int n, int nb, int& x0, int& x1) {
  x0 = 0;
  x1 = n;
  if (J > 0) {
    int lo = (J - 1) * b;
    x0 = (lo + min(lo + b, n) + 1) >> 1;
  }
  if (J < nb - 1) {
    int lo = (J + 1) * b;
    x1 = (lo + min(lo + b, n)) >> 1;
  }
}

// a8 (Cartesian level): r_c[J] = Σ_{c ∈ S_J} P_cJ r_c, one CTA per coarse column,
// gathering its support box row by row (column J lives in the parity slot of J in
// every cell of S_J).  Every P entry is read exactly once; r (N doubles) stays in L2.
// Fixed-order reduction: deterministic, no atomics.
// a8 (Cartesian level): r_c = P^T r.  One CTA per coarse (Jy, Jz) row of blocks
// computes the restriction of all Jx of that row: it walks the (y, z) rows of the
// (Jy, Jz) support box over the FULL x extent, reading both x-parity slot planes of
// P and r with fully coalesced row loads (each P entry once; r shared by the two
// parities), keeps per-thread partial sums per x position and parity, and finally sums
// each column's x range from shared memory in a fixed order (deterministic, no
// atomics).  Thread layout: XL lanes along x (XL = pow2 >= nx, <= 256) x RG row
// groups; x positions beyond 256 take a second partial.
constexpr int RR2_THREADS = 256;
// P is read once per pass and, with A_c^{-1}, is most of an iteration's bytes; T, b, x and r
// (63 MB on config 2) are re-read by the next stencil passes.  The P loads here and in the
// prolongation therefore use ld.global.cs (evict-first), like the SYMV's tile loads, so the
// streams do not displace those vectors from L2: 67.4 -> 63.4 us per config-2 iteration
// (profiles/r02i/p_stream_hint_ab.txt; a createpolicy evict_first hint measured the same,
// evict_last on T/b/x and reversed traversal orders measured no gain or slower).
// XP x positions per lane (x = xo + XL * e, e < XP): XP = ceil(nx / XL), 1 for nx <= 256.
// CS CTAs (one thread-block cluster) share one (Jy, Jz) unit: rank q walks the rows
// q, q + CS, ... of each row group; the CTAs' per-(parity, x) totals are summed by rank 0
// over distributed shared memory in rank order (deterministic).
template <int XP, int CS>
__device__ __forceinline__ void restrict_row_body(const LevelView& L, const double* __restrict__ r,
                                                  double* __restrict__ rc, int unit,
                                                  double* rsh, bool done) {
  const int N = L.g.nxy * L.g.nz;
  const int nx = L.g.nx, sxy = L.g.nxy;
  const int Jy = unit % L.nb1, Jz = unit / L.nb1;
  int y0, y1, z0, z1;
  support_range(Jy, L.b1, L.g.ny, L.nb1, y0, y1);
  support_range(Jz, L.b2, L.g.nz, L.nb2, z0, z1);
  const int wy = y1 - y0, rows = wy * (z1 - z0);
  const int sy = ((Jy & 1) << 1) | ((Jz & 1) << 2);
  const double* __restrict__ P0 = L.P + (size_t)sy * N;        // x parity 0
  const double* __restrict__ P1 = L.P + (size_t)(sy | 1) * N;  // x parity 1
  const int XL = XP > 1 ? 256 : (nx <= 32 ? 32 : (nx <= 64 ? 64 : (nx <= 128 ? 128 : 256)));
  const int RG = RR2_THREADS / XL;
  const int xo = threadIdx.x % XL, rg = threadIdx.x / XL;
  int rank = 0;
  if constexpr (CS > 1) rank = (int)cooperative_groups::this_cluster().block_rank();
  double a0[XP], a1[XP];  // parity 0 / 1 partials at x = xo + XL e
  bool xok[XP];
#pragma unroll
  for (int e = 0; e < XP; ++e) {
    a0[e] = a1[e] = 0.0;
    xok[e] = xo + XL * e < nx;
  }
  const int step = RG * CS;
  constexpr int U = XP > 2 ? 2 : 4;  // rows in flight per lane
  // the first rows this CTA loads (U per row group, both x-parity planes of P, which no pass
  // of the cycle writes) are bulk-prefetched into L2 while the residual pass drains; r
  // after the wait.  Only the first batch: beyond L2 (config 5) a whole-range prefetch
  // would be evicted before use.
  for (int t = threadIdx.x; t < min(rows, U * step); t += blockDim.x) {
    if ((t % step) / RG != rank) continue;
    const int tz = t / wy, ty = t - tz * wy;
    const size_t c = (size_t)nx * (y0 + ty) + (size_t)sxy * (z0 + tz);
    prefetch_l2(P0 + c, (size_t)nx * sizeof(double));
    prefetch_l2(P1 + c, (size_t)nx * sizeof(double));
  }
  pdl_wait();
  pdl_trigger();
  int row = rg + RG * rank;
  int zz = row / wy, yy = row - zz * wy;
  const int dz = step / wy, dy = step - dz * wy;
  while (row < rows) {
    double p0[U][XP], p1[U][XP], rv[U][XP];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = row < rows;
      const size_t c = (size_t)nx * (y0 + yy) + (size_t)sxy * (z0 + zz) + xo;
#pragma unroll
      for (int e = 0; e < XP; ++e) {
        const bool v = ok && xok[e];
        p0[u][e] = v ? __ldcs(P0 + c + XL * e) : 0.0;  // streamed: see restrict_row_body's header
        p1[u][e] = v ? __ldcs(P1 + c + XL * e) : 0.0;
        rv[u][e] = v ? r[c + XL * e] : 0.0;
      }
      row += step;
      yy += dy;
      zz += dz;
      if (yy >= wy) {
        yy -= wy;
        ++zz;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < XP; ++e) {
        a0[e] += p0[u][e] * rv[u][e];
        a1[e] += p1[u][e] * rv[u][e];
      }
  }
  // per-(row group, parity, x) partials -> shared, summed over row groups in order
  const int XLX = XP * XL;  // rsh: [RG][2][XLX] then totals [2][XLX]
#pragma unroll
  for (int e = 0; e < XP; ++e) {
    rsh[(rg * 2 + 0) * XLX + XL * e + xo] = a0[e];
    rsh[(rg * 2 + 1) * XLX + XL * e + xo] = a1[e];
  }
  __syncthreads();
  double* tot = rsh + RG * 2 * XLX;
  for (int t = threadIdx.x; t < 2 * XLX; t += blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < RG; ++g) v += rsh[g * 2 * XLX + t];
    tot[t] = v;
  }
  if constexpr (CS > 1) {
    auto cl = cooperative_groups::this_cluster();
    cl.sync();  // every rank's totals are complete
    if (rank == 0) {
      for (int t = threadIdx.x; t < 2 * XLX; t += blockDim.x) {
        double v = tot[t];
#pragma unroll
        for (int q = 1; q < CS; ++q) v += cl.map_shared_rank(tot, q)[t];
        rsh[t] = v;  // the row-group partials are dead: reuse their space
      }
    }
    cl.sync();  // remote reads done before any rank exits
    if (rank != 0) return;
    tot = rsh;
  } else {
    __syncthreads();
  }
  __syncthreads();
  for (int Jx = threadIdx.x; Jx < L.nb0; Jx += blockDim.x) {
    int x0, x1;
    support_range(Jx, L.b0, nx, L.nb0, x0, x1);
    const double* tp = tot + (Jx & 1) * XLX;
    double v = 0.0;
    for (int x = x0; x < x1; ++x) v += tp[x];
    if (!done) rc[Jx + L.nb0 * (Jy + L.nb1 * Jz)] = v;
  }
}

template <int XP, int CS>
__global__ void __launch_bounds__(RR2_THREADS) k_restrict_cart(LevelView L,
                                                               const double* __restrict__ r,
                                                               double* __restrict__ rc,
                                                               const IterState* st) {
  extern __shared__ double rsh[];
  restrict_row_body<XP, CS>(L, r, rc, blockIdx.x / CS, rsh, is_done(st));
}

// CTAs (one cluster) per (Jy, Jz) unit: 680 instead of 340 CTAs on config 2's 148 SMs
// (measured 70.6 against 72.0 us per iteration; 4 per unit gave no further gain)
constexpr int RCS = 2;

static inline int restrict_xp(int nx) {
  return nx <= 256 ? 1 : (nx <= 512 ? 2 : (nx <= 1024 ? 4 : 8));
}

static inline size_t restrict_rows_smem(int nx) {
  const int XP = restrict_xp(nx);
  const int XL = XP > 1 ? 256 : (nx <= 32 ? 32 : (nx <= 64 ? 64 : (nx <= 128 ? 128 : 256)));
  const int RG = RR2_THREADS / XL;
  return (size_t)(RG + 1) * 2 * XP * XL * sizeof(double);
}

// k_restrict_cart<XP, CS> over `units` (Jy, Jz) rows, CS CTAs per unit in one cluster
template <int XP, int CS>
static msb_status launch_restrict(msb_ctx ctx, cudaStream_t st, unsigned units, size_t smem,
                                  const LevelView& V, const double* r, double* rc,
                                  const IterState* ist) {
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_restrict_cart<XP, CS>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  MSB_CUDA_TRY(ctx, launch_ex(k_restrict_cart<XP, CS>, dim3(units * CS), dim3(RR2_THREADS), smem, st,
                              kPDL, CS, V, r, rc, ist));
  return MSB_OK;  // the caller's MSB_LAUNCH_CHECK counts the launch

}

// a9 (Cartesian level): x += P x_c, one thread per cell: the six per-axis block
// indices come from the parity table, the eight (P, x_c) loads are predicated selects
// with no branches, so all sixteen are in flight together.  (Four cells per thread, as
// the stencil passes use, measured 27 us against 17 us here: the dependent x_c gathers
// need the occupancy more than the extra loads in flight.)
// bounded to 40 registers (6 CTAs per SM): the dependent x_c gathers need the occupancy
// (config 5 523 -> 501 us per iteration, config 2 61.9 -> 61.0; 7 and 8 CTAs per SM spill and
// measured 561 / 73.6 us; profiles/r02i/prolong_occupancy_ab.txt)
__global__ void __launch_bounds__(CT, 6) k_prolong_cart(LevelView L, double* __restrict__ x,
                                                     const double* __restrict__ xc,
                                                     const IterState* st) {
  const bool done = is_done(st);
  const int N = L.g.nxy * L.g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(L.g, c, i, j, k);
  const int2 tx = reinterpret_cast<const int2*>(L.tab)[i];
  const int2 ty = reinterpret_cast<const int2*>(L.tab)[L.g.nx + j];
  const int2 tz = reinterpret_cast<const int2*>(L.tab)[L.g.nx + L.g.ny + k];
  const double* __restrict__ base = L.P + c;
  double v[8], xv[8];
  int col[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int jx = (s & 1) ? tx.y : tx.x, jy = (s & 2) ? ty.y : ty.x, jz = (s & 4) ? tz.y : tz.x;
    const bool act = (jx | jy | jz) >= 0;
    col[s] = act ? jx + L.nb0 * (jy + L.nb1 * jz) : -1;
    v[s] = act ? __ldcs(base + (size_t)s * N) : 0.0;  // streamed (evict-first), as in the restriction
  }
  pdl_wait();  // P is an input; x_c and x come from the coarse solve and the smoother
  pdl_trigger();
#pragma unroll
  for (int s = 0; s < 8; ++s) xv[s] = col[s] >= 0 ? xc[col[s]] : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < 8; ++s) acc += v[s] * xv[s];
  const double xn = x[c] + acc;
  if (!done) x[c] = xn;
}

__global__ void k_zero_if(double* __restrict__ p, int n, const IterState* st) {
  if (is_done(st)) return;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) p[t] = 0.0;
}

// ---------------------------------------------------------------- dynamic partition kernels
__global__ void k_dp(const double* __restrict__ x, const double* __restrict__ xp, int64_t N,
                     double* __restrict__ dp) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < N) dp[c] = x[c] - xp[c];
}

// max|dp| (bit pattern of a non-negative double orders like the value): grid-stride,
// block reduction, one atomic per CTA (one per warp contended on the single word: 27 us)
__global__ void __launch_bounds__(256) k_absmax_vec(const double* __restrict__ dp, int64_t N,
                                                    unsigned long long* mx) {
  double a = 0.0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N;
       c += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs(dp[c]));
  for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = fmax(a, wm[w]);
    atomicMax(mx, (unsigned long long)__double_as_longlong(a));
  }
}

__global__ void k_bins(const double* __restrict__ dp, int64_t N, const unsigned long long* mx,
                       double e0, double e1, int32_t* __restrict__ bins) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double m = __longlong_as_double((long long)*mx);
  double a = fabs(dp[c]);
  bins[c] = (a >= e0 * m) + (a >= e1 * m);
}

// component sizes: runs of equal labels in consecutive lanes are counted with one atomic
// (a large component would otherwise send every cell's increment to one address)
// Component sizes.  Run lengths of equal labels within a warp, then a 16-slot shared table
// per CTA (a CTA's 256 consecutive cells carry few labels), one global atomic per distinct
// label per CTA: the large components' counters were hit by every warp (25 us).  Integer
// sums, so the result does not depend on the order.
__global__ void __launch_bounds__(256) k_sizes(const int32_t* __restrict__ lab, int64_t N,
                                               int32_t* __restrict__ cnt) {
  __shared__ int tkey[16], tval[16];
  if (threadIdx.x < 16) {
    tkey[threadIdx.x] = -1;
    tval[threadIdx.x] = 0;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = c < N ? lab[c] : -1;
  const int prev = __shfl_up_sync(full, key, 1);
  const unsigned heads = __ballot_sync(full, lane == 0 || prev != key);
  const int next = __shfl_down_sync(full, key, 1);
  if (key >= 0 && (lane == 31 || next != key)) {  // run tail: run length = lane - head + 1
    const int head = 31 - __clz(heads & ((2u << lane) - 1u));
    const int len = lane - head + 1;
    bool put = false;
    for (int p = 0; p < 16 && !put; ++p) {
      const int sl = (int)(((unsigned)key * 2654435761u >> 28) + p) & 15;
      const int old = atomicCAS(tkey + sl, -1, key);
      if (old == -1 || old == key) {
        atomicAdd(tval + sl, len);
        put = true;
      }
    }
    if (!put) atomicAdd(cnt + key, len);
  }
  __syncthreads();
  if (threadIdx.x < 16 && tkey[threadIdx.x] >= 0) atomicAdd(cnt + tkey[threadIdx.x], tval[threadIdx.x]);
}

// counts[0] = #roots with size >= smin; counts[1..3] = bin b has a small component
__global__ void k_merge_count(const int32_t* __restrict__ lab, const int32_t* __restrict__ cnt,
                              const int32_t* __restrict__ bins, int64_t N, int smin,
                              int32_t* __restrict__ counts) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  if (lab[c] != (int32_t)c) return;
  if (cnt[c] >= smin) atomicAdd(counts, 1);
  else atomicExch(counts + 1 + bins[c], 1);
}

// smin_dev (if set) overrides smin: the threshold chosen on the device (k_pick_smin)
__global__ void k_merge_rep(const int32_t* __restrict__ lab, const int32_t* __restrict__ cnt,
                            const int32_t* __restrict__ bins, int64_t N, int smin,
                            int32_t* __restrict__ rep, const int32_t* smin_dev = nullptr) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  if (smin_dev) smin = *smin_dev;
  if (cnt[lab[c]] < smin) atomicMin(rep + bins[c], (int32_t)c);
}

__global__ void k_merge_label(int32_t* __restrict__ lab, const int32_t* __restrict__ cnt,
                              const int32_t* __restrict__ bins, int64_t N, int smin,
                              const int32_t* __restrict__ rep, int32_t* __restrict__ out,
                              const int32_t* smin_dev = nullptr) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  if (smin_dev) smin = *smin_dev;
  int32_t r = lab[c];
  out[c] = cnt[r] < smin ? rep[bins[c]] : r;
}

// The A15 merge threshold without a host round trip: one pass histograms the component
// sizes by floor(log2) — over all roots and per bin — and k_pick_smin replays the host
// rule on the histograms: s_min = 1, 2, 4, ... until (#roots with size >= s_min) + (#bins
// with a component smaller than s_min) <= max_blocks or s_min > N.  For s_min = 2^s,
// "size >= s_min" is exactly "floor(log2 size) >= s".  hist[0..31] all roots, hist[32 +
// 32 b + k] bin b; hist[128] = s_min; hist[129..131] = the per-bin representatives.
__global__ void k_size_hist(const int32_t* __restrict__ lab, const int32_t* __restrict__ cnt,
                            const int32_t* __restrict__ bins, int64_t N, int32_t* __restrict__ hist) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N || lab[c] != (int32_t)c) return;
  const int k = 31 - __clz(max(cnt[c], 1));
  atomicAdd(hist + k, 1);
  atomicAdd(hist + 32 + 32 * bins[c] + k, 1);
}

__global__ void k_pick_smin(int32_t* __restrict__ hist, int max_blocks, int64_t N) {
  if (threadIdx.x != 0) return;
  int64_t smin = 1;
  for (int s = 0;; ++s, smin *= 2) {
    long long nb = 0;
    for (int k = s; k < 32; ++k) nb += hist[k];
    for (int b = 0; b < 3; ++b) {
      int small = 0;
      for (int k = 0; k < s && k < 32; ++k) small += hist[32 + 32 * b + k];
      nb += small > 0;
    }
    if (nb <= max_blocks || smin > N || s >= 31) break;
  }
  hist[128] = (int32_t)smin;
  hist[129] = hist[130] = hist[131] = INT32_MAX;
}

// NEXT-3 indicator partition: bin = #{e : edges[e] <= |ind|} (absolute edges)
struct BinEdges {
  int n;
  double v[8];
};
__global__ void k_bins_abs(const double* __restrict__ ind, int64_t N, BinEdges E,
                           int32_t* __restrict__ bins) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const double a = fabs(ind[c]);
  int b = 0;
  for (int e = 0; e < E.n; ++e) b += a >= E.v[e];
  bins[c] = b;
}

// The dynamic loop's small-path gate (after the rebuild's numbering): gate[4] = M_dyn when
// the stage runs on the graph-captured small path (max|Δp| > 0 and 0 < M_dyn <= SMALL_CHOL_M),
// else 0; gate[0] (read as IterState::done by the stage kernels) = 1 when they must not store.
__global__ void k_dyn_gate(const int32_t* __restrict__ Mtot, const unsigned long long* __restrict__ mx,
                           const IterState* st, int* __restrict__ gate) {
  const int M = *Mtot;
  const double m = __longlong_as_double((long long)*mx);
  const int Meff = (m > 0.0 && M > 0 && M <= SMALL_CHOL_M) ? M : 0;
  gate[4] = Meff;
  gate[0] = (Meff == 0 || st->done) ? 1 : 0;
}

__global__ void k_refill_const(const int32_t* __restrict__ part, int64_t N, int32_t* __restrict__ col,
                               double* __restrict__ P) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  col[c] = part[c];
  P[c] = 1.0;
}

}  // namespace msb

using namespace msb;

static StencilT stencil(msb_op op) {
  return StencilT{op->Tx, op->Ty, op->Tz, make_grid3(op->nx, op->ny, op->nz)};
}

static LevelView view(msb_level L) {
  return LevelView{L->kind, L->W, L->nb[0], L->nb[1], L->nb[2], L->bs[0], L->bs[1], L->bs[2],
                   make_grid3(L->nx, L->ny, L->nz), L->tab, L->col, L->P[L->cur],
                   (L->kind == 1 && L->W == 1 && L->unity) ? 1 : 0};
}
// Build the dynamic constant-basis stage from dp (device, length N) into s->dyn_level.
// The N-sized part of the dynamic rebuild (no host synchronisation; graph-capturable):
// max|Δp|, bins (A14), connected components, sizes, the merge threshold and merged labels
// (A15), canonical numbering; M_dyn and max|Δp| are copied to the pinned s->dyn_pin.
static msb_status dyn_labels(msb_ctx ctx, msb_solver s, const double* dp) {
  msb_op op = s->op;
  int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(s->scratch_i);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(mx, 0, 8, st));
  k_absmax_vec<<<(unsigned)std::min<int64_t>(grid_for(N, 256), 2 * ctx->sm_count), 256, 0, st>>>(dp, N, mx);
  MSB_LAUNCH_CHECK(ctx);
  k_bins<<<grid_for(N, 256), 256, 0, st>>>(dp, N, mx, s->edge0, s->edge1, s->bins);
  MSB_LAUNCH_CHECK(ctx);
  msb_status rc = cc_label(ctx, op, s->bins, s->lab, nullptr);
  if (rc) return rc;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(s->cnt, 0, N * sizeof(int32_t), st));
  k_sizes<<<grid_for(N, 256), 256, 0, st>>>(s->lab, N, s->cnt);
  MSB_LAUNCH_CHECK(ctx);
  // merge threshold on the device (k_size_hist + k_pick_smin): no readback here
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(s->mhist, 0, 132 * sizeof(int32_t), st));
  k_size_hist<<<grid_for(N, 256), 256, 0, st>>>(s->lab, s->cnt, s->bins, N, s->mhist);
  MSB_LAUNCH_CHECK(ctx);
  k_pick_smin<<<1, 32, 0, st>>>(s->mhist, s->dyn_max, N);
  MSB_LAUNCH_CHECK(ctx);
  k_merge_rep<<<grid_for(N, 256), 256, 0, st>>>(s->lab, s->cnt, s->bins, N, 1, s->mhist + 129,
                                                s->mhist + 128);
  MSB_LAUNCH_CHECK(ctx);
  k_merge_label<<<grid_for(N, 256), 256, 0, st>>>(s->lab, s->cnt, s->bins, N, 1, s->mhist + 129,
                                                  s->ids, s->mhist + 128);
  MSB_LAUNCH_CHECK(ctx);
  // canonical numbering: labels are minimum cells of their blocks
  const int32_t* Md = nullptr;
  rc = canonical_number_async(ctx, N, s->ids, s->lab, s->cnt /* 2N scratch: cnt|bins reused */, &Md);
  if (rc) return rc;
  char* pin = static_cast<char*>(s->dyn_pin);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(pin, Md, 4, cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(pin + 8, mx, 8, cudaMemcpyDeviceToHost, st));
  return MSB_OK;
}

// M_dyn and max|Δp| from the pinned buffer (after dyn_labels has completed)
static void dyn_read(msb_solver s, int32_t* M, double* mxv) {
  const char* pin = static_cast<const char*>(s->dyn_pin);
  memcpy(M, pin, 4);
  memcpy(mxv, pin + 8, 8);
}

// The M-sized part: the constant basis of the labels, A_c (exact) and its factorisation.
static msb_status dyn_finish(msb_ctx ctx, msb_solver s, int32_t M, int32_t* part_out) {
  msb_op op = s->op;
  int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  msb_level D = s->dyn_level;
  k_refill_const<<<grid_for(N, 256), 256, 0, st>>>(s->lab, N, D->col, D->P[0]);
  MSB_LAUNCH_CHECK(ctx);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(D->part, s->lab, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  D->cur = 0;
  D->M = M;
  if (part_out) MSB_CUDA_TRY(ctx, copy_out(ctx, part_out, D->part, N * sizeof(int32_t)));
  return coarse_assemble_dense(ctx, D, op);
}

static msb_status ensure_dyn_pin(msb_ctx ctx, msb_solver s) {
  if (!s->dyn_pin) MSB_CUDA_TRY(ctx, cudaHostAlloc(&s->dyn_pin, 64, cudaHostAllocDefault));
  return scan_reserve(ctx, s->op->N);
}

static msb_status build_dynamic(msb_ctx ctx, msb_solver s, const double* dp, int32_t* M_out,
                                int32_t* part_out) {
  msb_status rc = ensure_dyn_pin(ctx, s);
  if (rc) return rc;
  if ((rc = dyn_labels(ctx, s, dp))) return rc;
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  int32_t M = 0;
  double m = 0.0;
  dyn_read(s, &M, &m);
  if (!(m > 0.0)) {  // max|Δp| = 0: stage skipped
    *M_out = 0;
    return MSB_OK;
  }
  if ((rc = dyn_finish(ctx, s, M, part_out))) return rc;
  *M_out = M;
  return MSB_OK;
}

namespace msb {
// Column-major index of an explicit level's pattern for the gather restriction
// (k_restrict_csc); built once per level, before any graph capture.
static msb_status level_csc_build(msb_ctx ctx, msb_level L) {
  if (L->csc_ptr) return MSB_OK;
  const int64_t n = (int64_t)L->W * L->N;
  if (n >= INT32_MAX) return set_error(ctx, MSB_EDIM, "explicit pattern too large for int32 positions");
  cudaStream_t st = ctx->stream;
  const int M = L->M;
  int32_t* cnt = nullptr;
  unsigned long long *keys = nullptr, *sorted = nullptr;
  int* fill = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  msb_status rc = MSB_OK;
  int32_t total = 0;
  int end_bit = 32;
  while ((1ll << (end_bit - 32)) < (long long)M + 1) ++end_bit;
  MSB_ALLOC(ctx, L->csc_ptr, int32_t, M + 1);
  cnt = dalloc_n<int32_t>(ctx, M + 1);
  keys = dalloc_n<unsigned long long>(ctx, (size_t)L->nnz + 1);
  sorted = dalloc_n<unsigned long long>(ctx, (size_t)L->nnz + 1);
  fill = dalloc_n<int>(ctx, 1);
  L->csc_pos = dalloc_n<int32_t>(ctx, (size_t)L->nnz + 1);
  if (!cnt || !keys || !sorted || !fill || !L->csc_pos) {
    rc = set_error(ctx, MSB_ENOMEM, "restriction index");
    goto out;
  }
  if (cudaMemsetAsync(cnt, 0, (M + 1) * sizeof(int32_t), st) != cudaSuccess ||
      cudaMemsetAsync(fill, 0, sizeof(int), st) != cudaSuccess) {
    rc = set_error(ctx, MSB_ECUDA, "restriction index memset");
    goto out;
  }
  k_csc_keys<<<grid_for(n, 256), 256, 0, st>>>(L->col, n, cnt, keys, fill);
  count_launch();
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, sorted, (int)L->nnz, 0, end_bit, st);
  tmp = dalloc(ctx, tmp_bytes + 16);
  if (!tmp) {
    rc = set_error(ctx, MSB_ENOMEM, "restriction index sort");
    goto out;
  }
  if (cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, (int)L->nnz, 0, end_bit, st) !=
      cudaSuccess) {
    rc = set_error(ctx, MSB_ECUDA, "restriction index sort");
    goto out;
  }
  count_launch();
  k_csc_pos<<<grid_for(L->nnz, 256), 256, 0, st>>>(sorted, L->nnz, L->csc_pos);
  count_launch();
  rc = scan_exclusive(ctx, cnt, L->csc_ptr, M + 1, &total);
  if (!rc && total != L->nnz)
    rc = set_error(ctx, MSB_EINVAL, "restriction index: %d entries, level has %lld", total,
                   (long long)L->nnz);
out:
  if (cudaGetLastError() != cudaSuccess && !rc) rc = set_error(ctx, MSB_ECUDA, "restriction index build");
  cudaStreamSynchronize(st);
  dfree(ctx, cnt);
  dfree(ctx, keys);
  dfree(ctx, sorted);
  dfree(ctx, fill);
  dfree(ctx, tmp);
  if (rc) {
    dfree(ctx, L->csc_ptr);
    dfree(ctx, L->csc_pos);
    L->csc_ptr = L->csc_pos = nullptr;
  }
  return rc;
}

static bool use_csc(msb_solver s, msb_level L) {
  return L->kind == 1 && L->M > RRD_MAX_M && L != s->dyn_level && L->csc_ptr;
}
}  // namespace msb

extern "C" {

msb_status msb_solver_create(msb_ctx ctx, msb_op op, const msb_level* levels, int32_t n_levels,
                             double omega_s, int32_t nu, int32_t post_smooth, int32_t dyn_enable,
                             double dyn_edge0, double dyn_edge1, int32_t dyn_max_blocks,
                             msb_solver* out) {
  MSB_NVTX("msb_solver_create");
  if (!ctx || !op || !out || n_levels < 0 || (n_levels > 0 && !levels) || nu < 0)
    return set_error(ctx, MSB_EINVAL, "msb_solver_create args");
  if (n_levels == 0 && !dyn_enable) return set_error(ctx, MSB_EINVAL, "solver needs a level");
  {  // A must be nonsingular: every cell connected to the gauge cell (reading A7)
    bool conn = false;
    msb_status rc = op_connected(ctx, op, &conn);
    if (rc) return rc;
    if (!conn)
      return set_error(ctx, MSB_EINCONSISTENT,
                       "the faces with T > 0 split the grid into several compartments: A is "
                       "singular on every compartment without the gauge cell 0");
  }
  msb_solver s = new msb_solver_s();
  s->ctx = ctx;
  s->op = op;
  s->omega_s = omega_s;
  s->nu = nu;
  s->post = post_smooth ? 1 : 0;
  s->dyn = dyn_enable ? 1 : 0;
  s->edge0 = dyn_edge0;
  s->edge1 = dyn_edge1;
  s->dyn_max = dyn_max_blocks > 0 ? dyn_max_blocks : 1024;
  int maxM = 1;
  for (int l = 0; l < n_levels; ++l) {
    msb_level L = levels[l];
    if (!L || L->N != op->N) return set_error(ctx, MSB_EDIM, "level %d size mismatch", l);
    if (!L->co.ready) return set_error(ctx, MSB_EINVAL, "level %d not assembled", l);
    if (L->kind == 1 && L->M > RRD_MAX_M) {
      msb_status rc = level_csc_build(ctx, L);
      if (rc) return rc;
    }
    s->levels.push_back(L);
    maxM = std::max(maxM, L->M);
  }
  int64_t N = op->N;
  if (s->dyn) maxM = std::max(maxM, s->dyn_max + 3);
  s->maxM = maxM;
  MSB_ALLOC(ctx, s->xbuf[0], double, N);
  MSB_ALLOC(ctx, s->xbuf[1], double, N);
  MSB_ALLOC(ctx, s->rc, double, maxM + 2);
  MSB_ALLOC(ctx, s->xc, double, maxM + 2);
  MSB_ALLOC(ctx, s->partials, double, (size_t)grid_for(N, CT) * (CT / 32) + 32);
  MSB_ALLOC(ctx, s->r, double, N);
  s->st = dalloc_n<IterState>(ctx, 1);
  if (!s->st) return set_error(ctx, MSB_ENOMEM, "solver state");
  if (s->dyn) {
    MSB_ALLOC(ctx, s->xprev, double, N);
    MSB_ALLOC(ctx, s->dpbuf, double, N);
    MSB_ALLOC(ctx, s->lab, int32_t, N);
    MSB_ALLOC(ctx, s->ids, int32_t, N);
    MSB_ALLOC(ctx, s->cnt, int32_t, 2 * N);
    s->bins = s->cnt + N;  // bins live in the second half of the cnt scratch
    MSB_ALLOC(ctx, s->scratch_i, int32_t, 64);
    MSB_ALLOC(ctx, s->mhist, int32_t, 132);
    // constant-basis level reused across iterations
    msb_level D = new msb_level_s();
    D->ctx = ctx;
    D->kind = 1;
    D->N = N;
    D->W = 1;
    D->nnz = N;
    D->nx = op->nx; D->ny = op->ny; D->nz = op->nz;
    MSB_ALLOC(ctx, D->P[0], double, N);
    MSB_ALLOC(ctx, D->P[1], double, N);
    MSB_ALLOC(ctx, D->col, int32_t, N);
    MSB_ALLOC(ctx, D->part, int32_t, N);
    int cap = s->dyn_max + 3;
    MSB_ALLOC(ctx, D->co.Ac, double, (int64_t)cap * cap);
    MSB_ALLOC(ctx, D->co.L, double, (int64_t)cap * cap);
    MSB_ALLOC(ctx, D->co.Ainv, double, (int64_t)cap * cap);
    MSB_ALLOC(ctx, D->co.tri_y, double, cap);
    D->co.cap = cap;
    D->co.tri = true;  // factorised for exactly one solve per rebuild
    // the graph-captured small path needs fixed buffers: the exact-assembly accumulator and
    // the factor flags at full capacity, the restriction partials for M <= RRD_MAX_M, the gate
    MSB_ALLOC(ctx, D->co.acc, unsigned long long, 2 * (int64_t)cap * cap + 2);
    D->co.acc_cap = (size_t)cap * cap;
    MSB_ALLOC(ctx, D->co.flags, unsigned long long, 2);
    {
      const int64_t gpart = std::min<int64_t>(grid_for(N, CT), 4 * ctx->sm_count);
      const size_t need = (size_t)gpart * RRD_MAX_M;
      MSB_ALLOC(ctx, s->rc_part, double, need);
      s->rc_part_cap = need;
    }
    MSB_ALLOC(ctx, s->dyn_gate, int, 8);
    s->dyn_level = D;
  }
  // bins must not alias cnt during counting: give them their own buffer
  if (s->dyn) {
    int32_t* b;
    MSB_ALLOC(ctx, b, int32_t, N);
    s->bins = b;
  }
  *out = s;
  return MSB_OK;
}

msb_status msb_add_dynamic_basis(msb_ctx ctx, msb_solver s, const double* dp, int32_t* M_dyn_out,
                                 int32_t* part_out) {
  MSB_NVTX("msb_add_dynamic_basis");
  if (!ctx || !s || !dp) return set_error(ctx, MSB_EINVAL, "msb_add_dynamic_basis: null");
  if (!s->dyn) return set_error(ctx, MSB_EINVAL, "solver created without dynamic stage");
  void* o = nullptr;
  const double* d = (const double*)stage_in(ctx, dp, s->op->N * sizeof(double), &o);
  int32_t M = 0;
  msb_status st = build_dynamic(ctx, s, d, &M, part_out);
  if (o) {
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx, o);
  }
  if (st) return st;
  if (M == 0) s->dyn_level->M = 0;
  if (M_dyn_out) *M_dyn_out = M;
  return sync(ctx);
}

// Enqueue one stage (level L) on x buffers; `first` marks the iteration's first kernel.
// Enqueue one stage (level L) on the x double buffer; `first` marks the iteration's
// first kernel, which also emits the stop-test partials (finalised right after).
#define RES_LAUNCH(...)                                                                          \
  do {                                                                                           \
    if (rcpt == CPT_BIG)                                                                         \
      MSB_CUDA_TRY(ctx, launch_ex(k_residual<CPT_BIG>, dim3(gr), dim3(CT), 0, st, kPDL, 1, __VA_ARGS__)); \
    else if (rcpt == CPT_WAVE)                                                                   \
      MSB_CUDA_TRY(ctx, launch_ex(k_residual<CPT_WAVE>, dim3(gr), dim3(CT), 0, st, kPDL, 1, __VA_ARGS__)); \
    else                                                                                         \
      MSB_CUDA_TRY(ctx, launch_ex(k_residual<CPT>, dim3(gr), dim3(CT), 0, st, kPDL, 1, __VA_ARGS__));     \
  } while (0)
#define JAC_LAUNCH(...)                                                                          \
  do {                                                                                           \
    if (big)                                                                                     \
      MSB_CUDA_TRY(ctx, launch_ex(k_jacobi<CPT_BIG>, dim3(g4), dim3(CT), 0, st, kPDL, 1, __VA_ARGS__));   \
    else                                                                                         \
      MSB_CUDA_TRY(ctx, launch_ex(k_jacobi<CPT>, dim3(g4), dim3(CT), 0, st, kPDL, 1, __VA_ARGS__));       \
  } while (0)

static msb_status enqueue_stage(msb_ctx ctx, msb_solver s, msb_level L, const double* b, int& cur,
                                bool& first) {
  msb_op op = s->op;
  int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  StencilT S = stencil(op);
  LevelView V = view(L);
  unsigned g = grid_for(N, CT);
  const bool big = N >= CPT_BIG_MIN_N;
  const unsigned g4 = grid_for(N, CT * (big ? CPT_BIG : CPT));  // blocks of the smoother pass
  // With one pre-smoothed level and nu = 1 no kernel of an iteration writes the buffer
  // holding x_{k-1}, so the stop test's finalize runs on a side branch in parallel with
  // the rest of the iteration and is joined before the next iteration's first kernel
  // (kernels that have not yet seen `done` then do harmless work).
  const bool side = s->levels.size() == 1 && s->nu == 1 && !s->post && L->kind == 0 &&
                    s->smoother == 0;
  // the residual pass (48 registers at CPT_WAVE cells per thread: 5 CTAs per SM) takes CPT_WAVE
  // cells per thread when that makes its grid exactly one resident wave and CPT does not
  // (config 2: 731 CTAs on 740 slots instead of 1,096 on 888: 64.3 -> 61.9 us per iteration;
  // 5, 7, 8 cells and the same for the smoother measured slower, profiles/r02i/per_kernel_cpt_occ_ab.txt);
  // only in the single-level iteration: with the dynamic rebuild running beside the static
  // stages (config 3) 4 cells stay faster (0.710 against 0.719 ms per iteration)
  const int64_t slots = 5 * (int64_t)ctx->sm_count;
  const int rcpt = big ? CPT_BIG
                       : (side && (int64_t)grid_for(N, CT * CPT) > slots &&
                                  (int64_t)grid_for(N, CT * CPT_WAVE) <= slots
                              ? CPT_WAVE
                              : CPT);
  const unsigned gr = grid_for(N, CT * rcpt);  // blocks of the residual pass

  auto fin = [&](unsigned np) -> msb_status {  // np = blocks of the kernel that wrote partials
    if (side) {
      if (!s->side_stream) {
        MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->side_stream, cudaStreamNonBlocking));
        MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
        MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
      }
      MSB_CUDA_TRY(ctx, cudaEventRecord(s->ev_fork, st));
      MSB_CUDA_TRY(ctx, cudaStreamWaitEvent(s->side_stream, s->ev_fork, 0));
      k_finalize<<<1, 1024, 0, s->side_stream>>>(s->partials, (int)np, 0, s->st, s->res_dev);
      MSB_LAUNCH_CHECK(ctx);
      MSB_CUDA_TRY(ctx, cudaEventRecord(s->ev_join, s->side_stream));
      s->pending_join = true;
      return MSB_OK;
    }
    k_finalize<<<1, 1024, 0, st>>>(s->partials, (int)np, 0, s->st, s->res_dev);
    MSB_LAUNCH_CHECK(ctx);
    return MSB_OK;
  };
  if (first && s->pending_join) {
    MSB_CUDA_TRY(ctx, cudaStreamWaitEvent(st, s->ev_join, 0));
    s->pending_join = false;
  }
  auto ilu = [&]() -> msb_status {  // ν red-black ILU(0) steps on x in place (NEXT-2)
    for (int v = 0; v < s->nu; ++v) {
      RES_LAUNCH(S, s->xbuf[cur], b, s->r, first ? 1 : 0, s->partials, s->st);
      MSB_LAUNCH_CHECK(ctx);
      if (first) {
        msb_status rc = fin(gr);
        if (rc) return rc;
      }
      first = false;
      const unsigned gc = grid_for((int64_t)((op->nx + 1) / 2) * op->ny * op->nz, CT);
      k_ilu_black<<<gc, CT, 0, st>>>(S, s->ilu_d, s->r, s->xbuf[cur], s->st);
      MSB_LAUNCH_CHECK(ctx);
      k_ilu_red<<<gc, CT, 0, st>>>(S, s->ilu_d, s->r, s->xbuf[cur], s->st);
      MSB_LAUNCH_CHECK(ctx);
    }
    return MSB_OK;
  };
  auto jac = [&]() -> msb_status {
    if (s->smoother == 1) return ilu();
    for (int v = 0; v < s->nu; ++v) {
      JAC_LAUNCH(S, s->xbuf[cur], s->xbuf[cur ^ 1], b, s->omega_s, first ? 1 : 0,
                                 s->partials, s->st);
      MSB_LAUNCH_CHECK(ctx);
      if (first) {
        msb_status rc = fin(g4);
        if (rc) return rc;
      }
      first = false;
      cur ^= 1;
    }
    return MSB_OK;
  };
  auto corr = [&]() -> msb_status {
    if (L->kind == 0) {
      RES_LAUNCH(S, s->xbuf[cur], b, s->r, first ? 1 : 0, s->partials, s->st);
      MSB_LAUNCH_CHECK(ctx);
      if (first) {
        msb_status rc = fin(gr);
        if (rc) return rc;
      }
      first = false;
      if (op->nx > 2048)
        return set_error(ctx, MSB_EINVAL, "Cartesian restriction supports nx <= 2048 (nx=%d)", op->nx);
      {
        const int xp = restrict_xp(op->nx);
        const size_t smem = restrict_rows_smem(op->nx);
        const unsigned gr = (unsigned)(L->nb[1] * L->nb[2]);
        msb_status rc = MSB_OK;
#define MSB_RESTRICT_CS(XPV) \
  rc = launch_restrict<XPV, RCS>(ctx, st, gr, smem, V, s->r, s->rc, s->st)
        if (xp == 1) MSB_RESTRICT_CS(1);
        else if (xp == 2) MSB_RESTRICT_CS(2);
        else if (xp == 4) MSB_RESTRICT_CS(4);
        else MSB_RESTRICT_CS(8);
#undef MSB_RESTRICT_CS
        if (rc) return rc;
      }
      MSB_LAUNCH_CHECK(ctx);
      coarse_solve(ctx, L->co, s->rc, s->xc, &s->st->done);
      MSB_CUDA_TRY(ctx, launch_ex(k_prolong_cart, dim3(g), dim3(CT), 0, st, kPDL, 1, V, s->xbuf[cur],
                                  s->xc, s->st));
      MSB_LAUNCH_CHECK(ctx);
      return MSB_OK;
    }
    if (use_csc(s, L)) {
      RES_LAUNCH(S, s->xbuf[cur], b, s->r, first ? 1 : 0, s->partials, s->st);
      MSB_LAUNCH_CHECK(ctx);
      if (first) {
        msb_status rc = fin(gr);
        if (rc) return rc;
      }
      first = false;
      k_restrict_csc<<<(unsigned)((L->M + 7) / 8), 256, 0, st>>>(L->csc_ptr, L->csc_pos, L->P[L->cur],
                                                              s->r, (int)L->N, L->M, s->rc, s->st);
      MSB_LAUNCH_CHECK(ctx);
      coarse_solve(ctx, L->co, s->rc, s->xc, &s->st->done);
      k_prolong<<<g, CT, 0, st>>>(V, s->xbuf[cur], s->xc, s->st);
      MSB_LAUNCH_CHECK(ctx);
      return MSB_OK;
    }
    k_zero_if<<<grid_for(L->M, 256), 256, 0, st>>>(s->rc, L->M, s->st);
    MSB_LAUNCH_CHECK(ctx);
    unsigned gpart = g;  // blocks that write stop-test partials
    if (L->kind == 1 && L->M <= RRD_MAX_M) {
      gpart = (unsigned)std::min<int64_t>(g, 4 * ctx->sm_count);
      const size_t need = (size_t)gpart * L->M;
      if (s->rc_part_cap < need) {
        dfree(ctx, s->rc_part);
        s->rc_part = dalloc_n<double>(ctx, need);
        if (!s->rc_part) return set_error(ctx, MSB_ENOMEM, "restriction partials");
        s->rc_part_cap = need;
      }
      const size_t smem = (size_t)RRD_WARPS * L->M * sizeof(double);
      static bool attr = false;
      if (!attr) {
        MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_res_restrict_det,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(RRD_WARPS * RRD_MAX_M * sizeof(double))));
        attr = true;
      }
      k_res_restrict_det<<<gpart, CT, smem, st>>>(S, V, L->M, s->xbuf[cur], b, s->rc_part,
                                                  first ? 1 : 0, s->partials, s->st, nullptr);
      MSB_LAUNCH_CHECK(ctx);
      k_rc_combine<<<L->M, 256, 0, st>>>(s->rc_part, (int)gpart, L->M, s->rc, s->st, nullptr);
    } else {
      k_res_restrict<<<g, CT, 0, st>>>(S, V, s->xbuf[cur], b, s->rc, first ? 1 : 0, s->partials,
                                       s->st);
    }
    MSB_LAUNCH_CHECK(ctx);
    if (first) {
      msb_status rc = fin(gpart);
      if (rc) return rc;
    }
    first = false;
    coarse_solve(ctx, L->co, s->rc, s->xc, &s->st->done);
    k_prolong<<<g, CT, 0, st>>>(V, s->xbuf[cur], s->xc, s->st);
    MSB_LAUNCH_CHECK(ctx);
    return MSB_OK;
  };
  msb_status rc;
  if (s->post) {
    if ((rc = corr())) return rc;
    if ((rc = jac())) return rc;
  } else {
    if ((rc = jac())) return rc;
    if ((rc = corr())) return rc;
  }
  return MSB_OK;
}

static msb_status join_side(msb_ctx ctx, msb_solver s) {
  if (s->pending_join) {
    MSB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, s->ev_join, 0));
    s->pending_join = false;
  }
  return MSB_OK;
}

static msb_status enqueue_norm(msb_ctx ctx, msb_solver s, const double* x, const double* b,
                               int mode) {
  msb_op op = s->op;
  unsigned g = grid_for(op->N, CT);
  k_norm<<<g, CT, 0, ctx->stream>>>(stencil(op), x, b, mode, s->partials, s->st);
  MSB_LAUNCH_CHECK(ctx);
  k_finalize<<<1, 1024, 0, ctx->stream>>>(s->partials, (int)g, mode, s->st,
                                          s->res_dev);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

static void drop_graphs(msb_solver s) {
  for (int t = 0; t < 2; ++t) {
    if (s->gexec[t]) cudaGraphExecDestroy(s->gexec[t]);
    s->gexec[t] = nullptr;
    s->glaunches[t] = 0;
    if (s->sgexec[t]) cudaGraphExecDestroy(s->sgexec[t]);
    s->sgexec[t] = nullptr;
    if (s->dgexec[t]) cudaGraphExecDestroy(s->dgexec[t]);
    s->dgexec[t] = nullptr;
  }
  s->sgkey.clear();
  s->dgkey.clear();
}

// Capture `n` iterations of the static stages starting from x buffer `cur0` into a
// CUDA graph (on a private capture stream: the context stream may be the legacy
// default stream, which cannot be captured), instantiate once, reuse per chunk.
static msb_status chunk_graph(msb_ctx ctx, msb_solver s, const double* db, int cur0, int n,
                              cudaGraphExec_t* out) {
  *out = nullptr;
  std::vector<const void*> key = {db, s->res_dev, (const void*)(intptr_t)n};
  for (msb_level L : s->levels) {
    key.push_back(L->P[L->cur]);
    key.push_back(L->co.Ainv);
    key.push_back(L->co.sch);
    key.push_back(L->co.Xp);
  }
  if (key != s->gkey) {
    drop_graphs(s);
    s->gkey = key;
  }
  if (s->gexec[cur0]) {
    *out = s->gexec[cur0];
    return MSB_OK;
  }
  if (!s->cap_stream) {
    MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
  }
  cudaStream_t user = ctx->stream;
  ctx->stream = s->cap_stream;
  int64_t l0 = g_launches.load();
  msb_status rc = MSB_OK;
  cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    int cur = cur0;
    for (int t = 0; t < n && !rc; ++t) {
      bool first = true;
      for (msb_level L : s->levels)
        if ((rc = enqueue_stage(ctx, s, L, db, cur, first))) break;
    }
    if (!rc) rc = join_side(ctx, s);  // the side branch rejoins before the capture ends
    s->pending_join = false;
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(s->cap_stream, &graph);
    if (!rc && e2 == cudaSuccess) {
      e = cudaGraphInstantiate(&s->gexec[cur0], graph, 0);
    } else if (e2 != cudaSuccess) {
      e = e2;
    }
    if (graph) cudaGraphDestroy(graph);
  }
  ctx->stream = user;
  s->glaunches[cur0] = g_launches.load() - l0;
  g_launches.fetch_sub(s->glaunches[cur0]);  // captured, not launched
  if (rc) return rc;
  if (e != cudaSuccess) {
    cudaGetLastError();
    s->gexec[cur0] = nullptr;
    return set_error(ctx, MSB_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  }
  *out = s->gexec[cur0];
  return MSB_OK;
}

// Dynamic loop: one iteration of the static stages (norm already taken: no stop-test
// partials) from x buffer cur0, captured once and replayed; *cur_out = the buffer it ends in.
static msb_status static_graph(msb_ctx ctx, msb_solver s, const double* db, int cur0,
                               cudaGraphExec_t* out, int* cur_out) {
  *out = nullptr;
  std::vector<const void*> key = {db};
  for (msb_level L : s->levels) {
    key.push_back(L->P[L->cur]);
    key.push_back(L->co.Ainv);
    key.push_back(L->co.sch);
    key.push_back(L->co.Xp);
  }
  if (key != s->sgkey) {
    for (int t = 0; t < 2; ++t) {
      if (s->sgexec[t]) cudaGraphExecDestroy(s->sgexec[t]);
      s->sgexec[t] = nullptr;
    }
    s->sgkey = key;
  }
  if (!s->sgexec[cur0]) {
    if (!s->cap_stream)
      MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    ctx->stream = s->cap_stream;
    const int64_t l0 = g_launches.load();
    msb_status rc = MSB_OK;
    int cur = cur0;
    cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      bool first = false;
      for (msb_level L : s->levels)
        if ((rc = enqueue_stage(ctx, s, L, db, cur, first))) break;
      cudaGraph_t graph = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(s->cap_stream, &graph);
      if (!rc && e2 == cudaSuccess) e = cudaGraphInstantiate(&s->sgexec[cur0], graph, 0);
      else if (e2 != cudaSuccess) e = e2;
      if (graph) cudaGraphDestroy(graph);
    }
    ctx->stream = user;
    s->sglaunches[cur0] = g_launches.load() - l0;
    g_launches.fetch_sub(s->sglaunches[cur0]);  // captured, not launched
    s->scur_after[cur0] = cur;
    if (rc) return rc;
    if (e != cudaSuccess) {
      cudaGetLastError();
      s->sgexec[cur0] = nullptr;
      return set_error(ctx, MSB_ECUDA, "static-stage graph: %s", cudaGetErrorString(e));
    }
  }
  *out = s->sgexec[cur0];
  *cur_out = s->scur_after[cur0];
  return MSB_OK;
}

// Dynamic loop: the N-sized rebuild (dyn_labels on s->dpbuf) as one graph.
static msb_status labels_graph(msb_ctx ctx, msb_solver s, cudaGraphExec_t* out) {
  *out = nullptr;
  if (s->lgexec && s->lg_scan != (const void*)ctx->scan_scr) {  // the scan scratch moved
    cudaGraphExecDestroy(s->lgexec);
    s->lgexec = nullptr;
  }
  if (!s->lgexec) {
    msb_status rc = ensure_dyn_pin(ctx, s);
    if (rc) return rc;
    if (!s->cap_stream)
      MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    ctx->stream = s->cap_stream;
    const int64_t l0 = g_launches.load();
    cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      rc = dyn_labels(ctx, s, s->dpbuf);
      cudaGraph_t graph = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(s->cap_stream, &graph);
      if (!rc && e2 == cudaSuccess) e = cudaGraphInstantiate(&s->lgexec, graph, 0);
      else if (e2 != cudaSuccess) e = e2;
      if (graph) cudaGraphDestroy(graph);
    }
    ctx->stream = user;
    s->lglaunches = g_launches.load() - l0;
    g_launches.fetch_sub(s->lglaunches);
    s->lg_scan = ctx->scan_scr;
    if (rc) return rc;
    if (e != cudaSuccess) {
      cudaGetLastError();
      s->lgexec = nullptr;
      return set_error(ctx, MSB_ECUDA, "rebuild graph: %s", cudaGetErrorString(e));
    }
  }
  *out = s->lgexec;
  return MSB_OK;
}

// ---------------------------------------------------------------- graph-captured dynamic iteration
// For M_dyn <= SMALL_CHOL_M (most rebuilds) the whole iteration runs as one CUDA graph with
// M_dyn read on the device: Δp, then the static stages on the context stream in parallel with
// the rebuild on the rebuild stream (labels, the gate, the constant basis, exact A_c and the
// one-CTA factorisation), then the dynamic stage — no host enqueue after the M_dyn readback.
// When the gate is 0 (M_dyn > SMALL_CHOL_M, or max|Δp| = 0) the gated kernels return and the
// host runs the general path after the graph.  Launch shapes are those of M = SMALL_CHOL_M.
static int* dyn_gate_ptr(msb_solver s) { return reinterpret_cast<int*>(s->dyn_gate); }

static msb_status dyn_small_finish(msb_ctx ctx, msb_solver s) {
  msb_op op = s->op;
  const int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  msb_level D = s->dyn_level;
  const int* Md = dyn_gate_ptr(s) + 4;
  k_refill_const<<<grid_for(N, 256), 256, 0, st>>>(s->lab, N, D->col, D->P[0]);
  MSB_LAUNCH_CHECK(ctx);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(D->part, s->lab, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  msb_status rc = coarse_assemble_const_gated(ctx, D, op, Md, SMALL_CHOL_M);
  if (rc) return rc;
  return coarse_factor_small_gated(ctx, D->co, Md);
}

static msb_status dyn_small_stage(msb_ctx ctx, msb_solver s, const double* b, int& cur) {
  msb_op op = s->op;
  msb_level D = s->dyn_level;
  cudaStream_t st = ctx->stream;
  const int* gate = dyn_gate_ptr(s);
  const int* Md = gate + 4;
  const IterState* gst = reinterpret_cast<const IterState*>(gate);  // done = gate[0]
  StencilT S = stencil(op);
  LevelView V = view(D);
  const int64_t N = op->N;
  const unsigned g = grid_for(N, CT), g4 = grid_for(N, CT * CPT);
  const unsigned gpart = (unsigned)std::min<int64_t>(g, 4 * ctx->sm_count);
  auto jac = [&]() -> msb_status {
    for (int v = 0; v < s->nu; ++v) {
      k_jacobi<CPT><<<g4, CT, 0, st>>>(S, s->xbuf[cur], s->xbuf[cur ^ 1], b, s->omega_s, 0,
                                       s->partials, gst);
      MSB_LAUNCH_CHECK(ctx);
      cur ^= 1;
    }
    return MSB_OK;
  };
  auto corr = [&]() -> msb_status {
    k_zero_if<<<1, 256, 0, st>>>(s->rc, SMALL_CHOL_M, gst);
    MSB_LAUNCH_CHECK(ctx);
    static bool attr = false;
    if (!attr) {
      MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_res_restrict_det,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(RRD_WARPS * RRD_MAX_M * sizeof(double))));
      attr = true;
    }
    k_res_restrict_det<<<gpart, CT, (size_t)RRD_WARPS * SMALL_CHOL_M * sizeof(double), st>>>(
        S, V, 0, s->xbuf[cur], b, s->rc_part, 0, s->partials, gst, Md);
    MSB_LAUNCH_CHECK(ctx);
    k_rc_combine<<<SMALL_CHOL_M, 256, 0, st>>>(s->rc_part, (int)gpart, 0, s->rc, gst, Md);
    MSB_LAUNCH_CHECK(ctx);
    coarse_solve_small_gated(ctx, D->co, s->rc, s->xc, gate, Md);
    k_prolong<<<g, CT, 0, st>>>(V, s->xbuf[cur], s->xc, gst);
    MSB_LAUNCH_CHECK(ctx);
    return MSB_OK;
  };
  msb_status rc;
  if (s->post) {
    if ((rc = corr())) return rc;
    return jac();
  }
  if ((rc = jac())) return rc;
  return corr();
}

// the whole rebuild iteration from x buffer cur0 as one graph (see above); *cur_static = the
// buffer after the static stages, *cur_small = after the small dynamic stage
static msb_status dyn_graph(msb_ctx ctx, msb_solver s, const double* db, int cur0,
                            cudaGraphExec_t* out, int* cur_static, int* cur_small) {
  *out = nullptr;
  std::vector<const void*> key = {db, ctx->scan_scr, s->rc_part};
  for (msb_level L : s->levels) {
    key.push_back(L->P[L->cur]);
    key.push_back(L->co.Ainv);
    key.push_back(L->co.sch);
    key.push_back(L->co.Xp);
  }
  if (key != s->dgkey) {
    for (int t = 0; t < 2; ++t) {
      if (s->dgexec[t]) cudaGraphExecDestroy(s->dgexec[t]);
      s->dgexec[t] = nullptr;
    }
    s->dgkey = key;
  }
  if (!s->dgexec[cur0]) {
    msb_status rc = ensure_dyn_pin(ctx, s);
    if (rc) return rc;
    const unsigned long long* tm = nullptr;
    if ((rc = op_tmax(ctx, s->op, &tm))) return rc;  // cached before capture
    if (!s->cap_stream)
      MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    if (!s->cap_stream2)
      MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->cap_stream2, cudaStreamNonBlocking));
    if (!s->ev_cf) {
      MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_cf, cudaEventDisableTiming));
      MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_cj, cudaEventDisableTiming));
    }
    cudaStream_t user = ctx->stream;
    const int64_t l0 = g_launches.load();
    const int64_t N = s->op->N;
    int cur = cur0, cs = cur0;
    cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      do {
        ctx->stream = s->cap_stream;
        k_dp<<<grid_for(N, 256), 256, 0, s->cap_stream>>>(s->xbuf[cur], s->xprev, N, s->dpbuf);
        count_launch();
        if ((e = cudaEventRecord(s->ev_cf, s->cap_stream)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(s->xprev, s->xbuf[cur], N * sizeof(double), cudaMemcpyDeviceToDevice,
                                 s->cap_stream)) != cudaSuccess) break;
        // rebuild branch
        if ((e = cudaStreamWaitEvent(s->cap_stream2, s->ev_cf, 0)) != cudaSuccess) break;
        ctx->stream = s->cap_stream2;
        if ((rc = dyn_labels(ctx, s, s->dpbuf))) break;
        k_dyn_gate<<<1, 1, 0, s->cap_stream2>>>(ctx->scan_scr, reinterpret_cast<unsigned long long*>(s->scratch_i),
                                                s->st, dyn_gate_ptr(s));
        count_launch();
        if ((e = cudaEventRecordWithFlags(s->ev_lab, s->cap_stream2, cudaEventRecordExternal)) != cudaSuccess)
          break;
        if ((rc = dyn_small_finish(ctx, s))) break;
        if ((e = cudaEventRecord(s->ev_cj, s->cap_stream2)) != cudaSuccess) break;
        // static stages, then the (gated) dynamic stage
        ctx->stream = s->cap_stream;
        bool first = false;
        for (msb_level L : s->levels)
          if ((rc = enqueue_stage(ctx, s, L, db, cur, first))) break;
        if (rc) break;
        cs = cur;
        if ((e = cudaStreamWaitEvent(s->cap_stream, s->ev_cj, 0)) != cudaSuccess) break;
        if ((rc = dyn_small_stage(ctx, s, db, cur))) break;
      } while (false);
      cudaGraph_t graph = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(s->cap_stream, &graph);
      if (!rc && e == cudaSuccess && e2 == cudaSuccess) e = cudaGraphInstantiate(&s->dgexec[cur0], graph, 0);
      else if (e == cudaSuccess && e2 != cudaSuccess) e = e2;
      if (graph) cudaGraphDestroy(graph);
    }
    ctx->stream = user;
    s->dglaunches[cur0] = g_launches.load() - l0;
    g_launches.fetch_sub(s->dglaunches[cur0]);
    s->dcur_static[cur0] = cs;
    s->dcur_small[cur0] = cur;
    if (rc) return rc;
    if (e != cudaSuccess) {
      cudaGetLastError();
      s->dgexec[cur0] = nullptr;
      return set_error(ctx, MSB_ECUDA, "dynamic-iteration graph: %s", cudaGetErrorString(e));
    }
  }
  *out = s->dgexec[cur0];
  *cur_static = s->dcur_static[cur0];
  *cur_small = s->dcur_small[cur0];
  return MSB_OK;
}

msb_status msb_solver_set_smoother(msb_ctx ctx, msb_solver s, int32_t kind) {
  if (!ctx || !s || kind < 0 || kind > 1) return set_error(ctx, MSB_EINVAL, "msb_solver_set_smoother");
  if (kind != s->smoother) drop_graphs(s);
  s->smoother = kind;
  return MSB_OK;
}

msb_status msb_partition_indicator(msb_ctx ctx, msb_op op, const double* ind, const double* edges,
                                   int32_t n_edges, int32_t max_blocks, int32_t* part,
                                   int32_t* M_out) {
  if (!ctx || !op || !ind || !M_out || n_edges < 0 || n_edges > 8 || (n_edges && !edges) ||
      max_blocks < 1)
    return set_error(ctx, MSB_EINVAL, "msb_partition_indicator: args");
  BinEdges E{};
  E.n = n_edges;
  for (int e = 0; e < n_edges; ++e) {
    E.v[e] = edges[e];
    if (e > 0 && !(edges[e] > edges[e - 1]))
      return set_error(ctx, MSB_EINVAL, "msb_partition_indicator: edges not strictly increasing");
  }
  const int64_t N = op->N;
  const int nbin = n_edges + 1;
  cudaStream_t st = ctx->stream;
  void* o = nullptr;
  const double* d = (const double*)stage_in(ctx, ind, N * sizeof(double), &o);
  if (!d) return set_error(ctx, MSB_ENOMEM, "indicator staging");
  int32_t *bins, *lab, *ids, *cnt, *scr;
  MSB_ALLOC(ctx, bins, int32_t, N);
  MSB_ALLOC(ctx, lab, int32_t, N);
  MSB_ALLOC(ctx, ids, int32_t, N);
  MSB_ALLOC(ctx, cnt, int32_t, 2 * N);
  MSB_ALLOC(ctx, scr, int32_t, 2 * nbin + 2);
  int32_t* counts = scr;         // [0] roots >= s_min, [1 + b] bin b has a small component
  int32_t* rep = scr + nbin + 1;  // per bin: minimum cell of its small components
  k_bins_abs<<<grid_for(N, 256), 256, 0, st>>>(d, N, E, bins);
  MSB_LAUNCH_CHECK(ctx);
  msb_status rc = cc_label(ctx, op, bins, lab, nullptr);
  if (rc) return rc;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, N * sizeof(int32_t), st));
  k_sizes<<<grid_for(N, 256), 256, 0, st>>>(lab, N, cnt);
  MSB_LAUNCH_CHECK(ctx);
  int smin = 1;
  std::vector<int32_t> hc(nbin + 1);
  while (true) {  // s_min doubles until at most max_blocks blocks remain (A15)
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(counts, 0, (nbin + 1) * sizeof(int32_t), st));
    k_merge_count<<<grid_for(N, 256), 256, 0, st>>>(lab, cnt, bins, N, smin, counts);
    MSB_LAUNCH_CHECK(ctx);
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hc.data(), counts, hc.size() * sizeof(int32_t),
                                      cudaMemcpyDeviceToHost, st));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    int64_t nb = 0;
    for (int32_t v : hc) nb += v;
    if (nb <= max_blocks || (int64_t)smin > N) break;
    smin *= 2;
  }
  std::vector<int32_t> big(nbin, INT32_MAX);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(rep, big.data(), nbin * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_merge_rep<<<grid_for(N, 256), 256, 0, st>>>(lab, cnt, bins, N, smin, rep);
  MSB_LAUNCH_CHECK(ctx);
  k_merge_label<<<grid_for(N, 256), 256, 0, st>>>(lab, cnt, bins, N, smin, rep, ids);
  MSB_LAUNCH_CHECK(ctx);
  int32_t M = 0;
  if ((rc = canonical_number(ctx, N, ids, lab, cnt, &M))) return rc;
  if (part) MSB_CUDA_TRY(ctx, copy_out(ctx, part, lab, N * sizeof(int32_t)));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  dfree(ctx, bins);
  dfree(ctx, lab);
  dfree(ctx, ids);
  dfree(ctx, cnt);
  dfree(ctx, scr);
  if (o) dfree(ctx, o);
  *M_out = M;
  return MSB_OK;
}

msb_status msb_ms_iterate(msb_ctx ctx, msb_solver s, const double* b, double* x, double tol,
                          int32_t max_iter, int32_t fixed_iters, int32_t* iters_out,
                          double* res_hist, int32_t* dyn_M_hist) {
  MSB_NVTX("msb_ms_iterate");
  if (!ctx || !s || !x) return set_error(ctx, MSB_EINVAL, "msb_ms_iterate: null");
  if (max_iter < 0 || fixed_iters < 0) return set_error(ctx, MSB_EINVAL, "negative iteration count");
  msb_op op = s->op;
  int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  int cap = std::max(max_iter, fixed_iters) + 2;
  if (s->res_cap < cap) {
    dfree(ctx, s->res_dev);
    MSB_ALLOC(ctx, s->res_dev, double, cap);
    s->res_cap = cap;
  }
  void* ob = nullptr;
  const double* db = b ? (const double*)stage_in(ctx, b, N * sizeof(double), &ob) : op->q;
  if (!db) return set_error(ctx, MSB_ENOMEM, "rhs staging");
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(s->xbuf[0], x, N * sizeof(double), cudaMemcpyDefault, st));
  IterState h{};
  h.max_iter = max_iter;
  h.fixed = fixed_iters;
  h.tol = tol;
  h.bscale = 1.0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(s->st, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  msb_status rc = solver_smoother_setup(ctx, s);  // pivots from the operator's current T
  if (rc) return rc;
  rc = enqueue_norm(ctx, s, s->xbuf[0], db, 1);
  if (rc) return rc;
  int cur = 0;
  int target = fixed_iters > 0 ? fixed_iters : max_iter;
  std::vector<int> cur_after;  // buffer holding x_k
  cur_after.push_back(0);
  std::vector<int32_t> dynM;
  IterState hs{};
  if (!s->dyn) {
    const int chunk = 16;
    // x-buffer swaps per iteration (Jacobi writes out of place; ILU(0) updates in place)
    const int flips = s->smoother == 0 ? s->nu * (int)s->levels.size() : 0;
    int issued = 0;
    while (true) {
      int n = std::min(chunk, target - issued);
      cudaGraphExec_t ge = nullptr;
      if (n == chunk) {
        rc = chunk_graph(ctx, s, db, cur, chunk, &ge);
        if (rc) return rc;
      }
      if (ge) {
        MSB_CUDA_TRY(ctx, cudaGraphLaunch(ge, st));
        g_launches.fetch_add(s->glaunches[cur], std::memory_order_relaxed);
        for (int t = 0; t < n; ++t) {
          cur ^= flips & 1;
          cur_after.push_back(cur);
        }
      } else {
        for (int t = 0; t < n; ++t) {
          bool first = true;
          for (msb_level L : s->levels)
            if ((rc = enqueue_stage(ctx, s, L, db, cur, first))) return rc;
          cur_after.push_back(cur);
        }
      }
      issued += n;
      if ((rc = join_side(ctx, s))) return rc;
      if (issued >= target)
        if ((rc = enqueue_norm(ctx, s, s->xbuf[cur], db, 0))) return rc;
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, s->st, sizeof(hs), cudaMemcpyDeviceToHost, st));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
      if (hs.done || issued >= target) break;
    }
  } else {
    // dynamic stage: host-synchronous per iteration (M_dyn is data dependent)
    // the rebuilt level's singular-pivot flag is read with the stop-test state (one
    // synchronisation per iteration for both); a singular rebuild fails the call there
    msb_level D = s->dyn_level;
    int hsing = 0;
    // a singular flag left by an earlier call (a failed rebuild) must not fail this one
    // before it has rebuilt anything: only this call's rebuilds may set it
    if (D->co.flags) MSB_CUDA_TRY(ctx, cudaMemsetAsync(D->co.flags + 1, 0, sizeof(int), st));
    if (!s->dyn_stream) {
      MSB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s->dyn_stream, cudaStreamNonBlocking));
      MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_dp, cudaEventDisableTiming));
      MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_dyn, cudaEventDisableTiming));
      MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&s->ev_lab, cudaEventDisableTiming));
    }
    while (true) {
      if ((rc = enqueue_norm(ctx, s, s->xbuf[cur], db, 0))) return rc;
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, s->st, sizeof(hs), cudaMemcpyDeviceToHost, st));
      if (D->co.flags)
        MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hsing, D->co.flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
      if (hsing) {
        D->co.ready = false;
        return set_error(ctx, MSB_ESINGULAR, "dynamic stage: singular coarse matrix (M=%d)", D->M);
      }
      if (hs.done) break;
      int k = hs.k;  // iteration about to run (1-based)
      int32_t M = 0;
      const bool rebuild = k >= 2;
      if (rebuild && s->smoother == 0) {  // one graph; the general path only for large M_dyn
        cudaGraphExec_t dg = nullptr;
        int cs = cur, csm = cur;
        if ((rc = dyn_graph(ctx, s, db, cur, &dg, &cs, &csm))) return rc;
        MSB_CUDA_TRY(ctx, cudaGraphLaunch(dg, st));
        g_launches.fetch_add(s->dglaunches[cur], std::memory_order_relaxed);
        MSB_CUDA_TRY(ctx, cudaEventSynchronize(s->ev_lab));  // M_dyn, max|Δp| in dyn_pin
        double mxv = 0.0;
        dyn_read(s, &M, &mxv);
        if (!(mxv > 0.0)) M = 0;
        if (M > 0 && M <= SMALL_CHOL_M) {  // the graph ran the stage
          cur = csm;
          D->cur = 0;
          D->M = M;
          D->co.M = M;
          D->co.kind = 0;
          D->co.small = true;
          D->co.ready = true;
        } else {
          cur = cs;
          if (M > 0) {  // general path after the graph, on the context stream
            D->co.defer_check = true;
            rc = dyn_finish(ctx, s, M, nullptr);
            D->co.defer_check = false;
            if (rc) return rc;
            bool first = false;
            if ((rc = enqueue_stage(ctx, s, D, db, cur, first))) return rc;
          }
        }
        dynM.push_back(M);
        cur_after.push_back(cur);
        continue;
      }
      if (rebuild) {
        k_dp<<<grid_for(N, 256), 256, 0, st>>>(s->xbuf[cur], s->xprev, N, s->dpbuf);
        MSB_LAUNCH_CHECK(ctx);
        MSB_CUDA_TRY(ctx, cudaEventRecord(s->ev_dp, st));
      }
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(s->xprev, s->xbuf[cur], N * sizeof(double),
                                        cudaMemcpyDeviceToDevice, st));
      // The static stages do not depend on the new partition: they are enqueued first and
      // run on the context stream while the rebuild (bins, components, merge, numbering,
      // A_c, factor) runs on the solver's rebuild stream; the dynamic stage waits for both.
      // The rebuild only touches its own scratch and the dynamic level, whose last reader
      // (the previous iteration's dynamic stage) precedes the Δp kernel the rebuild waits on.
      {
        cudaGraphExec_t ge = nullptr;
        int cur_next = cur;
        if ((rc = static_graph(ctx, s, db, cur, &ge, &cur_next))) return rc;
        MSB_CUDA_TRY(ctx, cudaGraphLaunch(ge, st));
        g_launches.fetch_add(s->sglaunches[cur], std::memory_order_relaxed);
        cur = cur_next;
      }
      if (rebuild) {
        cudaGraphExec_t lg = nullptr;
        if ((rc = labels_graph(ctx, s, &lg))) return rc;
        MSB_CUDA_TRY(ctx, cudaStreamWaitEvent(s->dyn_stream, s->ev_dp, 0));
        MSB_CUDA_TRY(ctx, cudaGraphLaunch(lg, s->dyn_stream));
        g_launches.fetch_add(s->lglaunches, std::memory_order_relaxed);
        MSB_CUDA_TRY(ctx, cudaEventRecord(s->ev_lab, s->dyn_stream));
        MSB_CUDA_TRY(ctx, cudaEventSynchronize(s->ev_lab));  // M_dyn, max|Δp| in dyn_pin
        double mxv = 0.0;
        dyn_read(s, &M, &mxv);
        if (!(mxv > 0.0)) M = 0;
        if (M > 0) {
          D->co.defer_check = true;
          ctx->stream = s->dyn_stream;
          rc = dyn_finish(ctx, s, M, nullptr);
          ctx->stream = st;
          D->co.defer_check = false;
          if (rc) return rc;
        }
        MSB_CUDA_TRY(ctx, cudaEventRecord(s->ev_dyn, s->dyn_stream));
        MSB_CUDA_TRY(ctx, cudaStreamWaitEvent(st, s->ev_dyn, 0));
      }
      dynM.push_back(M);
      bool first = false;  // norm already taken
      if (M > 0)
        if ((rc = enqueue_stage(ctx, s, s->dyn_level, db, cur, first))) return rc;
      cur_after.push_back(cur);
    }
  }
  int k = hs.k;
  int xb = cur_after[std::min<size_t>(k, cur_after.size() - 1)];
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(x, s->xbuf[xb], N * sizeof(double), cudaMemcpyDefault, st));
  if (res_hist)
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(res_hist, s->res_dev, (k + 1) * sizeof(double),
                                      cudaMemcpyDefault, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (ob) dfree(ctx, ob);
  if (dyn_M_hist) {
    for (size_t t = 0; t < dynM.size() && (int)t < cap; ++t) dyn_M_hist[t] = dynM[t];
  }
  if (iters_out) *iters_out = k;
  if (hs.diverged) return set_error(ctx, MSB_EDIVERGED, "residual grew by more than 1e6");
  if (fixed_iters > 0) return MSB_OK;
  if (!hs.converged) return MSB_NOT_CONVERGED;
  return MSB_OK;
}

msb_status msb_solver_destroy(msb_solver s) {
  if (!s) return MSB_EINVAL;
  msb_ctx ctx = s->ctx;
  dfree(ctx, s->xbuf[0]);
  dfree(ctx, s->xbuf[1]);
  dfree(ctx, s->xprev);
  dfree(ctx, s->r);
  dfree(ctx, s->dpbuf);
  dfree(ctx, s->rc);
  dfree(ctx, s->xc);
  dfree(ctx, s->partials);
  dfree(ctx, s->rc_part);
  dfree(ctx, s->st);
  dfree(ctx, s->res_dev);
  dfree(ctx, s->lab);
  dfree(ctx, s->ids);
  dfree(ctx, s->cnt);
  dfree(ctx, s->bins);
  dfree(ctx, s->scratch_i);
  dfree(ctx, s->mhist);
  if (s->dyn_level) level_free(s->dyn_level);
  dfree(ctx, s->ilu_d);
  drop_graphs(s);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->side_stream) cudaStreamDestroy(s->side_stream);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->dyn_stream) cudaStreamDestroy(s->dyn_stream);
  if (s->ev_dp) cudaEventDestroy(s->ev_dp);
  if (s->ev_dyn) cudaEventDestroy(s->ev_dyn);
  if (s->ev_lab) cudaEventDestroy(s->ev_lab);
  if (s->cap_stream2) cudaStreamDestroy(s->cap_stream2);
  if (s->ev_cf) cudaEventDestroy(s->ev_cf);
  if (s->ev_cj) cudaEventDestroy(s->ev_cj);
  dfree(ctx, s->dyn_gate);
  if (s->lgexec) cudaGraphExecDestroy(s->lgexec);
  if (s->dyn_pin) cudaFreeHost(s->dyn_pin);
  delete s;
  return MSB_OK;
}

}  // extern "C"

// z = M^{-1} v for FGMRES (fgmres.cu): one iteration of Eq. (8) over the solver's static
// levels from x = 0 with right-hand side v (no stop test, no dynamic stage).
namespace msb {
msb_status solver_smoother_setup(msb_ctx ctx, msb_solver s) {
  if (s->smoother != 1) return MSB_OK;
  if (!s->ilu_d) MSB_ALLOC(ctx, s->ilu_d, double, s->op->N);
  k_ilu_diag<<<grid_for(s->op->N, CT), CT, 0, ctx->stream>>>(stencil(s->op), s->ilu_d);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}


// Cartesian level's r_c = P^T r and x += P x_c outside a solver (NEXT-4 predictor,
// cpr.cu); `done` is a device int kept 0 (the kernels' stop-test flag)
msb_status level_restrict(msb_ctx ctx, msb_level L, const double* r, double* rc, const int* done) {
  if (L->kind != 0) return set_error(ctx, MSB_EINVAL, "level_restrict: Cartesian level only");
  if (L->nx > 2048) return set_error(ctx, MSB_EINVAL, "Cartesian restriction supports nx <= 2048");
  const LevelView V = view(L);
  const IterState* ist = reinterpret_cast<const IterState*>(done);  // `done` is its first member
  const size_t smem = restrict_rows_smem(L->nx);
  const unsigned gr = (unsigned)(L->nb[1] * L->nb[2]);
  const int xp = restrict_xp(L->nx);
  cudaStream_t st = ctx->stream;
  msb_status rc2 = xp == 1   ? launch_restrict<1, RCS>(ctx, st, gr, smem, V, r, rc, ist)
                   : xp == 2 ? launch_restrict<2, RCS>(ctx, st, gr, smem, V, r, rc, ist)
                   : xp == 4 ? launch_restrict<4, RCS>(ctx, st, gr, smem, V, r, rc, ist)
                             : launch_restrict<8, RCS>(ctx, st, gr, smem, V, r, rc, ist);
  if (rc2) return rc2;
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

msb_status level_prolong_add(msb_ctx ctx, msb_level L, double* x, const double* xc, const int* done) {
  if (L->kind != 0) return set_error(ctx, MSB_EINVAL, "level_prolong_add: Cartesian level only");
  const IterState* ist = reinterpret_cast<const IterState*>(done);
  k_prolong_cart<<<grid_for(L->N, CT), CT, 0, ctx->stream>>>(view(L), x, xc, ist);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

msb_status solver_precondition(msb_ctx ctx, msb_solver s, const double* v, double* z) {
  cudaStream_t st = ctx->stream;
  const int64_t N = s->op->N;
  // no stop test runs inside the preconditioner (first = false): only `done` is read,
  // and it must be 0 — a memset, not a pageable host copy, so nothing waits on the host
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(s->st, 0, sizeof(IterState), st));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(s->xbuf[0], 0, N * sizeof(double), st));
  int cur = 0;
  bool first = false;
  msb_status rc;
  for (msb_level L : s->levels)
    if ((rc = enqueue_stage(ctx, s, L, v, cur, first))) return rc;
  // the installed dynamic stage (msb_add_dynamic_basis, or the last one msb_ms_iterate
  // built) stays fixed over the solve: reading B6
  if (s->dyn && s->dyn_level && s->dyn_level->M > 0)
    if ((rc = enqueue_stage(ctx, s, s->dyn_level, v, cur, first))) return rc;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(z, s->xbuf[cur], N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return MSB_OK;
}
}  // namespace msb

