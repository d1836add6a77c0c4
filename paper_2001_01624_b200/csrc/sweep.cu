// Row a3 — MsRSB restricted-smoothing sweep (G2 Cartesian parity slots, G3 ELL).
//
//   P^_ij = (1-ω) P_ij + (ω/D_i) Σ_{l~i} T_il P_lj   on the pattern (positive form, A5)
//   P_ij <- P^_ij / Σ_k P^_ik                         every row (A6)
//   δ_n  = max |P^{n+1} - P^n|                         (A16)
//
// One thread per cell, all slots of the cell in registers (so the row sum and the
// renormalisation are free), coalesced fp64 loads of each slot plane and of the
// cell-padded transmissibilities.  Sweep n reads buffer n&1 and writes buffer
// (n+1)&1.  δ_n is folded per block into one of DSLOTS atomicMax slots (spreading
// the atomic traffic over DSLOTS L2 lines); sweep n+1 starts by reading sweep n's
// slots and returns at once when δ_n <= tol, so a chunk of sweeps is enqueued
// without host round trips and without any grid-wide fence.
#include <algorithm>

#include "internal.cuh"

namespace msb {

constexpr int DSLOTS = 16;
constexpr int SWEEP_BLOCK = 256;

__device__ __forceinline__ double nmax(double a, double b) { return (b > a || b != b) ? b : a; }

// true if the previous sweep already met the tolerance (block-uniform)
__device__ __forceinline__ bool sweep_skip(const unsigned long long* __restrict__ dslots, int n,
                                           double tol) {
  __shared__ int skip;
  if (threadIdx.x < 32) {
    double d = 0.0;
    if (n > 0 && tol >= 0.0 && threadIdx.x < DSLOTS)
      d = __longlong_as_double((long long)dslots[(n - 1) * DSLOTS + threadIdx.x]);
    for (int o = 16; o > 0; o >>= 1) d = nmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (threadIdx.x == 0) skip = (n > 0 && tol >= 0.0 && d <= tol) ? 1 : 0;
  }
  __syncthreads();
  return skip != 0;
}

__device__ __forceinline__ void sweep_fold(double v, unsigned long long* __restrict__ dslots,
                                           int n) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w = nmax(w, __shfl_xor_sync(0xffffffffu, w, o));
    if (threadIdx.x == 0)
      atomicMax(dslots + n * DSLOTS + (blockIdx.x % DSLOTS),
                (unsigned long long)__double_as_longlong(w));
  }
}

// ---------------------------------------------------------------- G2: Cartesian sweep
// Per-axis coordinate masks (built once per level from the parity table):
//   bit p      slot parity p is a support of this coordinate
//   bit 2+p    the -1 neighbour holds the same column in parity p
//   bit 4+p    the +1 neighbour holds the same column in parity p
// so the sweep needs three byte loads per cell and no column arithmetic.
__global__ void k_axis_mask(const int32_t* __restrict__ tab, int n, int off,
                            uint8_t* __restrict__ mask) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int32_t* t = tab + 2 * (off + x);
  uint8_t m = 0;
  for (int p = 0; p < 2; ++p) {
    if (t[p] < 0) continue;
    m |= 1u << p;
    if (x > 0 && tab[2 * (off + x - 1) + p] == t[p]) m |= 1u << (2 + p);
    if (x < n - 1 && tab[2 * (off + x + 1) + p] == t[p]) m |= 1u << (4 + p);
  }
  mask[off + x] = m;
}

__global__ void __launch_bounds__(SWEEP_BLOCK, 4) k_sweep_cart(
    double* __restrict__ P0, double* __restrict__ P1, const double* __restrict__ Tx,
    const double* __restrict__ Ty, const double* __restrict__ Tz, const uint8_t* __restrict__ amask,
    Grid3 g, double omega, int n, double tol, unsigned long long* __restrict__ dslots) {
  if (sweep_skip(dslots, n, tol)) return;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int N = g.nxy * g.nz;
  const int nx = g.nx, sxy = g.nxy;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double dloc = 0.0;
  if (c < N) {
    int i, j, k;
    g3_coords(g, c, i, j, k);
    const unsigned mx = amask[i], my = amask[nx + j], mz = amask[nx + g.ny + k];
    double txp = Tx[c], typ = Ty[c], tzp = Tz[c];
    double txm = i > 0 ? Tx[c - 1] : 0.0;
    double tym = j > 0 ? Ty[c - nx] : 0.0;
    double tzm = k > 0 ? Tz[c - sxy] : 0.0;
    double D = txp + txm + typ + tym + tzp + tzm;
    double wD = omega / D;
    double om1 = 1.0 - omega;
    double ph[8];
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
      ph[s] = 0.0;
      if ((mx >> px) & (my >> py) & (mz >> pz) & 1u) {
        const double* __restrict__ base = Pin + (size_t)s * N;
        double acc = 0.0;
        if ((mz >> (2 + pz)) & 1u) acc += tzm * base[c - sxy];
        if ((my >> (2 + py)) & 1u) acc += tym * base[c - nx];
        if ((mx >> (2 + px)) & 1u) acc += txm * base[c - 1];
        if ((mx >> (4 + px)) & 1u) acc += txp * base[c + 1];
        if ((my >> (4 + py)) & 1u) acc += typ * base[c + nx];
        if ((mz >> (4 + pz)) & 1u) acc += tzp * base[c + sxy];
        double p = base[c];
        ph[s] = om1 * p + wD * acc;
        sum += ph[s];
      }
    }
    // second pass: the cell's own P values are re-read (L1 hits) instead of being
    // held in registers, which keeps the kernel at 4 blocks/SM
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
      if ((mx >> px) & (my >> py) & (mz >> pz) & 1u) {
        double pn = ph[s] / sum;
        double po = __ldca(Pin + (size_t)s * N + c);
        Pout[(size_t)s * N + c] = pn;
        dloc = nmax(dloc, fabs(pn - po));
      }
    }
  }
  sweep_fold(dloc, dslots, n);
}

// ---------------------------------------------------------------- G3: explicit (ELL) sweep
constexpr int ELL_MAXW = 16;

__global__ void __launch_bounds__(SWEEP_BLOCK) k_sweep_ell(
    double* __restrict__ P0, double* __restrict__ P1, const double* __restrict__ Tx,
    const double* __restrict__ Ty, const double* __restrict__ Tz, const int32_t* __restrict__ col,
    const int8_t* __restrict__ nbs, int W, Grid3 g, double omega, int n, double tol,
    unsigned long long* __restrict__ dslots) {
  if (sweep_skip(dslots, n, tol)) return;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int N = g.nxy * g.nz;
  const int nx = g.nx, sxy = g.nxy;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double dloc = 0.0;
  if (c < N) {
    int i, j, k;
    g3_coords(g, c, i, j, k);
    double t[6];
    int nb[6];
    t[0] = k > 0 ? Tz[c - sxy] : 0.0;       nb[0] = c - sxy;
    t[1] = j > 0 ? Ty[c - nx] : 0.0;        nb[1] = c - nx;
    t[2] = i > 0 ? Tx[c - 1] : 0.0;         nb[2] = c - 1;
    t[3] = Tx[c];                           nb[3] = c + 1;
    t[4] = Ty[c];                           nb[4] = c + nx;
    t[5] = Tz[c];                           nb[5] = c + sxy;
    double D = t[3] + t[2] + t[4] + t[1] + t[5] + t[0];
    double wD = omega / D;
    double om1 = 1.0 - omega;
    double ph[ELL_MAXW], po[ELL_MAXW];
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < ELL_MAXW; ++s) {
      ph[s] = 0.0;
      po[s] = 0.0;
      if (s < W && col[(size_t)s * N + c] >= 0) {
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          int sl = nbs[((size_t)d * W + s) * N + c];
          if (sl >= 0) acc += t[d] * Pin[(size_t)sl * N + nb[d]];
        }
        double p = Pin[(size_t)s * N + c];
        po[s] = p;
        ph[s] = om1 * p + wD * acc;
        sum += ph[s];
      }
    }
#pragma unroll
    for (int s = 0; s < ELL_MAXW; ++s) {
      if (s < W && col[(size_t)s * N + c] >= 0) {
        double pn = ph[s] / sum;
        Pout[(size_t)s * N + c] = pn;
        dloc = nmax(dloc, fabs(pn - po[s]));
      }
    }
  }
  sweep_fold(dloc, dslots, n);
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_smooth_basis(msb_ctx ctx, msb_level L, msb_op op, int32_t max_sweeps,
                                       double omega, double tol, int32_t* sweeps_done,
                                       double* last_delta, double* deltas) {
  if (!ctx || !L || !op) return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: null");
  if (max_sweeps < 0 || !(omega > 0.0) || !(omega <= 1.0))
    return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: bad max_sweeps/omega");
  if (L->N != op->N) return set_error(ctx, MSB_EDIM, "level/operator size mismatch");
  if (L->kind == 1 && L->W > ELL_MAXW)
    return set_error(ctx, MSB_EINVAL, "ELL width %d exceeds %d", L->W, ELL_MAXW);
  if (sweeps_done) *sweeps_done = 0;
  if (last_delta) *last_delta = 0.0;
  if (max_sweeps == 0) return MSB_OK;
  cudaStream_t st = ctx->stream;
  unsigned long long* dslots = dalloc_n<unsigned long long>(ctx, (size_t)max_sweeps * DSLOTS);
  if (!dslots) return set_error(ctx, MSB_ENOMEM, "sweep state");
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(dslots, 0, (size_t)max_sweeps * DSLOTS * 8, st));
  Grid3 g = make_grid3(op->nx, op->ny, op->nz);
  if (L->kind == 0 && !L->amask) {
    int tot = op->nx + op->ny + op->nz;
    MSB_ALLOC(ctx, L->amask, uint8_t, tot);
    int dims[3] = {op->nx, op->ny, op->nz};
    int off = 0;
    for (int a = 0; a < 3; ++a) {
      k_axis_mask<<<grid_for(dims[a], 128), 128, 0, st>>>(L->tab, dims[a], off, L->amask);
      MSB_LAUNCH_CHECK(ctx);
      off += dims[a];
    }
  }
  double* Pa = L->P[L->cur];
  double* Pb = L->P[L->cur ^ 1];
  const unsigned grid = grid_for(L->N, SWEEP_BLOCK);
  const int chunk = 32;
  int issued = 0, n = 0;
  double last = 0.0;
  bool bad = false, done = false;
  std::vector<unsigned long long> hb;
  while (!done && issued < max_sweeps) {
    int nl = std::min(chunk, max_sweeps - issued);
    for (int t = 0; t < nl; ++t) {
      int idx = issued + t;
      if (L->kind == 0)
        k_sweep_cart<<<grid, SWEEP_BLOCK, 0, st>>>(Pa, Pb, op->Tx, op->Ty, op->Tz, L->amask, g,
                                                   omega, idx, tol, dslots);
      else
        k_sweep_ell<<<grid, SWEEP_BLOCK, 0, st>>>(Pa, Pb, op->Tx, op->Ty, op->Tz, L->col, L->nbs,
                                                  L->W, g, omega, idx, tol, dslots);
      MSB_LAUNCH_CHECK(ctx);
    }
    hb.resize((size_t)nl * DSLOTS);
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hb.data(), dslots + (size_t)issued * DSLOTS,
                                      hb.size() * 8, cudaMemcpyDeviceToHost, st));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    for (int t = 0; t < nl && !done; ++t) {
      double d = 0.0;
      for (int q = 0; q < DSLOTS; ++q) {
        double v;
        memcpy(&v, &hb[(size_t)t * DSLOTS + q], 8);
        d = (v > d || v != v) ? v : d;
      }
      if (!(d == d)) bad = true;
      if (deltas) deltas[issued + t] = d;
      last = d;
      n = issued + t + 1;
      if (tol >= 0.0 && d <= tol) done = true;
    }
    issued += nl;
  }
  dfree(ctx, dslots);
  if (n & 1) L->cur ^= 1;
  if (sweeps_done) *sweeps_done = n;
  if (last_delta) *last_delta = last;
  if (bad) return set_error(ctx, MSB_EZERO_DIAG, "non-finite update: zero diagonal in A_T");
  if (tol >= 0.0 && !done) return MSB_NOT_CONVERGED;
  return MSB_OK;
}
