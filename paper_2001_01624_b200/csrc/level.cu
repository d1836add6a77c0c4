// Rows a2 (Cartesian supports) and a3 (MsRSB restricted smoothing sweep, G2/G3).
//
// Prolongation storage: W slot planes, P[s*N + c] (SoA, fp64), double-buffered.
//
// Cartesian level (kind 0): under the open-box support rule (reading A3) a cell lies
// in the supports of at most two consecutive blocks per axis, and consecutive block
// indices have different parity.  Slot s = (px | py<<1 | pz<<2) therefore holds the
// basis function whose block index along axis a has parity p_a, for every cell —
// the column a slot refers to is a pure function of (cell, slot), and a neighbour's
// value of the same column sits in the SAME slot plane whenever the neighbour lies
// in that column's support (checked with the per-axis parity table).  Each slot
// plane is then an independent masked 7-point stencil with coalesced loads; no
// column indices are stored or read.
//
// Explicit level (kind 1, fault-split / constant bases): W ELL slots per cell with a
// column index plane and a per-direction neighbour-slot map (int8).
#include "internal.cuh"

namespace msb {

struct SweepState {
  int done;
  int n;          // sweeps completed
  int arrive;
  int max_sweeps;
  double tol;     // < 0: never stop on δ
};

// ---------------------------------------------------------------- axis parity table
// tab[(off_a + x)*2 + p] = block index with parity p whose support contains x, or -1.
__global__ void k_axis_tab(int n, int b, int off, int32_t* __restrict__ tab) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  int nb = (n + b - 1) / b;
  int J = x / b;
  int loJ = J * b, hiJ = min(loJ + b, n);
  int C = loJ + hiJ;  // doubled centre of block J
  int other = -1;
  if (J > 0 && 2 * x + 1 < C) other = J - 1;
  if (J < nb - 1 && 2 * x + 1 > C) other = J + 1;
  int t[2] = {-1, -1};
  t[J & 1] = J;
  if (other >= 0) t[other & 1] = other;
  tab[(off + x) * 2 + 0] = t[0];
  tab[(off + x) * 2 + 1] = t[1];
}

__global__ void k_cart_init(const int32_t* __restrict__ tab, int nx, int ny, int nz, int nbx,
                            int nby, double* __restrict__ P, const int32_t* __restrict__ part,
                            unsigned long long* __restrict__ nnz) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cnt = 0;
  if (c < N) {
    int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((int64_t)nx * ny));
    const int32_t* tx = tab + 2 * i;
    const int32_t* ty = tab + 2 * (nx + j);
    const int32_t* tz = tab + 2 * (nx + ny + k);
    for (int s = 0; s < 8; ++s) {
      cnt += (tx[s & 1] >= 0 && ty[(s >> 1) & 1] >= 0 && tz[s >> 2] >= 0);
      P[(int64_t)s * N + c] = 0.0;
    }
    int J = part[c];
    int ox = J % nbx, oy = (J / nbx) % nby, oz = J / (nbx * nby);
    int so = (ox & 1) | ((oy & 1) << 1) | ((oz & 1) << 2);
    P[(int64_t)so * N + c] = 1.0;   // P^0 = indicator of the partition
  }
  __shared__ int sh[32];
  int v = cnt;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (threadIdx.x == 0) atomicAdd(nnz, (unsigned long long)w);
  }
}

__global__ void k_cart_part(int nx, int ny, int nz, int bx, int by, int bz, int nbx, int nby,
                            int32_t* __restrict__ part) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((int64_t)nx * ny));
  part[c] = i / bx + nbx * (j / by + nby * (k / bz));
}

// ---------------------------------------------------------------- reductions
// NaN-propagating max (a zero diagonal must surface as a non-finite δ).
__device__ __forceinline__ double nmax(double a, double b) { return (b > a || b != b) ? b : a; }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block max of nonnegative v, folded into *slot (as ordered bits); the last block to
// arrive finalises the sweep.
__device__ __forceinline__ void sweep_epilogue(double v, unsigned long long* dmax,
                                               SweepState* st, int n) {
  __shared__ double sh[32];
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    w = warp_max(w);
    if (threadIdx.x == 0) {
      atomicMax(dmax + n, (unsigned long long)__double_as_longlong(w));
      __threadfence();
      int t = atomicAdd(&st->arrive, 1);
      if (t == (int)gridDim.x - 1) {
        __threadfence();
        unsigned long long bits = atomicAdd(dmax + n, 0ull);
        double d = __longlong_as_double((long long)bits);
        int nn = n + 1;
        st->n = nn;
        if ((st->tol >= 0.0 && d <= st->tol) || nn >= st->max_sweeps) st->done = 1;
        st->arrive = 0;
        __threadfence();
      }
    }
  }
}

// ---------------------------------------------------------------- G2: Cartesian sweep
__global__ void __launch_bounds__(256) k_sweep_cart(double* __restrict__ P0, double* __restrict__ P1,
                                                    const double* __restrict__ Tx,
                                                    const double* __restrict__ Ty,
                                                    const double* __restrict__ Tz,
                                                    const int32_t* __restrict__ tab, int nx,
                                                    int ny, int nz, double omega,
                                                    SweepState* st,
                                                    unsigned long long* __restrict__ dmax) {
  if (*(volatile int*)&st->done) return;
  const int n = *(volatile int*)&st->n;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int64_t N = (int64_t)nx * ny * nz;
  const int64_t sxy = (int64_t)nx * ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double dloc = 0.0;
  if (c < N) {
    int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
    int2 bx = *(const int2*)(tab + 2 * i);
    int2 by = *(const int2*)(tab + 2 * (nx + j));
    int2 bz = *(const int2*)(tab + 2 * (nx + ny + k));
    int2 bxm = i > 0 ? *(const int2*)(tab + 2 * (i - 1)) : make_int2(-2, -2);
    int2 bxp = i < nx - 1 ? *(const int2*)(tab + 2 * (i + 1)) : make_int2(-2, -2);
    int2 bym = j > 0 ? *(const int2*)(tab + 2 * (nx + j - 1)) : make_int2(-2, -2);
    int2 byp = j < ny - 1 ? *(const int2*)(tab + 2 * (nx + j + 1)) : make_int2(-2, -2);
    int2 bzm = k > 0 ? *(const int2*)(tab + 2 * (nx + ny + k - 1)) : make_int2(-2, -2);
    int2 bzp = k < nz - 1 ? *(const int2*)(tab + 2 * (nx + ny + k + 1)) : make_int2(-2, -2);
    double txp = Tx[c], typ = Ty[c], tzp = Tz[c];
    double txm = i > 0 ? Tx[c - 1] : 0.0;
    double tym = j > 0 ? Ty[c - nx] : 0.0;
    double tzm = k > 0 ? Tz[c - sxy] : 0.0;
    double D = txp + txm + typ + tym + tzp + tzm;
    double wD = omega / D;
    double om1 = 1.0 - omega;
    double ph[8], po[8];
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
      int jx = px ? bx.y : bx.x;
      int jy = py ? by.y : by.x;
      int jz = pz ? bz.y : bz.x;
      ph[s] = 0.0;
      po[s] = 0.0;
      if (jx >= 0 && jy >= 0 && jz >= 0) {
        const double* __restrict__ base = Pin + (int64_t)s * N;
        double acc = 0.0;
        if ((pz ? bzm.y : bzm.x) == jz) acc += tzm * base[c - sxy];
        if ((py ? bym.y : bym.x) == jy) acc += tym * base[c - nx];
        if ((px ? bxm.y : bxm.x) == jx) acc += txm * base[c - 1];
        if ((px ? bxp.y : bxp.x) == jx) acc += txp * base[c + 1];
        if ((py ? byp.y : byp.x) == jy) acc += typ * base[c + nx];
        if ((pz ? bzp.y : bzp.x) == jz) acc += tzp * base[c + sxy];
        double p = base[c];
        po[s] = p;
        ph[s] = om1 * p + wD * acc;
        sum += ph[s];
      }
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
      int jx = px ? bx.y : bx.x;
      int jy = py ? by.y : by.x;
      int jz = pz ? bz.y : bz.x;
      if (jx >= 0 && jy >= 0 && jz >= 0) {
        double pn = ph[s] / sum;
        Pout[(int64_t)s * N + c] = pn;
        dloc = nmax(dloc, fabs(pn - po[s]));
      }
    }
  }
  sweep_epilogue(dloc, dmax, st, n);
}

// ---------------------------------------------------------------- G3: explicit (ELL) sweep
__global__ void __launch_bounds__(256) k_sweep_ell(double* __restrict__ P0, double* __restrict__ P1,
                                                   const double* __restrict__ Tx,
                                                   const double* __restrict__ Ty,
                                                   const double* __restrict__ Tz,
                                                   const int32_t* __restrict__ col,
                                                   const int8_t* __restrict__ nbs, int W, int nx,
                                                   int ny, int nz, double omega, SweepState* st,
                                                   unsigned long long* __restrict__ dmax) {
  if (*(volatile int*)&st->done) return;
  const int n = *(volatile int*)&st->n;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int64_t N = (int64_t)nx * ny * nz;
  const int64_t sxy = (int64_t)nx * ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double dloc = 0.0;
  if (c < N) {
    int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
    double t[6];
    int64_t nb[6];
    t[0] = k > 0 ? Tz[c - sxy] : 0.0;       nb[0] = c - sxy;
    t[1] = j > 0 ? Ty[c - nx] : 0.0;        nb[1] = c - nx;
    t[2] = i > 0 ? Tx[c - 1] : 0.0;         nb[2] = c - 1;
    t[3] = Tx[c];                           nb[3] = c + 1;
    t[4] = Ty[c];                           nb[4] = c + nx;
    t[5] = Tz[c];                           nb[5] = c + sxy;
    double D = t[3] + t[2] + t[4] + t[1] + t[5] + t[0];
    double wD = omega / D;
    double om1 = 1.0 - omega;
    double sum = 0.0;
    // pass 1: row sum of P^
    for (int s = 0; s < W; ++s) {
      if (col[(int64_t)s * N + c] < 0) continue;
      double acc = 0.0;
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        int sl = nbs[((int64_t)d * W + s) * N + c];
        if (sl >= 0) acc += t[d] * Pin[(int64_t)sl * N + nb[d]];
      }
      sum += om1 * Pin[(int64_t)s * N + c] + wD * acc;
    }
    // pass 2: recompute (identical arithmetic) and normalise
    for (int s = 0; s < W; ++s) {
      if (col[(int64_t)s * N + c] < 0) continue;
      double acc = 0.0;
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        int sl = nbs[((int64_t)d * W + s) * N + c];
        if (sl >= 0) acc += t[d] * Pin[(int64_t)sl * N + nb[d]];
      }
      double p = Pin[(int64_t)s * N + c];
      double pn = (om1 * p + wD * acc) / sum;
      Pout[(int64_t)s * N + c] = pn;
      dloc = nmax(dloc, fabs(pn - p));
    }
  }
  sweep_epilogue(dloc, dmax, st, n);
}

// ---------------------------------------------------------------- export helpers
// per-cell active count
__global__ void k_row_counts(const msb_level_s L, int32_t* __restrict__ cnt) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.N) return;
  int n = 0;
  if (L.kind == 0) {
    int i = (int)(c % L.nx), j = (int)((c / L.nx) % L.ny), k = (int)(c / ((int64_t)L.nx * L.ny));
    const int32_t* tx = L.tab + 2 * i;
    const int32_t* ty = L.tab + 2 * (L.nx + j);
    const int32_t* tz = L.tab + 2 * (L.nx + L.ny + k);
    for (int s = 0; s < 8; ++s) n += (tx[s & 1] >= 0 && ty[(s >> 1) & 1] >= 0 && tz[s >> 2] >= 0);
  } else {
    for (int s = 0; s < L.W; ++s) n += L.col[(int64_t)s * L.N + c] >= 0;
  }
  cnt[c] = n;
}

__device__ __forceinline__ int slot_col(const msb_level_s& L, int64_t c, int s) {
  if (L.kind == 1) return L.col[(int64_t)s * L.N + c];
  int i = (int)(c % L.nx), j = (int)((c / L.nx) % L.ny), k = (int)(c / ((int64_t)L.nx * L.ny));
  int jx = L.tab[2 * i + (s & 1)], jy = L.tab[2 * (L.nx + j) + ((s >> 1) & 1)],
      jz = L.tab[2 * (L.nx + L.ny + k) + (s >> 2)];
  if (jx < 0 || jy < 0 || jz < 0) return -1;
  return jx + L.nb[0] * (jy + L.nb[1] * jz);
}

__global__ void k_export_csr(const msb_level_s L, const double* __restrict__ P,
                             const int32_t* __restrict__ start, int32_t* __restrict__ cols,
                             double* __restrict__ vals) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.N) return;
  int cc[32];
  double vv[32];
  int n = 0;
  for (int s = 0; s < L.W && n < 32; ++s) {
    int j = slot_col(L, c, s);
    if (j < 0) continue;
    double v = P[(int64_t)s * L.N + c];
    int p = n++;
    while (p > 0 && cc[p - 1] > j) {
      cc[p] = cc[p - 1];
      vv[p] = vv[p - 1];
      --p;
    }
    cc[p] = j;
    vv[p] = v;
  }
  int64_t o = start[c];
  for (int t = 0; t < n; ++t) {
    if (cols) cols[o + t] = cc[t];
    if (vals) vals[o + t] = vv[t];
  }
}

__global__ void k_import_csr(const msb_level_s L, double* __restrict__ P,
                             const int32_t* __restrict__ start, const double* __restrict__ vals) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.N) return;
  // ranks of slot columns give the CSR offset
  int cols_[32], slots[32];
  int n = 0;
  for (int s = 0; s < L.W && n < 32; ++s) {
    int j = slot_col(L, c, s);
    if (j < 0) continue;
    int p = n++;
    while (p > 0 && cols_[p - 1] > j) {
      cols_[p] = cols_[p - 1];
      slots[p] = slots[p - 1];
      --p;
    }
    cols_[p] = j;
    slots[p] = s;
  }
  int64_t o = start[c];
  for (int t = 0; t < n; ++t) P[(int64_t)slots[t] * L.N + c] = vals[o + t];
}

__global__ void k_i32_to_i64_rowptr(const int32_t* __restrict__ start, int64_t n, int64_t total,
                                    int64_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = start[i];
  if (i == n) out[n] = total;
}

// ---------------------------------------------------------------- constant (explicit) level
__global__ void k_const_init(const int32_t* __restrict__ part, int64_t N, int M,
                             int32_t* __restrict__ col, double* __restrict__ P0,
                             double* __restrict__ P1, int* __restrict__ bad) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int j = part[c];
  if (j < 0 || j >= M) atomicExch(bad, 1);
  col[c] = j;
  P0[c] = 1.0;
  P1[c] = 1.0;
}

__global__ void k_nbs_ell(const int32_t* __restrict__ col, int W, int nx, int ny, int nz,
                          int8_t* __restrict__ nbs) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t sxy = (int64_t)nx * ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  int64_t nb[6] = {c - sxy, c - nx, c - 1, c + 1, c + nx, c + sxy};
  bool ex[6] = {k > 0, j > 0, i > 0, i < nx - 1, j < ny - 1, k < nz - 1};
  for (int s = 0; s < W; ++s) {
    int jc = col[(int64_t)s * N + c];
    for (int d = 0; d < 6; ++d) {
      int r = -1;
      if (jc >= 0 && ex[d]) {
        for (int t = 0; t < W; ++t)
          if (col[(int64_t)t * N + nb[d]] == jc) {
            r = t;
            break;
          }
      }
      nbs[((int64_t)d * W + s) * N + c] = (int8_t)r;
    }
  }
}

msb_status level_build_explicit_from_part(msb_ctx ctx, msb_op op, const int32_t* part_dev,
                                          int M, msb_level* out) {
  msb_level L = new msb_level_s();
  L->ctx = ctx;
  L->kind = 1;
  L->N = op->N;
  L->M = M;
  L->W = 1;
  L->nnz = op->N;
  L->nx = op->nx; L->ny = op->ny; L->nz = op->nz;
  MSB_ALLOC(ctx, L->P[0], double, op->N);
  MSB_ALLOC(ctx, L->P[1], double, op->N);
  MSB_ALLOC(ctx, L->col, int32_t, op->N);
  MSB_ALLOC(ctx, L->part, int32_t, op->N);
  MSB_ALLOC(ctx, L->nbs, int8_t, 6 * op->N);
  int* bad = dalloc_n<int>(ctx, 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(L->part, part_dev, op->N * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  k_const_init<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(L->part, op->N, M, L->col, L->P[0],
                                                              L->P[1], bad);
  MSB_LAUNCH_CHECK(ctx);
  k_nbs_ell<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(L->col, 1, op->nx, op->ny, op->nz,
                                                           L->nbs);
  MSB_LAUNCH_CHECK(ctx);
  int hbad = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, bad);
  if (hbad) {
    level_free(L);
    return set_error(ctx, MSB_EINVAL, "partition value out of [0, M)");
  }
  *out = L;
  return MSB_OK;
}

void level_free(msb_level L) {
  if (!L) return;
  msb_ctx ctx = L->ctx;
  dfree(ctx, L->P[0]);
  dfree(ctx, L->P[1]);
  dfree(ctx, L->part);
  dfree(ctx, L->tab);
  dfree(ctx, L->col);
  dfree(ctx, L->nbs);
  coarse_free(ctx, L->co);
  delete L;
}

}  // namespace msb

using namespace msb;

extern "C" {

msb_status msb_partition_cartesian(msb_ctx ctx, const msb_grid* g, int32_t bx, int32_t by,
                                   int32_t bz, int32_t* part, int32_t* M_out) {
  if (!ctx || !g || bx < 1 || by < 1 || bz < 1) return set_error(ctx, MSB_EINVAL, "partition args");
  int nbx = (g->nx + bx - 1) / bx, nby = (g->ny + by - 1) / by, nbz = (g->nz + bz - 1) / bz;
  if (M_out) *M_out = nbx * nby * nbz;
  if (part) {
    int64_t N = (int64_t)g->nx * g->ny * g->nz;
    int32_t* d = part;
    bool dev = is_device_ptr(part);
    if (!dev) d = dalloc_n<int32_t>(ctx, N);
    k_cart_part<<<grid_for(N, 256), 256, 0, ctx->stream>>>(g->nx, g->ny, g->nz, bx, by, bz, nbx,
                                                           nby, d);
    MSB_LAUNCH_CHECK(ctx);
    if (!dev) {
      MSB_CUDA_TRY(ctx, copy_out(ctx, part, d, N * sizeof(int32_t)));
      dfree(ctx, d);
    }
  }
  return MSB_OK;
}

msb_status msb_level_create_cartesian(msb_ctx ctx, msb_op op, int32_t bx, int32_t by, int32_t bz,
                                      msb_level* out, int64_t* nnz_out) {
  if (!ctx || !op || !out || bx < 1 || by < 1 || bz < 1)
    return set_error(ctx, MSB_EINVAL, "msb_level_create_cartesian args");
  msb_level L = new msb_level_s();
  L->ctx = ctx;
  L->kind = 0;
  L->N = op->N;
  L->nx = op->nx; L->ny = op->ny; L->nz = op->nz;
  L->bs[0] = bx; L->bs[1] = by; L->bs[2] = bz;
  L->nb[0] = (op->nx + bx - 1) / bx;
  L->nb[1] = (op->ny + by - 1) / by;
  L->nb[2] = (op->nz + bz - 1) / bz;
  L->M = L->nb[0] * L->nb[1] * L->nb[2];
  L->W = 8;
  MSB_ALLOC(ctx, L->tab, int32_t, 2 * (op->nx + op->ny + op->nz));
  MSB_ALLOC(ctx, L->P[0], double, 8 * op->N);
  MSB_ALLOC(ctx, L->P[1], double, 8 * op->N);
  MSB_ALLOC(ctx, L->part, int32_t, op->N);
  int dims[3] = {op->nx, op->ny, op->nz};
  int off = 0;
  for (int a = 0; a < 3; ++a) {
    k_axis_tab<<<grid_for(dims[a], 128), 128, 0, ctx->stream>>>(dims[a], L->bs[a], off, L->tab);
    MSB_LAUNCH_CHECK(ctx);
    off += dims[a];
  }
  k_cart_part<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(op->nx, op->ny, op->nz, bx, by, bz,
                                                             L->nb[0], L->nb[1], L->part);
  MSB_LAUNCH_CHECK(ctx);
  unsigned long long* dn = dalloc_n<unsigned long long>(ctx, 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(dn, 0, 8, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(L->P[1], 0, 8 * op->N * sizeof(double), ctx->stream));
  k_cart_init<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(L->tab, op->nx, op->ny, op->nz,
                                                             L->nb[0], L->nb[1], L->P[0], L->part,
                                                             dn);
  MSB_LAUNCH_CHECK(ctx);
  unsigned long long hn = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hn, dn, 8, cudaMemcpyDeviceToHost, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, dn);
  L->nnz = (int64_t)hn;
  if (nnz_out) *nnz_out = L->nnz;
  *out = L;
  return MSB_OK;
}

msb_status msb_level_create_constant(msb_ctx ctx, msb_op op, const int32_t* part, int32_t M,
                                     msb_level* out) {
  if (!ctx || !op || !part || !out || M < 1) return set_error(ctx, MSB_EINVAL, "constant level args");
  void* o = nullptr;
  const int32_t* d = (const int32_t*)stage_in(ctx, part, op->N * sizeof(int32_t), &o);
  msb_status st = level_build_explicit_from_part(ctx, op, d, M, out);
  if (o) {
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx, o);
  }
  return st;
}

msb_status msb_level_info(msb_ctx ctx, msb_level L, int32_t* M, int64_t* nnz, int32_t* W,
                          int32_t* part) {
  if (!ctx || !L) return set_error(ctx, MSB_EINVAL, "msb_level_info: null");
  if (M) *M = L->M;
  if (nnz) *nnz = L->nnz;
  if (W) *W = L->W;
  if (part) MSB_CUDA_TRY(ctx, copy_out(ctx, part, L->part, L->N * sizeof(int32_t)));
  return sync(ctx);
}

msb_status msb_level_export(msb_ctx ctx, msb_level L, int64_t* rowptr, int32_t* cols,
                            double* vals, double* Ac) {
  if (!ctx || !L) return set_error(ctx, MSB_EINVAL, "msb_level_export: null");
  int64_t N = L->N;
  if (rowptr || cols || vals) {
    int32_t* cnt = dalloc_n<int32_t>(ctx, N);
    int32_t* start = dalloc_n<int32_t>(ctx, N);
    k_row_counts<<<grid_for(N, 256), 256, 0, ctx->stream>>>(*L, cnt);
    MSB_LAUNCH_CHECK(ctx);
    int32_t total = 0;
    msb_status st = scan_exclusive(ctx, cnt, start, N, &total);
    if (st != MSB_OK) return st;
    if (total != L->nnz) return set_error(ctx, MSB_EINVAL, "nnz mismatch %d vs %lld", total, (long long)L->nnz);
    int32_t* dcols = nullptr;
    double* dvals = nullptr;
    if (cols) dcols = dalloc_n<int32_t>(ctx, total);
    if (vals) dvals = dalloc_n<double>(ctx, total);
    k_export_csr<<<grid_for(N, 128), 128, 0, ctx->stream>>>(*L, L->P[L->cur], start, dcols, dvals);
    MSB_LAUNCH_CHECK(ctx);
    if (rowptr) {
      int64_t* drp = dalloc_n<int64_t>(ctx, N + 1);
      k_i32_to_i64_rowptr<<<grid_for(N + 1, 256), 256, 0, ctx->stream>>>(start, N, total, drp);
      MSB_LAUNCH_CHECK(ctx);
      MSB_CUDA_TRY(ctx, copy_out(ctx, rowptr, drp, (N + 1) * sizeof(int64_t)));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      dfree(ctx, drp);
    }
    if (cols) MSB_CUDA_TRY(ctx, copy_out(ctx, cols, dcols, (size_t)total * sizeof(int32_t)));
    if (vals) MSB_CUDA_TRY(ctx, copy_out(ctx, vals, dvals, (size_t)total * sizeof(double)));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    dfree(ctx, dcols);
    dfree(ctx, dvals);
    dfree(ctx, cnt);
    dfree(ctx, start);
  }
  if (Ac) {
    if (!L->co.Ac) return set_error(ctx, MSB_EINVAL, "no dense coarse operator assembled");
    MSB_CUDA_TRY(ctx, copy_out(ctx, Ac, L->co.Ac, (size_t)L->M * L->M * sizeof(double)));
  }
  return sync(ctx);
}

msb_status msb_level_import_values(msb_ctx ctx, msb_level L, const double* vals) {
  if (!ctx || !L || !vals) return set_error(ctx, MSB_EINVAL, "import: null");
  int64_t N = L->N;
  int32_t* cnt = dalloc_n<int32_t>(ctx, N);
  int32_t* start = dalloc_n<int32_t>(ctx, N);
  k_row_counts<<<grid_for(N, 256), 256, 0, ctx->stream>>>(*L, cnt);
  MSB_LAUNCH_CHECK(ctx);
  int32_t total = 0;
  msb_status st = scan_exclusive(ctx, cnt, start, N, &total);
  if (st != MSB_OK) return st;
  void* o = nullptr;
  const double* d = (const double*)stage_in(ctx, vals, (size_t)total * sizeof(double), &o);
  k_import_csr<<<grid_for(N, 128), 128, 0, ctx->stream>>>(*L, L->P[L->cur], start, d);
  MSB_LAUNCH_CHECK(ctx);
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (o) dfree(ctx, o);
  dfree(ctx, cnt);
  dfree(ctx, start);
  return MSB_OK;
}

msb_status msb_level_destroy(msb_level L) {
  if (!L) return MSB_EINVAL;
  level_free(L);
  return MSB_OK;
}

msb_status msb_smooth_basis(msb_ctx ctx, msb_level L, msb_op op, int32_t max_sweeps, double omega,
                            double tol, int32_t* sweeps_done, double* last_delta, double* deltas) {
  if (!ctx || !L || !op) return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: null");
  if (max_sweeps < 0 || !(omega > 0.0) || !(omega <= 1.0))
    return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: bad max_sweeps/omega");
  if (L->N != op->N) return set_error(ctx, MSB_EDIM, "level/operator size mismatch");
  if (sweeps_done) *sweeps_done = 0;
  if (max_sweeps == 0) return MSB_OK;
  SweepState* st = dalloc_n<SweepState>(ctx, 1);
  unsigned long long* dmax = dalloc_n<unsigned long long>(ctx, max_sweeps);
  if (!st || !dmax) return set_error(ctx, MSB_ENOMEM, "sweep state");
  SweepState h{0, 0, 0, max_sweeps, tol};
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(dmax, 0, max_sweeps * sizeof(unsigned long long), ctx->stream));
  // zero-diagonal check is part of every sweep: D = 0 gives inf/nan and
  // is detected on the δ history below.
  double* Pa = L->P[L->cur];
  double* Pb = L->P[L->cur ^ 1];
  const int chunk = 32;
  int issued = 0;
  SweepState hs{};
  while (true) {
    int nlaunch = std::min(chunk, max_sweeps - issued);
    for (int t = 0; t < nlaunch; ++t) {
      if (L->kind == 0) {
        k_sweep_cart<<<grid_for(L->N, 256), 256, 0, ctx->stream>>>(
            Pa, Pb, op->Tx, op->Ty, op->Tz, L->tab, op->nx, op->ny, op->nz, omega, st, dmax);
      } else {
        k_sweep_ell<<<grid_for(L->N, 256), 256, 0, ctx->stream>>>(
            Pa, Pb, op->Tx, op->Ty, op->Tz, L->col, L->nbs, L->W, op->nx, op->ny, op->nz, omega,
            st, dmax);
      }
      MSB_LAUNCH_CHECK(ctx);
    }
    issued += nlaunch;
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (hs.done || issued >= max_sweeps) break;
  }
  int n = hs.n;
  std::vector<unsigned long long> bits(max_sweeps);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(bits.data(), dmax, max_sweeps * 8, cudaMemcpyDeviceToHost,
                                    ctx->stream));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, st);
  dfree(ctx, dmax);
  if (n & 1) L->cur ^= 1;
  double last = 0.0;
  bool bad = false;
  for (int t = 0; t < n; ++t) {
    double d;
    memcpy(&d, &bits[t], 8);
    if (!(d == d)) bad = true;
    if (deltas) deltas[t] = d;
    last = d;
  }
  if (sweeps_done) *sweeps_done = n;
  if (last_delta) *last_delta = last;
  if (bad) return set_error(ctx, MSB_EZERO_DIAG, "non-finite update: zero diagonal in A_T");
  if (tol >= 0.0 && n >= max_sweeps && !(last <= tol)) return MSB_NOT_CONVERGED;
  return MSB_OK;
}

}  // extern "C"
