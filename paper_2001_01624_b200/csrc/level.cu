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
  dfree(ctx, L->amask);
  dfree(ctx, L->col);
  dfree(ctx, L->nbs);
  dfree(ctx, L->csc_ptr);
  dfree(ctx, L->csc_pos);
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
  MSB_NVTX("msb_level_create_cartesian");
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
  L->unity = false;  // arbitrary values: the coarse assembly accumulates every entry
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

}  // extern "C"
