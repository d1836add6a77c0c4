// Row a1 — two-point flux transmissibilities (G1), rhs, face-open mask, A x.
//
// PAPER.md:101 (two-point flux, single-point upstream mobility); SPEC.md:159-167:
//   t = K * A_face / (Δ/2),  T_f = (1/t_i + 1/t_l)^{-1} * mult_f * mob_f.
// Storage: cell-padded face arrays Tx[c] (face c|c+1), Ty[c] (c|c+nx), Tz[c]
// (c|c+nx*ny), zero where the face does not exist; 24 B/cell, read with
// coalesced fp64 loads by every stencil kernel.
#include <climits>

#include "internal.cuh"

namespace msb {

__device__ __forceinline__ double half_t(double K, double area, double d) {
  return K * area / (d / 2.0);
}

// One thread per cell writes the three faces on its +x, +y, +z sides.
__global__ void k_tpfa(const double* __restrict__ K, const double* __restrict__ mult,
                       const double* __restrict__ mob, int nx, int ny, int nz, double dx,
                       double dy, double dz, double* __restrict__ Tx, double* __restrict__ Ty,
                       double* __restrict__ Tz, double* __restrict__ Tb,
                       uint8_t* __restrict__ open, int* __restrict__ bad) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx);
  int j = (int)((c / nx) % ny);
  int k = (int)(c / ((int64_t)nx * ny));
  const double* Kx = K;
  const double* Ky = K + N;
  const double* Kz = K + 2 * N;
  if (!(Kx[c] > 0.0) || !(Ky[c] > 0.0) || !(Kz[c] > 0.0)) atomicExch(bad, 1);
  int64_t nfx = (int64_t)(nx - 1) * ny * nz;
  int64_t nfy = (int64_t)nx * (ny - 1) * nz;
  uint8_t o = 0;
  double tx = 0.0, ty = 0.0, tz = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
  if (i < nx - 1) {
    int64_t f = i + (int64_t)(nx - 1) * (j + (int64_t)ny * k);
    double tl = half_t(Kx[c], dy * dz, dx), tr = half_t(Kx[c + 1], dy * dz, dx);
    double m = mult ? mult[f] : 1.0;
    double lam = mob ? mob[f] : 1.0;
    bx = 1.0 / (1.0 / tl + 1.0 / tr) * m;
    tx = 1.0 / (1.0 / tl + 1.0 / tr) * m * lam;
    if (m == 1.0) o |= 1;
  }
  if (j < ny - 1) {
    int64_t f = i + (int64_t)nx * (j + (int64_t)(ny - 1) * k);
    double tl = half_t(Ky[c], dx * dz, dy), tr = half_t(Ky[c + nx], dx * dz, dy);
    double m = mult ? mult[nfx + f] : 1.0;
    double lam = mob ? mob[nfx + f] : 1.0;
    by = 1.0 / (1.0 / tl + 1.0 / tr) * m;
    ty = 1.0 / (1.0 / tl + 1.0 / tr) * m * lam;
    if (m == 1.0) o |= 2;
  }
  if (k < nz - 1) {
    int64_t f = c;
    int64_t s = (int64_t)nx * ny;
    double tl = half_t(Kz[c], dx * dy, dz), tr = half_t(Kz[c + s], dx * dy, dz);
    double m = mult ? mult[nfx + nfy + f] : 1.0;
    double lam = mob ? mob[nfx + nfy + f] : 1.0;
    bz = 1.0 / (1.0 / tl + 1.0 / tr) * m;
    tz = 1.0 / (1.0 / tl + 1.0 / tr) * m * lam;
    if (m == 1.0) o |= 4;
  }
  Tx[c] = tx;
  Ty[c] = ty;
  Tz[c] = tz;
  Tb[c] = bx;
  Tb[N + c] = by;
  Tb[2 * N + c] = bz;
  open[c] = o;
}

// T = Tb * mob (compact face layout) — config-4 mobility refresh.
__global__ void k_apply_mob(const double* __restrict__ Tb, const double* __restrict__ mob, int nx,
                            int ny, int nz, double* __restrict__ Tx, double* __restrict__ Ty,
                            double* __restrict__ Tz) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx);
  int j = (int)((c / nx) % ny);
  int k = (int)(c / ((int64_t)nx * ny));
  int64_t nfx = (int64_t)(nx - 1) * ny * nz;
  int64_t nfy = (int64_t)nx * (ny - 1) * nz;
  Tx[c] = (i < nx - 1) ? Tb[c] * mob[i + (int64_t)(nx - 1) * (j + (int64_t)ny * k)] : 0.0;
  Ty[c] = (j < ny - 1) ? Tb[N + c] * mob[nfx + i + (int64_t)nx * (j + (int64_t)(ny - 1) * k)] : 0.0;
  Tz[c] = (k < nz - 1) ? Tb[2 * N + c] * mob[nfx + nfy + c] : 0.0;
}

__global__ void k_sources(const msb_source* __restrict__ src, int n, double* __restrict__ q,
                          int64_t N, int* __restrict__ bad) {
  // sequential over sources: deterministic sum order for repeated cells
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int s = 0; s < n; ++s) {
    int c = src[s].cell;
    if (c < 0 || c >= N) {
      *bad = 1;
      continue;
    }
    q[c] += src[s].rate;
  }
}

// Compact face export: T (x|y|z compact faces) from cell-padded arrays.
__global__ void k_export_T(const double* __restrict__ Tx, const double* __restrict__ Ty,
                           const double* __restrict__ Tz, int nx, int ny, int nz,
                           double* __restrict__ out) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx);
  int j = (int)((c / nx) % ny);
  int k = (int)(c / ((int64_t)nx * ny));
  int64_t nfx = (int64_t)(nx - 1) * ny * nz;
  int64_t nfy = (int64_t)nx * (ny - 1) * nz;
  if (i < nx - 1) out[i + (int64_t)(nx - 1) * (j + (int64_t)ny * k)] = Tx[c];
  if (j < ny - 1) out[nfx + i + (int64_t)nx * (j + (int64_t)(ny - 1) * k)] = Ty[c];
  if (k < nz - 1) out[nfx + nfy + c] = Tz[c];
}

// y = A x with A = A_T + A_T[0,0] e0 e0^T.
__global__ void k_apply_A(const double* __restrict__ Tx, const double* __restrict__ Ty,
                          const double* __restrict__ Tz, int nx, int ny, int nz,
                          const double* __restrict__ x, double* __restrict__ y) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int64_t sxy = (int64_t)nx * ny;
  int i = (int)(c % nx);
  int j = (int)((c / nx) % ny);
  int k = (int)(c / sxy);
  double xc = x[c];
  double tzm = k > 0 ? Tz[c - sxy] : 0.0, tym = j > 0 ? Ty[c - nx] : 0.0,
         txm = i > 0 ? Tx[c - 1] : 0.0;
  double txp = Tx[c], typ = Ty[c], tzp = Tz[c];
  double D = txp + txm + typ + tym + tzp + tzm;
  double off = 0.0;
  if (k > 0) off += tzm * x[c - sxy];
  if (j > 0) off += tym * x[c - nx];
  if (i > 0) off += txm * x[c - 1];
  if (i < nx - 1) off += txp * x[c + 1];
  if (j < ny - 1) off += typ * x[c + nx];
  if (k < nz - 1) off += tzp * x[c + sxy];
  double dA = (c == 0) ? 2.0 * D : D;
  y[c] = dA * xc - off;
}

}  // namespace msb

using namespace msb;

extern "C" {

msb_status msb_build_tpfa(msb_ctx ctx, const msb_grid* g, const double* K, const double* mult,
                          const double* mob, const msb_source* src, int32_t n_src, msb_op* out) {
  MSB_NVTX("msb_build_tpfa");
  if (!ctx || !g || !K || !out || n_src < 0 || (n_src > 0 && !src))
    return set_error(ctx, MSB_EINVAL, "msb_build_tpfa: null argument");
  if (g->nx < 1 || g->ny < 1 || g->nz < 1 || !(g->dx > 0) || !(g->dy > 0) || !(g->dz > 0))
    return set_error(ctx, MSB_EINVAL, "msb_build_tpfa: bad grid");
  *out = nullptr;
  int64_t N = (int64_t)g->nx * g->ny * g->nz;
  // cells are indexed with int32 on the device (config 5: 10^7), and the
  // 8-slot planes of P with size_t: 3N (the T block) must stay addressable as int32 offsets
  if (3 * N >= (int64_t)INT32_MAX)
    return set_error(ctx, MSB_EDIM, "msb_build_tpfa: %lld cells exceed the int32 cell indexing",
                     (long long)N);
  int64_t nf = (int64_t)(g->nx - 1) * g->ny * g->nz + (int64_t)g->nx * (g->ny - 1) * g->nz +
               (int64_t)g->nx * g->ny * (g->nz - 1);
  msb_op op = new msb_op_s();
  op->ctx = ctx;
  op->nx = g->nx; op->ny = g->ny; op->nz = g->nz; op->N = N;
  op->dx = g->dx; op->dy = g->dy; op->dz = g->dz;
  // one 3N block: Tx | Ty | Tz, so a kernel can stage all three with one 4D TMA box
  MSB_ALLOC(ctx, op->Tx, double, 3 * N);
  op->Ty = op->Tx + N;
  op->Tz = op->Tx + 2 * N;
  MSB_ALLOC(ctx, op->Tb, double, 3 * N);
  MSB_ALLOC(ctx, op->q, double, N);
  MSB_ALLOC(ctx, op->open, uint8_t, N);
  void *oK = nullptr, *oM = nullptr, *oL = nullptr;
  const double* dK = (const double*)stage_in(ctx, K, 3 * N * sizeof(double), &oK);
  const double* dM = mult ? (const double*)stage_in(ctx, mult, nf * sizeof(double), &oM) : nullptr;
  const double* dL = mob ? (const double*)stage_in(ctx, mob, nf * sizeof(double), &oL) : nullptr;
  if (!dK || (mult && !dM) || (mob && !dL)) return set_error(ctx, MSB_ENOMEM, "tpfa staging");
  int* bad = dalloc_n<int>(ctx, 2);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, 2 * sizeof(int), ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(op->q, 0, N * sizeof(double), ctx->stream));
  k_tpfa<<<grid_for(N, 256), 256, 0, ctx->stream>>>(dK, dM, dL, g->nx, g->ny, g->nz, g->dx, g->dy,
                                                    g->dz, op->Tx, op->Ty, op->Tz, op->Tb,
                                                    op->open, bad);
  MSB_LAUNCH_CHECK(ctx);
  if (n_src > 0) {
    msb_source* dsrc = dalloc_n<msb_source>(ctx, n_src);
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(dsrc, src, n_src * sizeof(msb_source), cudaMemcpyHostToDevice,
                                      ctx->stream));
    k_sources<<<1, 1, 0, ctx->stream>>>(dsrc, n_src, op->q, N, bad + 1);
    MSB_LAUNCH_CHECK(ctx);
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    dfree(ctx, dsrc);
  }
  int hbad[2] = {0, 0};
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, bad);
  if (oK) dfree(ctx, oK);
  if (oM) dfree(ctx, oM);
  if (oL) dfree(ctx, oL);

  if (hbad[0]) {
    msb_op_destroy(op);
    return set_error(ctx, MSB_EINVAL, "nonpositive permeability (SPEC.md:163)");
  }
  if (hbad[1]) {
    msb_op_destroy(op);
    return set_error(ctx, MSB_EINVAL, "source cell out of range");
  }
  *out = op;
  return MSB_OK;
}

msb_status msb_op_set_mobility(msb_ctx ctx, msb_op op, const double* mob) {
  MSB_NVTX("msb_op_set_mobility");
  if (!ctx || !op || !mob) return set_error(ctx, MSB_EINVAL, "msb_op_set_mobility: null");
  op->tmax_valid = false;  // T changes below
  int64_t nf = (int64_t)(op->nx - 1) * op->ny * op->nz + (int64_t)op->nx * (op->ny - 1) * op->nz +
               (int64_t)op->nx * op->ny * (op->nz - 1);
  void* o = nullptr;
  const double* d = (const double*)stage_in(ctx, mob, nf * sizeof(double), &o);
  if (!d) return set_error(ctx, MSB_ENOMEM, "mobility staging");
  k_apply_mob<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(op->Tb, d, op->nx, op->ny, op->nz,
                                                             op->Tx, op->Ty, op->Tz);
  MSB_LAUNCH_CHECK(ctx);
  if (o) {
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    dfree(ctx, o);
  }
  return MSB_OK;
}

msb_status msb_op_export(msb_ctx ctx, msb_op op, double* T_faces, double* q) {
  if (!ctx || !op) return set_error(ctx, MSB_EINVAL, "msb_op_export: null");
  if (T_faces) {
    int64_t nf = (int64_t)(op->nx - 1) * op->ny * op->nz +
                 (int64_t)op->nx * (op->ny - 1) * op->nz + (int64_t)op->nx * op->ny * (op->nz - 1);
    double* tmp = dalloc_n<double>(ctx, nf);
    k_export_T<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(op->Tx, op->Ty, op->Tz, op->nx,
                                                              op->ny, op->nz, tmp);
    MSB_LAUNCH_CHECK(ctx);
    MSB_CUDA_TRY(ctx, copy_out(ctx, T_faces, tmp, nf * sizeof(double)));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    dfree(ctx, tmp);
  }
  if (q) MSB_CUDA_TRY(ctx, copy_out(ctx, q, op->q, op->N * sizeof(double)));
  return sync(ctx);
}

msb_status msb_op_apply(msb_ctx ctx, msb_op op, const double* x, double* y) {
  if (!ctx || !op || !x || !y) return set_error(ctx, MSB_EINVAL, "msb_op_apply: null");
  k_apply_A<<<grid_for(op->N, 256), 256, 0, ctx->stream>>>(op->Tx, op->Ty, op->Tz, op->nx, op->ny,
                                                           op->nz, x, y);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

msb_status msb_op_destroy(msb_op op) {
  if (!op) return MSB_EINVAL;
  msb_ctx ctx = op->ctx;
  dfree(ctx, op->Tx);  // Ty, Tz live in the same block
  dfree(ctx, op->tmax);
  dfree(ctx, op->Tb);
  dfree(ctx, op->q);
  dfree(ctx, op->open);
  delete op;
  return MSB_OK;
}

}  // extern "C"
