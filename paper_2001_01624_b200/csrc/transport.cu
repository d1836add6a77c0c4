// Row a12 (auxiliary, config 4): face fluxes, explicit single-point-upstream
// transport of water saturation, and the upstream total mobility for the next
// pressure step (PAPER.md:41 sequential splitting, :101 single-point upstream;
// readings A17, A18).  Quadratic relative permeabilities:
//   λ_w = S^2/μ_w, λ_o = (1-S)^2/μ_o, λ_t = λ_w + λ_o, f_w = λ_w/λ_t.
// fw_max' is the largest forward-difference slope of f_w on the grid S = k/1000
// (the same rule in the oracle), so both sides pick the same sub-step count.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "internal.cuh"

namespace msb {

__device__ __host__ __forceinline__ double fw(double S, double muw, double muo) {
  double lw = S * S / muw, lo = (1.0 - S) * (1.0 - S) / muo;
  return lw / (lw + lo);
}

__device__ __forceinline__ double lam_t(double S, double muw, double muo) {
  return S * S / muw + (1.0 - S) * (1.0 - S) / muo;
}

struct FluxView {
  const double* Tx;
  const double* Ty;
  const double* Tz;
  int nx, ny, nz;
};

// outflow_i = Σ_{faces} max(F_out, 0) + q_i^-   (q^- = -min(q, 0)); reduce min φ/out.
__global__ void k_cfl(FluxView F, const double* __restrict__ p, const double* __restrict__ q,
                      const double* __restrict__ phi, double vol,
                      unsigned long long* __restrict__ minbits) {
  int64_t N = (int64_t)F.nx * F.ny * F.nz;
  int64_t sxy = (int64_t)F.nx * F.ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = INFINITY;
  if (c < N) {
    int i = (int)(c % F.nx), j = (int)((c / F.nx) % F.ny), k = (int)(c / sxy);
    double out = 0.0;
    double pc = p[c];
    if (i < F.nx - 1) out += fmax(F.Tx[c] * (pc - p[c + 1]), 0.0);
    if (i > 0) out += fmax(F.Tx[c - 1] * (pc - p[c - 1]), 0.0);
    if (j < F.ny - 1) out += fmax(F.Ty[c] * (pc - p[c + F.nx]), 0.0);
    if (j > 0) out += fmax(F.Ty[c - F.nx] * (pc - p[c - F.nx]), 0.0);
    if (k < F.nz - 1) out += fmax(F.Tz[c] * (pc - p[c + sxy]), 0.0);
    if (k > 0) out += fmax(F.Tz[c - sxy] * (pc - p[c - sxy]), 0.0);
    out += fmax(-q[c], 0.0);
    if (out > 0.0) v = phi[c] * vol / out;
  }
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMin(minbits, (unsigned long long)__double_as_longlong(v));
}

__global__ void k_transport_step(FluxView F, const double* __restrict__ p,
                                 const double* __restrict__ q, const double* __restrict__ phi,
                                 double vol, double muw, double muo, double h,
                                 const double* __restrict__ S, double* __restrict__ So) {
  int64_t N = (int64_t)F.nx * F.ny * F.nz;
  int64_t sxy = (int64_t)F.nx * F.ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % F.nx), j = (int)((c / F.nx) % F.ny), k = (int)(c / sxy);
  double pc = p[c], sc = S[c];
  double fc = fw(sc, muw, muo);
  double net = 0.0;
  // flux F = T (p_c - p_l) leaves c when positive
  auto face = [&](double T, int64_t l) {
    double Fl = T * (pc - p[l]);
    if (Fl > 0.0) net -= Fl * fc;
    else net -= Fl * fw(S[l], muw, muo);  // inflow: -F > 0 carries f_w(S_l)
  };
  if (k > 0) face(F.Tz[c - sxy], c - sxy);
  if (j > 0) face(F.Ty[c - F.nx], c - F.nx);
  if (i > 0) face(F.Tx[c - 1], c - 1);
  if (i < F.nx - 1) face(F.Tx[c], c + 1);
  if (j < F.ny - 1) face(F.Ty[c], c + F.nx);
  if (k < F.nz - 1) face(F.Tz[c], c + sxy);
  double qc = q[c];
  if (qc > 0.0) net += qc;           // injected water, f_w = 1
  else net += qc * fc;               // produced at f_w(S_c)
  So[c] = sc + h / (phi[c] * vol) * net;
}

// Face fluxes of the step, once per msb_transport_upwind call (p is fixed during the
// sub-steps): Fx[c] = Tx[c] (p_c - p_{c+1}) etc., cell-padded like T (0 past the last
// column / row / plane).  The sub-step kernel below reads them with the orientation
// sign instead of re-forming T (p_c - p_l) every sub-step; T (a - b) and T (b - a) are
// exact negatives, so the arithmetic is bit-for-bit that of k_transport_step.
__global__ void k_face_fluxes(FluxView F, Grid3 g, const double* __restrict__ p,
                              double* __restrict__ Fx, double* __restrict__ Fy,
                              double* __restrict__ Fz) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const double pc = p[c];
  Fx[c] = i < F.nx - 1 ? F.Tx[c] * (pc - p[c + 1]) : 0.0;
  Fy[c] = j < F.ny - 1 ? F.Ty[c] * (pc - p[c + F.nx]) : 0.0;
  Fz[c] = k < F.nz - 1 ? F.Tz[c] * (pc - p[c + g.nxy]) : 0.0;
}

// One explicit upwind sub-step from precomputed face fluxes (same order of terms as
// k_transport_step: -z, -y, -x, +x, +y, +z, then the source), 32-bit cell indexing.
__global__ void __launch_bounds__(256) k_transport_flux_step(
    Grid3 g, const double* __restrict__ Fx, const double* __restrict__ Fy,
    const double* __restrict__ Fz, const double* __restrict__ q, const double* __restrict__ phi,
    double vol, double muw, double muo, double h, const double* __restrict__ S,
    double* __restrict__ So) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const int nx = g.nx, sxy = g.nxy;
  const double sc = S[c];
  const double fc = fw(sc, muw, muo);
  double net = 0.0;
  auto face = [&](double Fl, int l) {  // Fl: flux leaving c through the face
    if (Fl > 0.0) net -= Fl * fc;
    else net -= Fl * fw(S[l], muw, muo);
  };
  if (k > 0) face(-Fz[c - sxy], c - sxy);
  if (j > 0) face(-Fy[c - nx], c - nx);
  if (i > 0) face(-Fx[c - 1], c - 1);
  if (i < g.nx - 1) face(Fx[c], c + 1);
  if (j < g.ny - 1) face(Fy[c], c + nx);
  if (k < g.nz - 1) face(Fz[c], c + sxy);
  const double qc = q[c];
  if (qc > 0.0) net += qc;
  else net += qc * fc;
  So[c] = sc + h / (phi[c] * vol) * net;
}

// Upstream total mobility per face (compact face layout); ties (F = 0) -> lower cell.
__global__ void k_upstream_mob(FluxView F, const double* __restrict__ p, const double* __restrict__ S,
                               double muw, double muo, double* __restrict__ mob) {
  int64_t N = (int64_t)F.nx * F.ny * F.nz;
  int64_t sxy = (int64_t)F.nx * F.ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int nx = F.nx, ny = F.ny, nz = F.nz;
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  int64_t nfx = (int64_t)(nx - 1) * ny * nz;
  int64_t nfy = (int64_t)nx * (ny - 1) * nz;
  double pc = p[c];
  if (i < nx - 1) {
    int64_t l = c + 1;
    double s = (pc - p[l] >= 0.0) ? S[c] : S[l];
    mob[i + (int64_t)(nx - 1) * (j + (int64_t)ny * k)] = lam_t(s, muw, muo);
  }
  if (j < ny - 1) {
    int64_t l = c + nx;
    double s = (pc - p[l] >= 0.0) ? S[c] : S[l];
    mob[nfx + i + (int64_t)nx * (j + (int64_t)(ny - 1) * k)] = lam_t(s, muw, muo);
  }
  if (k < nz - 1) {
    int64_t l = c + sxy;
    double s = (pc - p[l] >= 0.0) ? S[c] : S[l];
    mob[nfx + nfy + c] = lam_t(s, muw, muo);
  }
}

// Σ φ_i and Σ max(q_i, 0): per-CTA partials in a fixed order, then one CTA sums them
// in a fixed order (deterministic).
__global__ void __launch_bounds__(256) k_pv_parts(const double* __restrict__ phi,
                                                  const double* __restrict__ q, int64_t N,
                                                  double* __restrict__ part) {
  double a = 0.0, b = 0.0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N;
       c += (int64_t)gridDim.x * blockDim.x) {
    a += phi[c];
    b += fmax(q[c], 0.0);
  }
  __shared__ double sa[8], sb[8];
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = a;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int w = 0; w < 8; ++w) {
      ta += sa[w];
      tb += sb[w];
    }
    part[2 * blockIdx.x] = ta;
    part[2 * blockIdx.x + 1] = tb;
  }
}

__global__ void k_pv_final(const double* __restrict__ part, int n, double vol, double pv,
                           double* __restrict__ dt) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int t = 0; t < n; ++t) {
    a += part[2 * t];
    b += part[2 * t + 1];
  }
  *dt = b > 0.0 ? pv * (a * vol) / b : 0.0;
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_upstream_mobility(msb_ctx ctx, msb_op op, const double* p,
                                            const double* S, double mu_w, double mu_o,
                                            double* mob_out) {
  if (!ctx || !op || !mob_out) return set_error(ctx, MSB_EINVAL, "msb_upstream_mobility: null");
  if (!(mu_w > 0) || !(mu_o > 0)) return set_error(ctx, MSB_EINVAL, "msb_upstream_mobility: bad viscosity");
  const int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  // NULL p (no previous flux) and NULL S (dry reservoir) read as zero vectors
  double* z = nullptr;
  if (!p || !S) {
    z = dalloc_n<double>(ctx, N);
    if (!z) return set_error(ctx, MSB_ENOMEM, "mobility scratch");
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(z, 0, N * sizeof(double), st));
  }
  void *op_, *os_;
  const double* dp = p ? (const double*)stage_in(ctx, p, N * sizeof(double), &op_) : z;
  if (!p) op_ = nullptr;
  const double* ds = S ? (const double*)stage_in(ctx, S, N * sizeof(double), &os_) : z;
  if (!S) os_ = nullptr;
  const int64_t nf = (int64_t)(op->nx - 1) * op->ny * op->nz +
                     (int64_t)op->nx * (op->ny - 1) * op->nz + (int64_t)op->nx * op->ny * (op->nz - 1);
  const bool dev = is_device_ptr(mob_out);
  double* d = dev ? mob_out : dalloc_n<double>(ctx, nf + 1);
  msb_status rc = MSB_OK;
  if (!dp || !ds || !d) rc = set_error(ctx, MSB_ENOMEM, "mobility staging");
  if (!rc) {
    FluxView F{op->Tx, op->Ty, op->Tz, op->nx, op->ny, op->nz};
    k_upstream_mob<<<grid_for(N, 256), 256, 0, st>>>(F, dp, ds, mu_w, mu_o, d);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) rc = set_error(ctx, MSB_ECUDA, "k_upstream_mob launch");
  }
  if (!rc && !dev && copy_out(ctx, mob_out, d, nf * sizeof(double)) != cudaSuccess)
    rc = set_error(ctx, MSB_ECUDA, "mobility copy-out");
  cudaStreamSynchronize(st);
  if (!dev) dfree(ctx, d);
  dfree(ctx, z);
  dfree(ctx, op_);
  dfree(ctx, os_);
  return rc;
}

extern "C" msb_status msb_transport_step_size(msb_ctx ctx, msb_op op, const double* phi,
                                              double pv_per_step, double* dt_out) {
  if (!ctx || !op || !phi || !dt_out || !(pv_per_step >= 0))
    return set_error(ctx, MSB_EINVAL, "msb_transport_step_size: args");
  const int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  void* o = nullptr;
  const double* dphi = (const double*)stage_in(ctx, phi, N * sizeof(double), &o);
  const int nb = 2 * ctx->sm_count;
  double* part = dalloc_n<double>(ctx, 2 * (size_t)nb + 1);
  msb_status rc = MSB_OK;
  if (!dphi || !part) rc = set_error(ctx, MSB_ENOMEM, "step-size scratch");
  double h = 0.0;
  if (!rc) {
    k_pv_parts<<<nb, 256, 0, st>>>(dphi, op->q, N, part);
    k_pv_final<<<1, 32, 0, st>>>(part, nb, op->dx * op->dy * op->dz, pv_per_step, part + 2 * nb);
    count_launch();
    count_launch();
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&h, part + 2 * nb, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = set_error(ctx, MSB_ECUDA, "step-size reduction");
  }
  cudaStreamSynchronize(st);
  dfree(ctx, part);
  dfree(ctx, o);
  if (!rc) *dt_out = h;
  return rc;
}

extern "C" msb_status msb_transport_upwind(msb_ctx ctx, msb_op op, const double* p, double* S,
                                           const double* phi, double mu_w, double mu_o, double dt,
                                           double* mob_out, int32_t* substeps_out) {
  MSB_NVTX("msb_transport_upwind");
  if (!ctx || !op || !p || !S || !phi) return set_error(ctx, MSB_EINVAL, "transport: null");
  if (!(mu_w > 0) || !(mu_o > 0) || !(dt >= 0)) return set_error(ctx, MSB_EINVAL, "transport: bad args");
  int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  FluxView F{op->Tx, op->Ty, op->Tz, op->nx, op->ny, op->nz};
  double vol = op->dx * op->dy * op->dz;
  // fw_max' on the uniform grid k/1000 (forward differences), as in the oracle
  double fmaxd = 0.0;
  for (int t = 0; t < 1000; ++t) {
    double a = fw(t / 1000.0, mu_w, mu_o), b = fw((t + 1) / 1000.0, mu_w, mu_o);
    fmaxd = std::max(fmaxd, (b - a) * 1000.0);
  }
  unsigned long long* mb = dalloc_n<unsigned long long>(ctx, 1);
  double inf = INFINITY;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(mb, &inf, 8, cudaMemcpyHostToDevice, st));
  k_cfl<<<grid_for(N, 256), 256, 0, st>>>(F, p, op->q, phi, vol, mb);
  MSB_LAUNCH_CHECK(ctx);
  unsigned long long hb = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hb, mb, 8, cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  double mn;
  memcpy(&mn, &hb, 8);
  int nsub = 1;
  if (std::isfinite(mn) && fmaxd > 0.0) {
    double dt_cfl = 0.5 * mn / fmaxd;
    nsub = std::max(1, (int)std::ceil(dt / dt_cfl));
  }
  double h = dt / nsub;
  double* tmp = dalloc_n<double>(ctx, 4 * N);  // S ping-pong + the three face-flux planes
  if (!tmp) return set_error(ctx, MSB_ENOMEM, "transport scratch");
  double* a = S;
  double* b = tmp;
  if (N > INT32_MAX / 2) {  // the per-face kernel (64-bit indices) beyond int32 cell ids
    for (int t = 0; t < nsub; ++t) {
      k_transport_step<<<grid_for(N, 256), 256, 0, st>>>(F, p, op->q, phi, vol, mu_w, mu_o, h, a, b);
      MSB_LAUNCH_CHECK(ctx);
      std::swap(a, b);
    }
  } else {
    const Grid3 g = make_grid3(op->nx, op->ny, op->nz);
    double* Fx = tmp + N;
    double* Fy = tmp + 2 * N;
    double* Fz = tmp + 3 * N;
    k_face_fluxes<<<grid_for(N, 256), 256, 0, st>>>(F, g, p, Fx, Fy, Fz);
    MSB_LAUNCH_CHECK(ctx);
    for (int t = 0; t < nsub; ++t) {
      k_transport_flux_step<<<grid_for(N, 256), 256, 0, st>>>(g, Fx, Fy, Fz, op->q, phi, vol, mu_w,
                                                               mu_o, h, a, b);
      MSB_LAUNCH_CHECK(ctx);
      std::swap(a, b);
    }
  }
  if (a != S) MSB_CUDA_TRY(ctx, cudaMemcpyAsync(S, a, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (mob_out) {
    int64_t nf = (int64_t)(op->nx - 1) * op->ny * op->nz + (int64_t)op->nx * (op->ny - 1) * op->nz +
                 (int64_t)op->nx * op->ny * (op->nz - 1);
    bool dev = is_device_ptr(mob_out);
    double* d = dev ? mob_out : dalloc_n<double>(ctx, nf);
    k_upstream_mob<<<grid_for(N, 256), 256, 0, st>>>(F, p, S, mu_w, mu_o, d);
    MSB_LAUNCH_CHECK(ctx);
    if (!dev) {
      MSB_CUDA_TRY(ctx, copy_out(ctx, mob_out, d, nf * sizeof(double)));
      dfree(ctx, d);
    }
  }
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  dfree(ctx, tmp);
  dfree(ctx, mb);
  if (substeps_out) *substeps_out = nsub;
  return MSB_OK;
}
