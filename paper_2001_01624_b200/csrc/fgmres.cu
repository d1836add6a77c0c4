// NEXT-1 — flexible GMRES with the multibasis cycle as right preconditioner
// (PAPER.md:287).  Same algorithm and stopping rule as
// oracle/fgmres.py, with classical Gram-Schmidt applied twice (CGS2: two fused passes
// of "all dots, then all updates" over the basis instead of j dependent MGS passes —
// mathematically the same Arnoldi basis; reading B6).  Each step: z_j = M^{-1} v_j (one
// Eq.-(8) cycle over the static levels), w = A z_j, CGS2, ||w||; the (j+1) x j
// Hessenberg matrix and its Givens rotations live on the host (m <= 64 scalars).
// Reductions are block partials summed in a fixed order: deterministic.
#include <algorithm>
#include <cmath>
#include <functional>
#include <vector>

#include "internal.cuh"

namespace msb {

constexpr int FG_T = 256;

__device__ __forceinline__ double fg_block_sum(double v) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double w = 0.0;
  if (threadIdx.x < 32) {
    w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  __syncthreads();
  return w;
}

// part[i * gridDim.x + block] = partial (V_i, w) over this block's cells, i < nv
__global__ void __launch_bounds__(FG_T) k_multidot(const double* __restrict__ V, int nv, int64_t N,
                                                   const double* __restrict__ w,
                                                   double* __restrict__ part) {
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < nv; ++i) {
    const double* __restrict__ vi = V + (size_t)i * N;
    double acc = 0.0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gs)
      acc += vi[c] * w[c];
    acc = fg_block_sum(acc);
    if (threadIdx.x == 0) part[(size_t)i * gridDim.x + blockIdx.x] = acc;
  }
}

// out[i] = sum over blocks of part[i][.], fixed order (one CTA per i)
__global__ void __launch_bounds__(FG_T) k_reduce_parts(const double* __restrict__ part, int nb,
                                                       double* __restrict__ out) {
  const double* p = part + (size_t)blockIdx.x * nb;
  double acc = 0.0;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) acc += p[t];
  acc = fg_block_sum(acc);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// w[c] += alpha * sum_i coef[i] V_i[c]   (coef on the device)
__global__ void __launch_bounds__(FG_T) k_multiaxpy(const double* __restrict__ V, int nv, int64_t N,
                                                    const double* __restrict__ coef, double alpha,
                                                    double* __restrict__ w) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double acc = 0.0;
  for (int i = 0; i < nv; ++i) acc += coef[i] * V[(size_t)i * N + c];
  w[c] += alpha * acc;
}

// Arnoldi column on the device: h_i = (0 + d1_i) + d2_i (the two CGS passes, in the order
// the host accumulated them before), h_{j+1} = sqrt(w.w)
__global__ void k_hcol(const double* __restrict__ d1, const double* __restrict__ d2,
                       const double* __restrict__ ww, int j, double* __restrict__ h) {
  const int i = threadIdx.x;
  if (i <= j) h[i] = (0.0 + d1[i]) + d2[i];
  if (i == 0) h[j + 1] = sqrt(*ww);
}

// v_{j+1} = w / h_{j+1} (as (1 / h) w), or 0 on breakdown (h = 0), h read on the device
__global__ void k_scale_by(const double* __restrict__ h, const double* __restrict__ w,
                           double* __restrict__ v, int64_t N) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const double hn = *h;
  v[c] = hn != 0.0 ? (1.0 / hn) * w[c] : 0.0;
}

// y = x - y  (r = b - A x with y = A x on entry)
__global__ void k_xmy(const double* __restrict__ x, double* __restrict__ y, int64_t N) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < N) y[c] = x[c] - y[c];
}

// y = a * x (y is write-only: a fresh Krylov slot may hold anything, NaN included)
__global__ void k_scale(double a, const double* x, double* y, int64_t N) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < N) y[c] = a * x[c];
}

}  // namespace msb

namespace msb {

// Flexible GMRES(m) on a device operator: ops.A (y = A x) and ops.M (z = M^{-1} v) over
// vectors of length N; db the device rhs, x host|dev in x0 / out x.
msb_status fgmres_core(msb_ctx ctx, int64_t N, const FgOps& ops, const double* db, double* x,
                       double tol, int32_t restart, int32_t max_iter, int32_t fixed_iters,
                       int32_t* iters_out, double* res_hist) {
  if (restart < 1 || restart > 64 || max_iter < 0 || fixed_iters < 0)
    return set_error(ctx, MSB_EINVAL, "fgmres: restart must be in [1, 64]");
  cudaStream_t st = ctx->stream;
  const int m = restart;
  // the Krylov workspace is released on every return path: the stream is drained first,
  // so no enqueued kernel still reads a freed buffer
  struct Workspace {
    msb_ctx ctx;
    double *V = nullptr, *Z = nullptr, *w = nullptr, *xd = nullptr, *part = nullptr,
           *dots = nullptr;
    ~Workspace() {
      cudaStreamSynchronize(ctx->stream);
      for (void* p : {(void*)V, (void*)Z, (void*)w, (void*)xd, (void*)part, (void*)dots})
        dfree(ctx, p);
    }
  } ws{ctx};
  double *&V = ws.V, *&Z = ws.Z, *&w = ws.w, *&xd = ws.xd, *&part = ws.part, *&dots = ws.dots;
  MSB_ALLOC(ctx, V, double, (size_t)(m + 1) * N);
  MSB_ALLOC(ctx, Z, double, (size_t)m * N);
  MSB_ALLOC(ctx, w, double, N);
  MSB_ALLOC(ctx, xd, double, N);
  const int nb = 4 * ctx->sm_count;
  MSB_ALLOC(ctx, part, double, (size_t)(m + 1) * nb);
  MSB_ALLOC(ctx, dots, double, 3 * (m + 2) + 1);  // pass-1 dots | pass-2 dots | H column | w.w
  double* dots2 = dots + (m + 2);
  double* hcol = dots + 2 * (m + 2);
  double* wwd = dots + 3 * (m + 2);
  double* hpin = static_cast<double*>(pinned_scratch(ctx, (m + 2) * sizeof(double)));
  if (!hpin) return set_error(ctx, MSB_ENOMEM, "pinned readback buffer");
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(xd, x, N * sizeof(double), cudaMemcpyDefault, st));
  const unsigned ge = grid_for(N, FG_T);
  msb_status rc = MSB_OK;
  // host-side reductions of device vectors
  std::vector<double> hd(m + 2);
  auto multidot = [&](const double* Vb, int nv, const double* wv) -> msb_status {
    k_multidot<<<nb, FG_T, 0, st>>>(Vb, nv, N, wv, part);
    MSB_LAUNCH_CHECK(ctx);
    k_reduce_parts<<<nv, FG_T, 0, st>>>(part, nb, dots);
    MSB_LAUNCH_CHECK(ctx);
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hd.data(), dots, nv * sizeof(double), cudaMemcpyDeviceToHost, st));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return MSB_OK;
  };
  auto nrm2 = [&](const double* v, double* out) -> msb_status {
    msb_status r2 = multidot(v, 1, v);
    if (r2) return r2;
    *out = std::sqrt(hd[0]);
    return MSB_OK;
  };
  // residual r = b - A x into V_0
  auto residual = [&](double* r) -> msb_status {
    msb_status r2 = ops.A(xd, r);
    if (r2) return r2;
    k_xmy<<<ge, FG_T, 0, st>>>(db, r, N);
    MSB_LAUNCH_CHECK(ctx);
    return MSB_OK;
  };
  double bnorm;
  if ((rc = nrm2(db, &bnorm))) return rc;
  const double scale = bnorm > 0.0 ? bnorm : 1.0;
  std::vector<double> res;
  int k = 0;
  bool converged = false;
  const int target = fixed_iters > 0 ? fixed_iters : max_iter;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
  while (true) {
    if ((rc = residual(V))) return rc;
    double beta;
    if ((rc = nrm2(V, &beta))) return rc;
    if (k == 0) res.push_back(beta / scale);
    if (fixed_iters <= 0 && beta / scale <= tol) {
      converged = true;
      break;
    }
    if (k >= target || beta == 0.0) break;
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    k_scale<<<ge, FG_T, 0, st>>>(1.0 / beta, V, V, N);  // V_0 = r / beta
    MSB_LAUNCH_CHECK(ctx);
    int jused = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = V + (size_t)j * N;
      double* zj = Z + (size_t)j * N;
      if ((rc = ops.M(vj, zj))) return rc;
      if ((rc = ops.A(zj, w))) return rc;
      // CGS2: h = V^T w; w -= V h; twice — all on the device, then ||w||, the Arnoldi
      // column and v_{j+1}; one host round trip per step reads the column for the rotations
      for (int pass = 0; pass < 2; ++pass) {
        double* dd = pass ? dots2 : dots;
        k_multidot<<<nb, FG_T, 0, st>>>(V, j + 1, N, w, part);
        MSB_LAUNCH_CHECK(ctx);
        k_reduce_parts<<<j + 1, FG_T, 0, st>>>(part, nb, dd);
        MSB_LAUNCH_CHECK(ctx);
        k_multiaxpy<<<ge, FG_T, 0, st>>>(V, j + 1, N, dd, -1.0, w);
        MSB_LAUNCH_CHECK(ctx);
      }
      k_multidot<<<nb, FG_T, 0, st>>>(w, 1, N, w, part);
      MSB_LAUNCH_CHECK(ctx);
      k_reduce_parts<<<1, FG_T, 0, st>>>(part, nb, wwd);
      MSB_LAUNCH_CHECK(ctx);
      k_hcol<<<1, 64, 0, st>>>(dots, dots2, wwd, j, hcol);
      MSB_LAUNCH_CHECK(ctx);
      k_scale_by<<<ge, FG_T, 0, st>>>(hcol + j + 1, w, V + (size_t)(j + 1) * N, N);
      MSB_LAUNCH_CHECK(ctx);
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hpin, hcol, (j + 2) * sizeof(double),
                                        cudaMemcpyDeviceToHost, st));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
      for (int i = 0; i <= j + 1; ++i) Hij(i, j) = hpin[i];
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double d = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = d != 0.0 ? Hij(j, j) / d : 1.0;
      sn[j] = d != 0.0 ? Hij(j + 1, j) / d : 0.0;
      Hij(j, j) = d;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++k;
      jused = j + 1;
      res.push_back(std::fabs(g[j + 1]) / scale);
      if (fixed_iters > 0) {
        if (k >= fixed_iters) break;
      } else if (std::fabs(g[j + 1]) / scale <= tol || k >= max_iter) {
        break;
      }
    }
    for (int i = jused - 1; i >= 0; --i) {
      double acc = g[i];
      for (int t = i + 1; t < jused; ++t) acc -= Hij(i, t) * y[t];
      y[i] = acc / Hij(i, i);
    }
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(dots, y.data(), jused * sizeof(double), cudaMemcpyHostToDevice, st));
    k_multiaxpy<<<ge, FG_T, 0, st>>>(Z, jused, N, dots, 1.0, xd);
    MSB_LAUNCH_CHECK(ctx);
    if (fixed_iters > 0 && k >= fixed_iters) break;
  }
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(x, xd, N * sizeof(double), cudaMemcpyDefault, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (res_hist)
    for (size_t t = 0; t < res.size(); ++t) res_hist[t] = res[t];
  if (iters_out) *iters_out = k;
  if (fixed_iters > 0) return MSB_OK;
  return converged ? MSB_OK : MSB_NOT_CONVERGED;
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_fgmres(msb_ctx ctx, msb_solver s, const double* b, double* x, double tol,
                                 int32_t restart, int32_t max_iter, int32_t fixed_iters,
                                 int32_t* iters_out, double* res_hist) {
  MSB_NVTX("msb_fgmres");
  if (!ctx || !s || !x) return set_error(ctx, MSB_EINVAL, "msb_fgmres: null");
  if (restart < 1 || restart > 64 || max_iter < 0 || fixed_iters < 0)
    return set_error(ctx, MSB_EINVAL, "msb_fgmres: restart must be in [1, 64]");
  if (s->levels.empty() && !(s->dyn && s->dyn_level && s->dyn_level->M > 0))
    return set_error(ctx, MSB_EINVAL, "msb_fgmres: solver has no stage to precondition with");
  msb_op op = s->op;
  const int64_t N = op->N;
  struct Staged {
    msb_ctx ctx;
    void* ob = nullptr;
    ~Staged() {
      cudaStreamSynchronize(ctx->stream);
      dfree(ctx, ob);
    }
  } sb{ctx};
  const double* db = b ? (const double*)stage_in(ctx, b, N * sizeof(double), &sb.ob) : op->q;
  if (!db) return set_error(ctx, MSB_ENOMEM, "rhs staging");
  {
    msb_status r0 = solver_smoother_setup(ctx, s);
    if (r0) return r0;
  }
  FgOps ops;
  ops.A = [&](const double* xv, double* yv) { return msb_op_apply(ctx, op, xv, yv); };
  ops.M = [&](const double* v, double* z) { return solver_precondition(ctx, s, v, z); };
  return fgmres_core(ctx, N, ops, db, x, tol, restart, max_iter, fixed_iters, iters_out, res_hist);
}
