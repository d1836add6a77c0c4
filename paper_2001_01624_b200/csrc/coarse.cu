// Rows a4 (Galerkin A_c = P^T A P, G6) and a5 (coarse factor + solve, G7).
//
// RAP: A = Σ_f T_f (e_i - e_l)(e_i - e_l)^T + A^T_00 e_0 e_0^T, so
//   A_c = Σ_f T_f g_f g_f^T + A^T_00 (P_0.)^T P_0.,   g_f = (P_i. - P_l.)^T,
// one thread per cell (its +x/+y/+z faces), g over the union of the two rows'
// columns (<= 2W entries), fp64 atomics into the dense row-major A_c.
//
// Factor: SPD A_c (Galerkin of the SPD gauged A) -> blocked
// right-looking Cholesky (LU without pivoting of an SPD matrix; PAPER.md:410
// "dense matrix inverted by direct Gaussian elimination"), pivot test
// d_jj <= 1e-14 max|A_c| -> MSB_ESINGULAR.  The explicit inverse
// X = L^-T L^-1 is formed once, so every coarse solve in the cycle is a single
// bandwidth-bound GEMV (M^2 doubles) instead of two latency-bound triangular solves.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace msb {

constexpr int NB = 32;  // panel width

// ---------------------------------------------------------------- RAP
__device__ __forceinline__ int row_entries(const msb_level_s& L, const double* __restrict__ P,
                                           int64_t c, int* cols, double* vals) {
  int n = 0;
  if (L.kind == 0) {
    int i = (int)(c % L.nx), j = (int)((c / L.nx) % L.ny), k = (int)(c / ((int64_t)L.nx * L.ny));
    const int32_t* tx = L.tab + 2 * i;
    const int32_t* ty = L.tab + 2 * (L.nx + j);
    const int32_t* tz = L.tab + 2 * (L.nx + L.ny + k);
    for (int s = 0; s < 8; ++s) {
      int jx = tx[s & 1], jy = ty[(s >> 1) & 1], jz = tz[s >> 2];
      if (jx < 0 || jy < 0 || jz < 0) continue;
      cols[n] = jx + L.nb[0] * (jy + L.nb[1] * jz);
      vals[n] = P[(int64_t)s * L.N + c];
      ++n;
    }
  } else {
    for (int s = 0; s < L.W; ++s) {
      int jc = L.col[(int64_t)s * L.N + c];
      if (jc < 0) continue;
      cols[n] = jc;
      vals[n] = P[(int64_t)s * L.N + c];
      ++n;
    }
  }
  return n;
}

constexpr int RMAX = 32;

__global__ void k_rap(const msb_level_s L, const double* __restrict__ P, const double* __restrict__ Tx,
                      const double* __restrict__ Ty, const double* __restrict__ Tz,
                      double* __restrict__ Ac) {
  int64_t N = L.N;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int M = L.M;
  int64_t sxy = (int64_t)L.nx * L.ny;
  int i = (int)(c % L.nx), j = (int)((c / L.nx) % L.ny), k = (int)(c / sxy);
  int cc[RMAX];
  double cv[RMAX];
  int nc = row_entries(L, P, c, cc, cv);
  double Tf[3] = {i < L.nx - 1 ? Tx[c] : 0.0, j < L.ny - 1 ? Ty[c] : 0.0,
                  k < L.nz - 1 ? Tz[c] : 0.0};
  int64_t nbr[3] = {c + 1, c + L.nx, c + sxy};
  for (int d = 0; d < 3; ++d) {
    double T = Tf[d];
    if (!(T != 0.0)) continue;
    int gc[2 * RMAX];
    double gv[2 * RMAX];
    int ng = nc;
    for (int t = 0; t < nc; ++t) {
      gc[t] = cc[t];
      gv[t] = cv[t];
    }
    int lc[RMAX];
    double lv[RMAX];
    int nl = row_entries(L, P, nbr[d], lc, lv);
    for (int t = 0; t < nl; ++t) {
      int u = 0;
      while (u < ng && gc[u] != lc[t]) ++u;
      if (u < ng) {
        gv[u] -= lv[t];
      } else {
        gc[ng] = lc[t];
        gv[ng] = -lv[t];
        ++ng;
      }
    }
    for (int a = 0; a < ng; ++a) {
      if (gv[a] == 0.0) continue;
      double ta = T * gv[a];
      for (int b = 0; b < ng; ++b) {
        if (gv[b] == 0.0) continue;
        atomicAdd(Ac + (int64_t)gc[a] * M + gc[b], ta * gv[b]);
      }
    }
  }
  if (c == 0) {  // gauge: A_00 doubled adds A^T_00 (P_0.)^T P_0.
    double d0 = Tf[0] + 0.0 + Tf[1] + 0.0 + Tf[2] + 0.0;
    for (int a = 0; a < nc; ++a)
      for (int b = 0; b < nc; ++b) atomicAdd(Ac + (int64_t)cc[a] * M + cc[b], d0 * cv[a] * cv[b]);
  }
}

// ---------------------------------------------------------------- max |A|
__global__ void k_absmax(const double* __restrict__ A, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------------------- Cholesky pieces
// Unblocked Cholesky of the kb x kb diagonal block at (k, k), in shared memory.
__global__ void k_potrf_diag(double* __restrict__ A, int M, int k, int kb, const unsigned long long* amax_bits,
                             int* __restrict__ singular) {
  __shared__ double a[NB][NB + 1];
  int t = threadIdx.x;  // NB*NB threads
  int r = t / NB, c = t % NB;
  if (r < kb && c < kb) a[r][c] = A[(int64_t)(k + r) * M + k + c];
  __syncthreads();
  double amax = __longlong_as_double((long long)*amax_bits);
  for (int j = 0; j < kb; ++j) {
    if (t == 0) {
      double d = a[j][j];
      if (!(d > 1e-14 * amax)) {
        atomicExch(singular, 1);
        d = 1.0;
      }
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    if (c == j && r > j && r < kb) a[r][j] /= a[j][j];
    __syncthreads();
    if (r > j && c > j && r < kb && c <= r) a[r][c] -= a[r][j] * a[c][j];
    __syncthreads();
  }
  if (r < kb && c < kb) A[(int64_t)(k + r) * M + k + c] = (c <= r) ? a[r][c] : 0.0;
}

// L21 = A21 L11^{-T}: one warp per row i in [k+kb, M).
__global__ void k_trsm_panel(double* __restrict__ A, int M, int k, int kb) {
  __shared__ double l[NB][NB + 1];
  for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
    int r = t / NB, c = t % NB;
    l[r][c] = (r < kb && c < kb) ? A[(int64_t)(k + r) * M + k + c] : 0.0;
  }
  __syncthreads();
  int lane = threadIdx.x & 31;
  int64_t row = (int64_t)k + kb + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= M) return;
  double* a = A + row * M + k;
  double v = lane < kb ? a[lane] : 0.0;
  for (int j = 0; j < kb; ++j) {
    double xj = __shfl_sync(0xffffffffu, v / l[j][j], j);
    if (lane == j) v = xj;
    if (lane > j) v -= xj * l[lane][j];
  }
  if (lane < kb) a[lane] = v;
}

// C(m x n) -= op(A)(m x kk) * op(B)(kk x n); kk <= NB.  64x64 tiles, 256 threads.
// lower_only: skip tiles strictly above the diagonal (tile row < tile col) — SYRK.
__global__ void __launch_bounds__(256) k_gemm_sub(double* __restrict__ C, int64_t ldc,
                                                  const double* __restrict__ A, int64_t lda,
                                                  int transA, const double* __restrict__ B,
                                                  int64_t ldb, int transB, int m, int n, int kk,
                                                  int lower_only) {
  int ti = blockIdx.y, tj = blockIdx.x;
  if (lower_only && ti < tj) return;
  __shared__ double As[NB][64 + 1];  // [t][i]
  __shared__ double Bs[NB][64 + 1];  // [t][j]
  int i0 = ti * 64, j0 = tj * 64;
  for (int e = threadIdx.x; e < NB * 64; e += 256) {
    int t = e / 64, q = e % 64;
    double va = 0.0, vb = 0.0;
    if (t < kk && i0 + q < m) va = transA ? A[(int64_t)t * lda + i0 + q] : A[(int64_t)(i0 + q) * lda + t];
    if (t < kk && j0 + q < n) vb = transB ? B[(int64_t)(j0 + q) * ldb + t] : B[(int64_t)t * ldb + j0 + q];
    As[t][q] = va;
    Bs[t][q] = vb;
  }
  __syncthreads();
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int t = 0; t < kk; ++t) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = As[t][ty + 16 * u];
      b[u] = Bs[t][tx + 16 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] += a[u] * b[v];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < m && j < n) C[(int64_t)i * ldc + j] -= acc[u][v];
    }
}

// Solve L_kk X = B (lower, forward) or L_kk^T X = B (backward) for rows k..k+kb of
// the M x n right-hand side X (row-major, in place); one thread per column.
__global__ void k_trsm_diag_rhs(const double* __restrict__ Lm, int M, int k, int kb,
                                double* __restrict__ X, int n, int upper) {
  __shared__ double l[NB][NB + 1];
  for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
    int r = t / NB, c = t % NB;
    l[r][c] = (r < kb && c < kb) ? Lm[(int64_t)(k + r) * M + k + c] : 0.0;
  }
  __syncthreads();
  int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double x[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) x[r] = r < kb ? X[(int64_t)(k + r) * n + col] : 0.0;
  if (!upper) {
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (r < kb) {
        double s = x[r];
        for (int t = 0; t < r; ++t) s -= l[r][t] * x[t];
        x[r] = s / l[r][r];
      }
    }
  } else {
#pragma unroll
    for (int rr = NB - 1; rr >= 0; --rr) {
      if (rr < kb) {
        double s = x[rr];
        for (int t = rr + 1; t < kb; ++t) s -= l[t][rr] * x[t];
        x[rr] = s / l[rr][rr];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NB; ++r)
    if (r < kb) X[(int64_t)(k + r) * n + col] = x[r];
}

__global__ void k_identity(double* __restrict__ X, int M) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * M) return;
  X[e] = (e / M == e % M) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- GEMV solve
// xc = X rc, one CTA per row: 256 threads each issue all of their (<= 8 at M <= 4096)
// 16-byte loads of the row at once, so a row costs one memory round trip and ~8 rows
// per SM are in flight; fixed-order per-thread sums + shuffle/smem tree: deterministic.
// The done flag is read at entry and tested before the store.
template <bool kStream>
__global__ void __launch_bounds__(256) k_gemv(const double* __restrict__ X, int M,
                                              const double* __restrict__ rc,
                                              double* __restrict__ xc, const int* done) {
  const bool skip = done && *(volatile const int*)done;
  const int64_t row = blockIdx.x;
  const double* a = X + row * M;
  double s = 0.0;
  if ((M & 1) == 0) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* r2 = reinterpret_cast<const double2*>(rc);
    const int h = M >> 1;
    for (int t0 = threadIdx.x; t0 < h; t0 += 8 * 256) {
      double2 av[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + 256 * u;
        av[u] = t < h ? (kStream ? __ldcs(a2 + t) : a2[t]) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + 256 * u;
        const double2 b = t < h ? r2[t] : make_double2(0.0, 0.0);
        s += av[u].x * b.x + av[u].y * b.y;
      }
    }
  } else {
    for (int t = threadIdx.x; t < M; t += 256) s += (kStream ? __ldcs(a + t) : a[t]) * rc[t];
  }
  __shared__ double sh[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0 && !skip) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sh[w];
    xc[row] = t;
  }
}

// ---------------------------------------------------------------- drivers
msb_status coarse_factor_dense(msb_ctx ctx, Coarse& co) {
  int M = co.M;
  cudaStream_t s = ctx->stream;
  if (!co.L) MSB_ALLOC(ctx, co.L, double, (int64_t)M * M);
  if (!co.Ainv) MSB_ALLOC(ctx, co.Ainv, double, (int64_t)M * M);
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(co.L, co.Ac, (size_t)M * M * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
  unsigned long long* amax = dalloc_n<unsigned long long>(ctx, 1);
  int* sing = dalloc_n<int>(ctx, 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(amax, 0, 8, s));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(sing, 0, 4, s));
  k_absmax<<<std::min<int64_t>(grid_for((int64_t)M * M, 256), 4 * ctx->sm_count), 256, 0, s>>>(
      co.L, (int64_t)M * M, amax);
  MSB_LAUNCH_CHECK(ctx);
  double* Lm = co.L;
  for (int k = 0; k < M; k += NB) {
    int kb = std::min(NB, M - k);
    k_potrf_diag<<<1, NB * NB, 0, s>>>(Lm, M, k, kb, amax, sing);
    MSB_LAUNCH_CHECK(ctx);
    int rows = M - k - kb;
    if (rows > 0) {
      k_trsm_panel<<<grid_for(rows, 8), 256, 0, s>>>(Lm, M, k, kb);
      MSB_LAUNCH_CHECK(ctx);
      dim3 g(grid_for(rows, 64), grid_for(rows, 64));
      double* A22 = Lm + (int64_t)(k + kb) * M + (k + kb);
      const double* L21 = Lm + (int64_t)(k + kb) * M + k;
      k_gemm_sub<<<g, 256, 0, s>>>(A22, M, L21, M, 0, L21, M, 1, rows, rows, kb, 1);
      MSB_LAUNCH_CHECK(ctx);
    }
  }
  int hs = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, sing, 4, cudaMemcpyDeviceToHost, s));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  dfree(ctx, amax);
  dfree(ctx, sing);
  if (hs) {
    co.ready = false;
    return set_error(ctx, MSB_ESINGULAR, "singular coarse matrix: pivot <= 1e-14 max|A_c| (M=%d)", M);
  }
  // X = A^{-1}: forward L Y = I, then backward L^T X = Y, blocked, in place in Ainv.
  double* X = co.Ainv;
  k_identity<<<grid_for((int64_t)M * M, 256), 256, 0, s>>>(X, M);
  MSB_LAUNCH_CHECK(ctx);
  for (int k = 0; k < M; k += NB) {
    int kb = std::min(NB, M - k);
    k_trsm_diag_rhs<<<grid_for(M, 128), 128, 0, s>>>(Lm, M, k, kb, X, M, 0);
    MSB_LAUNCH_CHECK(ctx);
    int rows = M - k - kb;
    if (rows > 0) {
      dim3 g(grid_for(M, 64), grid_for(rows, 64));
      k_gemm_sub<<<g, 256, 0, s>>>(X + (int64_t)(k + kb) * M, M, Lm + (int64_t)(k + kb) * M + k, M,
                                   0, X + (int64_t)k * M, M, 0, rows, M, kb, 0);
      MSB_LAUNCH_CHECK(ctx);
    }
  }
  int last = ((M - 1) / NB) * NB;
  for (int k = last; k >= 0; k -= NB) {
    int kb = std::min(NB, M - k);
    k_trsm_diag_rhs<<<grid_for(M, 128), 128, 0, s>>>(Lm, M, k, kb, X, M, 1);
    MSB_LAUNCH_CHECK(ctx);
    if (k > 0) {
      // rows 0..k-1: X[i,:] -= sum_{t in blk} L[t][i] X[t,:]  (op(A) = (L[blk, 0:k])^T)
      dim3 g(grid_for(M, 64), grid_for(k, 64));
      k_gemm_sub<<<g, 256, 0, s>>>(X, M, Lm + (int64_t)k * M, M, 1, X + (int64_t)k * M, M, 0, k, M,
                                   kb, 0);
      MSB_LAUNCH_CHECK(ctx);
    }
  }
  co.ready = true;
  return MSB_OK;
}

// L2 residency of the dense inverse (B200: 126 MB L2).  The inverse is the only operand
// of the cycle that is read unchanged every stage, so when the device allows a
// persisting carve-out the GEMV is launched with an access-policy window over it:
// after the first solve its lines stay in L2 and the per-stage M^2 HBM stream becomes
// an L2 read.  Opt-in (MSB_L2_PERSIST=1): measured on config 2 the carve-out cost the
// sweep 2x (its working set loses L2) for a 0.7 % cycle gain (profiles/r01_v1/).
static size_t persist_bytes(msb_ctx ctx, size_t want) {
  static int state = -1;  // -1 unknown, 0 off, 1 on
  static size_t max_win = 0, max_persist = 0;
  if (state < 0) {
    const char* e = getenv("MSB_L2_PERSIST");
    state = (e && e[0] == '1') ? 1 : 0;
    int v = 0;
    if (state && cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device) == cudaSuccess)
      max_win = (size_t)v;
    if (state && cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, ctx->device) == cudaSuccess)
      max_persist = (size_t)v;
    if (!max_win || !max_persist) state = 0;
    if (state && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, max_persist) != cudaSuccess) state = 0;
    cudaGetLastError();
  }
  if (!state) return 0;
  return std::min(want, std::min(max_win, max_persist));
}

void coarse_persist_init(msb_ctx ctx) { persist_bytes(ctx, 0); }

void coarse_solve_dense(msb_ctx ctx, const Coarse& co, const double* rc, double* xc,
                        const int* done) {
  const size_t bytes = (size_t)co.M * co.M * sizeof(double);
  const size_t win = persist_bytes(ctx, bytes);
  if (win) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(co.M);
    cfg.blockDim = dim3(256);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = co.Ainv;
    at[0].val.accessPolicyWindow.num_bytes = win;
    at[0].val.accessPolicyWindow.hitRatio = 1.0f;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_gemv<false>, (const double*)co.Ainv, co.M, rc, xc, done) ==
        cudaSuccess) {
      count_launch();
      return;
    }
    cudaGetLastError();
  }
  k_gemv<true><<<co.M, 256, 0, ctx->stream>>>(co.Ainv, co.M, rc, xc, done);
  count_launch();
}

msb_status coarse_assemble_dense(msb_ctx ctx, msb_level L, msb_op op) {
  int M = L->M;
  Coarse& co = L->co;
  if (co.cap < M) {
    coarse_free(ctx, co);
    int cap = M;
    MSB_ALLOC(ctx, co.Ac, double, (int64_t)cap * cap);
    MSB_ALLOC(ctx, co.L, double, (int64_t)cap * cap);
    MSB_ALLOC(ctx, co.Ainv, double, (int64_t)cap * cap);
    co.cap = cap;
  }
  co.M = M;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.Ac, 0, (size_t)M * M * sizeof(double), ctx->stream));
  k_rap<<<grid_for(L->N, 128), 128, 0, ctx->stream>>>(*L, L->P[L->cur], op->Tx, op->Ty, op->Tz,
                                                      co.Ac);
  MSB_LAUNCH_CHECK(ctx);
  return coarse_factor_dense(ctx, co);
}

void coarse_free(msb_ctx ctx, Coarse& co) {
  dfree(ctx, co.Ac);
  dfree(ctx, co.Ainv);
  dfree(ctx, co.L);
  co.Ac = co.Ainv = co.L = nullptr;
  co.ready = false;
  co.cap = 0;
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_coarse_assemble(msb_ctx ctx, msb_level L, msb_op op) {
  if (!ctx || !L || !op) return set_error(ctx, MSB_EINVAL, "msb_coarse_assemble: null");
  if (L->N != op->N) return set_error(ctx, MSB_EDIM, "level/operator size mismatch");
  if ((int64_t)L->M * L->M > (int64_t)1 << 31)
    return set_error(ctx, MSB_EINVAL, "dense coarse operator too large (M=%d)", L->M);
  return coarse_assemble_dense(ctx, L, op);
}
