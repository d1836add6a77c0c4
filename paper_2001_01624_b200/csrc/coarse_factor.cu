// Row a5 — dense coarse factorisation and explicit inverse (G7).
//
// A_c is SPD (Galerkin of the SPD gauged A), so the "direct Gaussian
// elimination" of PAPER.md:410 is a Cholesky factorisation L L^T without pivoting
// (reading B1).  The cycle needs A_c^{-1} r_c once per stage, so the inverse is formed
// once per assembly and every solve is one HBM-streaming GEMV (coarse.cu):
//
//   recursive Cholesky + triangular inverse on [[A11, .], [A21, A22]]:
//     (L11, W11) = chol_inv(A11)                 W = L^{-1}
//     L21  = A21 L11^{-T}                        (recursive blocked TRSM: GEMMs + leaf
//                                                 inverses, as LAPACK dpotrf)
//     A22 -= L21 L21^T                           (GEMM, lower tiles only)
//     (L22, W22) = chol_inv(A22)
//     W21  = -W22 (L21 W11)                      (two GEMMs)
//   A_c^{-1} = W^T W                             (GEMM over the nonzero K range, lower
//                                                 tiles, then mirrored)
//
// so all O(M^3) work is in plain GEMM / SYRK products and the leaves (n <= 64) are
// one-CTA kernels.  The products go to cuBLAS (DGEMM/DSYRK: 33-36 TFLOP/s fp64 on B200
// at these sizes, scripts/probes/dgemm_probe.py) — plain library GEMMs — resolved at run
// time with dlopen so the library has no link dependency; without it (or with
// MSB_OWN_DGEMM=1) they run on k_dgemm below, a register-blocked fp64 GEMM (128x128
// tiles, 8x8 per thread, double-buffered shared memory; lower-tile and triangular-K
// variants for the symmetric products).  Either way every step runs on the GPU.
// Flops: M^3/3 (chol) + M^3/3 (inverse of L) + M^3/3 (W^T W, triangular K range on
// k_dgemm; the DSYRK form does not skip W's zero upper triangle: M^3) ~ M^3 .. 5M^3/3.
// Pivot test: d_jj <= 1e-14 max|A_c| -> MSB_ESINGULAR.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>

#include <cublas_v2.h>

#include "internal.cuh"

namespace msb {

constexpr int GB = 128;   // GEMM tile (rows and columns)
constexpr int GK = 16;    // GEMM k step
constexpr int GPAD = 4;   // smem row padding (doubles)
constexpr int LEAF = 64;  // recursion leaf

// C (m x n, ldc) = alpha * op(A) op(B) + beta * C,
//   op(A)(i,t) = TA ? A[t*lda + i] : A[i*lda + t],   op(B)(t,j) = TB ? B[j*ldb + t] : B[t*ldb + j].
// lower: skip tiles strictly above the diagonal (row tile < col tile).
// tri_k: op(A)(i,t) = 0 for t < i and op(B)(t,j) = 0 for t < j (A = B = W^T W case):
//        the K loop of tile (bi, bj) starts at max(bi, bj) * GB.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm(int m, int n, int K, double alpha,
                                               const double* __restrict__ A, int64_t lda,
                                               const double* __restrict__ B, int64_t ldb,
                                               double beta, double* __restrict__ C, int64_t ldc,
                                               int lower, int tri_k) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (lower && bi < bj) return;
  extern __shared__ double gsm[];
  double* As = gsm;                           // [2][GK][GB + GPAD]
  double* Bs = gsm + 2 * GK * (GB + GPAD);    // [2][GK][GB + GPAD]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int i0 = bi * GB, j0 = bj * GB;
  int kbeg = tri_k ? max(i0, j0) : 0;
  kbeg = min(kbeg, K);
  const int nk = (K - kbeg + GK - 1) / GK;
  double acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  double ra[8], rb[8];
  // global -> register tile loader: 2048 elements of each operand per k step, 8/thread
  auto load = [&](int kk) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = tid + 256 * e;
      int i, t;
      if (TA) { t = idx >> 7; i = idx & 127; } else { i = idx >> 4; t = idx & 15; }
      const int gi = i0 + i, gt = kk + t;
      ra[e] = (gi < m && gt < K) ? (TA ? A[(int64_t)gt * lda + gi] : A[(int64_t)gi * lda + gt]) : 0.0;
      int j, tb;
      if (TB) { j = idx >> 4; tb = idx & 15; } else { tb = idx >> 7; j = idx & 127; }
      const int gj = j0 + j, gtb = kk + tb;
      rb[e] = (gj < n && gtb < K) ? (TB ? B[(int64_t)gj * ldb + gtb] : B[(int64_t)gtb * ldb + gj]) : 0.0;
    }
  };
  auto store = [&](int buf) {
    double* as = As + buf * GK * (GB + GPAD);
    double* bs = Bs + buf * GK * (GB + GPAD);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = tid + 256 * e;
      int i, t;
      if (TA) { t = idx >> 7; i = idx & 127; } else { i = idx >> 4; t = idx & 15; }
      as[t * (GB + GPAD) + i] = ra[e];
      int j, tb;
      if (TB) { j = idx >> 4; tb = idx & 15; } else { tb = idx >> 7; j = idx & 127; }
      bs[tb * (GB + GPAD) + j] = rb[e];
    }
  };
  if (nk > 0) {
    load(kbeg);
    store(0);
    __syncthreads();
  }
  for (int s = 0; s < nk; ++s) {
    const int buf = s & 1;
    if (s + 1 < nk) load(kbeg + (s + 1) * GK);
    const double* as = As + buf * GK * (GB + GPAD);
    const double* bs = Bs + buf * GK * (GB + GPAD);
#pragma unroll
    for (int t = 0; t < GK; ++t) {
      double a[8], b[8];
      const double2* ap = reinterpret_cast<const double2*>(as + t * (GB + GPAD));
      const double2* bp = reinterpret_cast<const double2*>(bs + t * (GB + GPAD));
      double2 a0 = ap[ty * 2], a1 = ap[ty * 2 + 1], a2 = ap[32 + ty * 2], a3 = ap[32 + ty * 2 + 1];
      double2 b0 = bp[tx * 2], b1 = bp[tx * 2 + 1], b2 = bp[32 + tx * 2], b3 = bp[32 + tx * 2 + 1];
      a[0] = a0.x; a[1] = a0.y; a[2] = a1.x; a[3] = a1.y;
      a[4] = a2.x; a[5] = a2.y; a[6] = a3.x; a[7] = a3.y;
      b[0] = b0.x; b[1] = b0.y; b[2] = b1.x; b[3] = b1.y;
      b[4] = b2.x; b[5] = b2.y; b[6] = b3.x; b[7] = b3.y;
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    if (s + 1 < nk) {
      store(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int i = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + (u - 4));
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int j = j0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + (v - 4));
      if (j >= n) continue;
      double* c = C + (int64_t)i * ldc + j;
      *c = beta == 0.0 ? alpha * acc[u][v] : fma(alpha, acc[u][v], beta * *c);
    }
  }
}

// ---------------------------------------------------------------- cuBLAS (run-time bound)
struct BlasApi {
  bool ok = false;
  cublasHandle_t h = nullptr;
  decltype(&cublasSetStream_v2) set_stream = nullptr;
  decltype(&cublasDgemm_v2) dgemm = nullptr;
  decltype(&cublasDsyrk_v2) dsyrk = nullptr;
  decltype(&cublasDtrmm_v2) dtrmm = nullptr;
};

static BlasApi* blas(msb_ctx ctx) {
  static BlasApi api[64];
  static bool tried[64];
  const int d = ctx->device;
  if (d < 0 || d >= 64) return nullptr;
  if (!tried[d]) {
    tried[d] = true;
    const char* own = getenv("MSB_OWN_DGEMM");
    if (own && own[0] == '1') return nullptr;
    void* lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return nullptr;
    auto create = reinterpret_cast<decltype(&cublasCreate_v2)>(dlsym(lib, "cublasCreate_v2"));
    BlasApi& a = api[d];
    a.set_stream = reinterpret_cast<decltype(&cublasSetStream_v2)>(dlsym(lib, "cublasSetStream_v2"));
    a.dgemm = reinterpret_cast<decltype(&cublasDgemm_v2)>(dlsym(lib, "cublasDgemm_v2"));
    a.dsyrk = reinterpret_cast<decltype(&cublasDsyrk_v2)>(dlsym(lib, "cublasDsyrk_v2"));
    a.dtrmm = reinterpret_cast<decltype(&cublasDtrmm_v2)>(dlsym(lib, "cublasDtrmm_v2"));
    auto set_mode =
        reinterpret_cast<decltype(&cublasSetMathMode)>(dlsym(lib, "cublasSetMathMode"));
    if (!create || !a.set_stream || !a.dgemm || !a.dsyrk) return nullptr;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(d);
    const bool made = create(&a.h) == CUBLAS_STATUS_SUCCESS;
    if (prev >= 0) cudaSetDevice(prev);
    if (!made) return nullptr;
    if (set_mode) set_mode(a.h, CUBLAS_PEDANTIC_MATH);  // plain fp64, no emulation
    a.ok = true;
  }
  return api[d].ok ? &api[d] : nullptr;
}

// Row-major C (m x n, ldc) = alpha op(A) op(B) + beta C on cuBLAS (column-major): the
// same memory read column-major is the transpose, so C^T = op(B)^T op(A)^T.
template <bool TA, bool TB>
static bool blas_gemm(msb_ctx ctx, int m, int n, int K, double alpha, const double* A,
                      int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                      int64_t ldc) {
  BlasApi* b = blas(ctx);
  if (!b || b->set_stream(b->h, ctx->stream) != CUBLAS_STATUS_SUCCESS) return false;
  return b->dgemm(b->h, TB ? CUBLAS_OP_T : CUBLAS_OP_N, TA ? CUBLAS_OP_T : CUBLAS_OP_N, n, m, K,
                  &alpha, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc) == CUBLAS_STATUS_SUCCESS;
}

// Row-major lower triangle of C (n x n) = alpha X + beta C with X = A A^T (at = false,
// A n x k) or X = A^T A (at = true, A k x n); the row-major lower triangle is the
// column-major upper one.
static bool blas_syrk(msb_ctx ctx, bool at, int n, int k, double alpha, const double* A,
                      int64_t lda, double beta, double* C, int64_t ldc) {
  BlasApi* b = blas(ctx);
  if (!b || b->set_stream(b->h, ctx->stream) != CUBLAS_STATUS_SUCCESS) return false;
  return b->dsyrk(b->h, CUBLAS_FILL_MODE_UPPER, at ? CUBLAS_OP_N : CUBLAS_OP_T, n, k, &alpha, A,
                  (int)lda, &beta, C, (int)ldc) == CUBLAS_STATUS_SUCCESS;
}

// Row-major C (m x n, ldc) = W22^T W21 for W22 lower triangular (n x n, lda) and W21
// (n rows x m cols, ldb): in column-major terms C_cm = W21_cm W22_cm^T with W22_cm upper
// triangular — cuBLAS DTRMM, side right, out of place.
static bool blas_trmm_lt(msb_ctx ctx, int m, int n, const double* W22, int64_t lda,
                         const double* W21, int64_t ldb, double* C, int64_t ldc) {
  BlasApi* b = blas(ctx);
  if (!b || !b->dtrmm || b->set_stream(b->h, ctx->stream) != CUBLAS_STATUS_SUCCESS) return false;
  const double one = 1.0;
  return b->dtrmm(b->h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                  CUBLAS_DIAG_NON_UNIT, m, n, &one, W22, (int)lda, W21, (int)ldb, C,
                  (int)ldc) == CUBLAS_STATUS_SUCCESS;
}

constexpr size_t GEMM_SMEM = 2 * 2 * GK * (GB + GPAD) * sizeof(double);

template <bool TA, bool TB>
static msb_status gemm(msb_ctx ctx, int m, int n, int K, double alpha, const double* A, int64_t lda,
                       const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                       bool lower = false, bool tri_k = false) {
  if (m <= 0 || n <= 0) return MSB_OK;
  if (!lower && !tri_k && K > 0 &&
      blas_gemm<TA, TB>(ctx, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc)) {
    count_launch();
    return MSB_OK;
  }
  static bool attr = false;
  if (!attr) {
    MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_dgemm<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)GEMM_SMEM));
    attr = true;
  }
  dim3 g((n + GB - 1) / GB, (m + GB - 1) / GB);
  k_dgemm<TA, TB><<<g, 256, GEMM_SMEM, ctx->stream>>>(m, n, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                       lower ? 1 : 0, tri_k ? 1 : 0);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

// Leaf: Cholesky of the n x n (n <= LEAF) block at A (ld) in place (lower; upper zeroed)
// and its triangular inverse into W (ld, lower; upper zeroed).  One CTA, LEAF^2 smem.
__global__ void __launch_bounds__(1024) k_chol_inv_leaf(double* __restrict__ A, int64_t ld, int n,
                                                        double* __restrict__ W,
                                                        const unsigned long long* amax_bits,
                                                        int* __restrict__ singular) {
  static_assert(LEAF == 64, "thread-element map assumes 64 x 64 leaves and 1024 threads");
  extern __shared__ double lsm[];
  double (*a)[LEAF + 1] = reinterpret_cast<double (*)[LEAF + 1]>(lsm);
  double (*w)[LEAF + 1] = reinterpret_cast<double (*)[LEAF + 1]>(lsm + LEAF * (LEAF + 1));
  const int tid = threadIdx.x;
  for (int e = tid; e < LEAF * LEAF; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    a[r][c] = (r < n && c < n) ? A[(int64_t)r * ld + c] : 0.0;
    w[r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double amax = __longlong_as_double((long long)*amax_bits);
  // Right-looking Cholesky fused with the forward substitution W = L^{-1}: at step j the
  // pivot is taken, column j of L is scaled and row j of W finished (w[j][c] / L_jj), then
  // every later row receives its rank-1 updates of L and of W (w[r][c] -= L_rj W_jc, c <= j)
  // in parallel — the same operations in the same order as a column-by-column forward
  // substitution, so the result is unchanged, with 3 barriers per step instead of an
  // O(n^2) serial loop per column.
  for (int j = 0; j < n; ++j) {
    if (tid == 0) {
      double d = a[j][j];
      if (!(d > 1e-14 * amax)) {
        atomicExch(singular, 1);
        d = 1.0;
      }
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    const double ljj = a[j][j];
    if (tid < LEAF) {
      if (tid > j && tid < n) a[tid][j] /= ljj;
    } else if (tid < 2 * LEAF) {
      const int c = tid - LEAF;
      if (c <= j) w[j][c] = w[j][c] / ljj;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (LEAF * LEAF) / 1024; ++u) {
      const int e = tid + 1024 * u, r = e >> 6, c = e & 63;
      if (r > j && r < n) {
        if (c > j) {
          if (c <= r) a[r][c] -= a[r][j] * a[c][j];
        } else {
          w[r][c] -= a[r][j] * w[j][c];
        }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    A[(int64_t)r * ld + c] = c <= r ? a[r][c] : 0.0;
    W[(int64_t)r * ld + c] = c <= r ? w[r][c] : 0.0;
  }
}

// dst (rows x cols, ldd) = src (ld s)
__global__ void k_copy2d(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src,
                         int64_t lds, int rows, int cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * cols) return;
  const int r = (int)(e / cols), c = (int)(e % cols);
  dst[(int64_t)r * ldd + c] = src[(int64_t)r * lds + c];
}

// X[j][i] = X[i][j] for i > j (mirror the lower triangle), 32x32 tiles through smem
__global__ void k_mirror_lower(double* __restrict__ X, int M) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bi < bj) return;
  __shared__ double t[32][33];
  const int i = bi * 32 + threadIdx.y, j = bj * 32 + threadIdx.x;
  if (i < M && j < M) t[threadIdx.y][threadIdx.x] = X[(int64_t)i * M + j];
  __syncthreads();
  const int i2 = bj * 32 + threadIdx.y, j2 = bi * 32 + threadIdx.x;  // transposed tile
  if (i2 < M && j2 < M && j2 > i2) X[(int64_t)i2 * M + j2] = t[threadIdx.x][threadIdx.y];
}

// Split rule shared by chol_inv and rtrsm, so that rtrsm's leaves are exactly the
// diagonal blocks whose inverses chol_inv's leaves stored in W.
static inline int split1(int n) { return ((n / 2 + LEAF - 1) / LEAF) * LEAF; }

// X = B L^{-T} (solve X L^T = B) for B: m x n (ld), L: n x n lower (ld), recursively:
//   X_a = B_a L_a^{-T};  B_c -= X_a L_b^T;  X_c = B_c L_c^{-T}
// with leaves X = B W_leaf^T using the leaf inverses W (= L^{-1} diagonal blocks).
// B is overwritten (scratch).  This is the blocked TRSM of LAPACK dpotrf (backward
// stable up to the conditioning of the 64 x 64 leaf blocks), not a product with the
// full inverse of L11.
static msb_status rtrsm(msb_ctx ctx, double* B, double* X, int m, int n, const double* L,
                        const double* W, int64_t ld) {
  if (n <= LEAF) return gemm<false, true>(ctx, m, n, n, 1.0, B, ld, W, ld, 0.0, X, ld);
  const int na = split1(n), nc = n - na;
  msb_status rc;
  if ((rc = rtrsm(ctx, B, X, m, na, L, W, ld))) return rc;
  const double* Lb = L + (int64_t)na * ld;  // rows na..n, cols 0..na
  if ((rc = gemm<false, true>(ctx, m, nc, na, -1.0, X, ld, Lb, ld, 1.0, B + na, ld))) return rc;
  return rtrsm(ctx, B + na, X + na, m, nc, Lb + na, W + (int64_t)na * ld + na, ld);
}

// Recursive Cholesky + inverse of the n x n block at F (ld), inverse factor into Wb.
// F's strictly-upper triangle is used as scratch.
static msb_status chol_inv(msb_ctx ctx, double* F, double* Wb, int64_t ld, int n,
                           const unsigned long long* amax, int* sing) {
  if (n <= LEAF) {
    constexpr size_t smem = 2 * LEAF * (LEAF + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_chol_inv_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
      attr = true;
    }
    k_chol_inv_leaf<<<1, 1024, smem, ctx->stream>>>(F, ld, n, Wb, amax, sing);
    MSB_LAUNCH_CHECK(ctx);
    return MSB_OK;
  }
  const int n1 = split1(n), n2 = n - n1;
  double* F11 = F;
  double* F21 = F + (int64_t)n1 * ld;
  double* F12 = F + n1;
  double* F22 = F21 + n1;
  double* W11 = Wb;
  double* W21 = Wb + (int64_t)n1 * ld;
  double* W22 = W21 + n1;
  msb_status rc;
  if ((rc = chol_inv(ctx, F11, W11, ld, n1, amax, sing))) return rc;
  // L21 = A21 L11^{-T} (blocked TRSM into the W21 block, free until the last step)
  if ((rc = rtrsm(ctx, F21, W21, n2, n1, F11, W11, ld))) return rc;
  k_copy2d<<<grid_for((int64_t)n2 * n1, 256), 256, 0, ctx->stream>>>(F21, ld, W21, ld, n2, n1);
  MSB_LAUNCH_CHECK(ctx);
  // A22 -= L21 L21^T (lower tiles)
  if (blas_syrk(ctx, false, n2, n1, -1.0, F21, ld, 1.0, F22, ld))
    count_launch();
  else if ((rc = gemm<false, true>(ctx, n2, n2, n1, -1.0, F21, ld, F21, ld, 1.0, F22, ld, true)))
    return rc;
  if ((rc = chol_inv(ctx, F22, W22, ld, n2, amax, sing))) return rc;
  // triangular inverse (LAPACK dtrtri): T^T = W11^T L21^T (n1 x n2) into the free upper
  // block F12;  W21 = -W22 T
  if ((rc = gemm<true, true>(ctx, n1, n2, n1, 1.0, W11, ld, F21, ld, 0.0, F12, ld))) return rc;
  if ((rc = gemm<false, true>(ctx, n2, n1, n2, -1.0, W22, ld, F12, ld, 0.0, W21, ld))) return rc;
  return MSB_OK;
}

__global__ void k_absmax2(const double* __restrict__ A, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Lower triangle of F = W^T W for lower-triangular W (LAPACK dlauum, recursive):
//   [W11 0; W21 W22]: F11 = W11^T W11 + W21^T W21, F21 = W22^T W21, F22 = W22^T W22
// — M^3/3 flops instead of the M^3 of one DSYRK over the full (half-zero) W.  Leaves
// (n <= 512) are one DSYRK.  Returns false when cuBLAS is not available.
static bool lauum(msb_ctx ctx, const double* W, double* F, int n, int64_t ld) {
  if (n <= 512) return blas_syrk(ctx, true, n, n, 1.0, W, ld, 0.0, F, ld);
  const int n1 = split1(n), n2 = n - n1;
  const double* W21 = W + (int64_t)n1 * ld;
  const double* W22 = W21 + n1;
  double* F21 = F + (int64_t)n1 * ld;
  double* F22 = F21 + n1;
  if (!lauum(ctx, W, F, n1, ld)) return false;
  if (!blas_syrk(ctx, true, n1, n2, 1.0, W21, ld, 1.0, F, ld)) return false;
  if (!blas_trmm_lt(ctx, n1, n2, W22, ld, W21, ld, F21, ld)) return false;
  return lauum(ctx, W22, F22, n2, ld);
}

msb_status coarse_factor_dense(msb_ctx ctx, Coarse& co) {
  const int M = co.M;
  cudaStream_t s = ctx->stream;
  if (!co.flags) MSB_ALLOC(ctx, co.flags, unsigned long long, 2);
  unsigned long long* amax = co.flags;
  int* sing = reinterpret_cast<int*>(co.flags + 1);
  if (!co.L) MSB_ALLOC(ctx, co.L, double, (int64_t)M * M);
  if (!co.Ainv) MSB_ALLOC(ctx, co.Ainv, double, (int64_t)M * M);
  double* F = co.L;
  double* Wb = co.Ainv;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(F, co.Ac, (size_t)M * M * sizeof(double), cudaMemcpyDeviceToDevice, s));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(Wb, 0, (size_t)M * M * sizeof(double), s));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.flags, 0, 16, s));
  k_absmax2<<<std::min<int64_t>(grid_for((int64_t)M * M, 256), 4 * ctx->sm_count), 256, 0, s>>>(
      F, (int64_t)M * M, amax);
  MSB_LAUNCH_CHECK(ctx);
  msb_status rc = chol_inv(ctx, F, Wb, M, M, amax, sing);
  if (rc) return rc;
  int hs = 0;
  if (!co.defer_check) {  // the dynamic stage reads the flag with its next stop-test readback
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, sing, 4, cudaMemcpyDeviceToHost, s));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  }
  if (hs) {
    co.ready = false;
    return set_error(ctx, MSB_ESINGULAR, "singular coarse matrix: pivot <= 1e-14 max|A_c| (M=%d)", M);
  }
  // A_c^{-1} = W^T W: lower tiles with the K range restricted to the nonzeros of W,
  // written over the factor buffer (L is no longer needed), then mirrored; swap so
  // that co.Ainv holds the inverse and co.L the inverse factor W.
  static const bool full_syrk = getenv("MSB_FULL_SYRK") != nullptr;
  if (!full_syrk && lauum(ctx, Wb, F, M, M))
    count_launch();
  else if (blas_syrk(ctx, true, M, M, 1.0, Wb, M, 0.0, F, M))
    count_launch();
  else if ((rc = gemm<true, false>(ctx, M, M, M, 1.0, Wb, M, Wb, M, 0.0, F, M, true, true)))
    return rc;
  dim3 g((M + 31) / 32, (M + 31) / 32);
  k_mirror_lower<<<g, dim3(32, 32), 0, s>>>(F, M);
  MSB_LAUNCH_CHECK(ctx);
  std::swap(co.L, co.Ainv);
  if ((rc = coarse_pack_symmetric(ctx, co))) return rc;
  co.ready = true;
  return MSB_OK;
}

}  // namespace msb
