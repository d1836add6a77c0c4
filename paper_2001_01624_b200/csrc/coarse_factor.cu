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
// so all O(M^3) work is in plain GEMM / SYRK / TRMM products on the library's own fp64
// tensor-core GEMM (k_dgemm below, DMMA) and the leaves (n <= 64) are one-CTA kernels.
// Flops: M^3/3 (chol) + M^3/3 (inverse of L) + M^3/3 (W^T W, triangular K range) ~ M^3.
// Pivot test: d_jj <= 1e-14 max|A_c| -> MSB_ESINGULAR.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace msb {

constexpr int LEAF = 64;  // recursion leaf

// ---------------------------------------------------------------- fp64 tensor-core GEMM
// C (m x n, ldc) = alpha * op(A) op(B) + beta * C, row-major,
//   op(A)(i,t) = TA ? A[t*lda + i] : A[i*lda + t],   op(B)(t,j) = TB ? B[j*ldb + t] : B[t*ldb + j],
// on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64: the only fp64 MMA of sm_100a —
// tcgen05 has no f64 kind).  128 x 128 output tile per CTA, 8 warps as 2 (m) x 4 (n), each
// 64 x 32 = 8 x 4 fragments of 8 x 8; K in steps of 16 through a 3-stage cp.async ring
// (8-byte copies: leading dimensions may be odd; out-of-range elements zero-filled).
//   lower: skip tiles strictly above the diagonal (row tile < col tile): SYRK.
//   kmode 1: op(A)(i,t) = 0 for t < i (A^T of a lower-triangular A): TRMM, K from i0;
//   kmode 2: additionally op(B)(t,j) = 0 for t < j (W^T W): K from max(i0, j0).
// fp64 FMA throughout (DMMA rounds each product-sum exactly like an fp64 FMA chain, in a
// fixed order per output element), so results are deterministic run to run.
constexpr int DG_T = 128, DG_K = 16, DG_S = 3;
constexpr int DG_PAD = 4;
constexpr int DG_A_MK = DG_T * (DG_K + DG_PAD);  // [m][k] layout (TA = false)
constexpr int DG_A_KM = DG_K * (DG_T + DG_PAD);  // [k][m] layout (TA = true)
constexpr int DG_STAGE = (DG_A_MK > DG_A_KM ? DG_A_MK : DG_A_KM);
constexpr size_t DG_SMEM = (size_t)2 * DG_S * DG_STAGE * sizeof(double);

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm(int m, int n, int K, double alpha,
                                               const double* __restrict__ A, int64_t lda,
                                               const double* __restrict__ B, int64_t ldb,
                                               double beta, double* __restrict__ C, int64_t ldc,
                                               int lower, int kmode, double* __restrict__ ws) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (lower && bi < bj) return;
  extern __shared__ double dsm[];
  double* As = dsm;                       // [DG_S][DG_STAGE]
  double* Bs = dsm + DG_S * DG_STAGE;     // [DG_S][DG_STAGE]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile rows wm*64, cols wn*32
  const int i0 = bi * DG_T, j0 = bj * DG_T;
  int kbeg = kmode == 2 ? max(i0, j0) : (kmode == 1 ? i0 : 0);
  kbeg = min(kbeg, K);
  int nk = (K - kbeg + DG_K - 1) / DG_K;
  if (gridDim.z > 1) {  // split K: this CTA takes k-steps [z nk / S, (z + 1) nk / S)
    const int z = blockIdx.z, S = gridDim.z;
    const int s0 = (int)((int64_t)nk * z / S), s1 = (int)((int64_t)nk * (z + 1) / S);
    kbeg += s0 * DG_K;
    nk = s1 - s0;
  }
  const int kend = min(K, kbeg + nk * DG_K);
  // stage loader: 2048 elements of each operand, 8 per thread
  auto load = [&](int s, int kk) {
    double* as = As + s * DG_STAGE;
    double* bs = Bs + s * DG_STAGE;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = tid + 256 * e;
      if (TA) {  // memory rows t, contiguous i: smem [k][m]
        const int t = idx >> 7, i = idx & 127;
        const int gi = i0 + i, gt = kk + t;
        const bool ok = gi < m && gt < kend;
        cp_async8(as + t * (DG_T + DG_PAD) + i, ok ? A + (int64_t)gt * lda + gi : A, ok);
      } else {   // memory rows i, contiguous t: smem [m][k]
        const int i = idx >> 4, t = idx & 15;
        const int gi = i0 + i, gt = kk + t;
        const bool ok = gi < m && gt < kend;
        cp_async8(as + i * (DG_K + DG_PAD) + t, ok ? A + (int64_t)gi * lda + gt : A, ok);
      }
      if (TB) {  // memory rows j, contiguous t: smem [n][k]
        const int j = idx >> 4, t = idx & 15;
        const int gj = j0 + j, gt = kk + t;
        const bool ok = gj < n && gt < kend;
        cp_async8(bs + j * (DG_K + DG_PAD) + t, ok ? B + (int64_t)gj * ldb + gt : B, ok);
      } else {   // memory rows t, contiguous j: smem [k][n]
        const int t = idx >> 7, j = idx & 127;
        const int gj = j0 + j, gt = kk + t;
        const bool ok = gj < n && gt < kend;
        cp_async8(bs + t * (DG_T + DG_PAD) + j, ok ? B + (int64_t)gt * ldb + gj : B, ok);
      }
    }
  };
  double acc[8][4][2];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
#pragma unroll
  for (int s = 0; s < DG_S - 1; ++s) {
    if (s < nk) load(s, kbeg + s * DG_K);
    cp_async_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;  // fragment row / k index of this lane
  for (int st = 0; st < nk; ++st) {
    cp_async_wait<DG_S - 2>();
    __syncthreads();
    {  // prefetch stage st + DG_S - 1 into the slot consumed at st - 1
      const int nx = st + DG_S - 1;
      if (nx < nk) load(nx % DG_S, kbeg + nx * DG_K);
      cp_async_commit();
    }
    const double* as = As + (st % DG_S) * DG_STAGE;
    const double* bs = Bs + (st % DG_S) * DG_STAGE;
#pragma unroll
    for (int kq = 0; kq < DG_K; kq += 4) {
      double a[8], b[4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = wm * 64 + u * 8 + fr;
        a[u] = TA ? as[(kq + fc) * (DG_T + DG_PAD) + r] : as[r * (DG_K + DG_PAD) + kq + fc];
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int cidx = wn * 32 + v * 8 + fr;
        b[v] = TB ? bs[cidx * (DG_K + DG_PAD) + kq + fc] : bs[(kq + fc) * (DG_T + DG_PAD) + cidx];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) dmma(acc[u][v], a[u], b[v]);
    }
  }
  cp_async_wait<0>();
  if (ws) {  // split K: the raw partial tile, summed in split order by k_dgemm_splitk_sum
    double* wt = ws + (((int64_t)blockIdx.z * gridDim.y + bi) * gridDim.x + bj) * DG_T * DG_T;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int li = wm * 64 + u * 8 + fr, lj = wn * 32 + v * 8 + 2 * fc;
        *reinterpret_cast<double2*>(wt + li * DG_T + lj) = make_double2(acc[u][v][0], acc[u][v][1]);
      }
    return;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int i = i0 + wm * 64 + u * 8 + fr;
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + wn * 32 + v * 8 + 2 * fc + h;
        if (j >= n) continue;
        double* c = C + (int64_t)i * ldc + j;
        *c = beta == 0.0 ? alpha * acc[u][v][h] : fma(alpha, acc[u][v][h], beta * *c);
      }
    }
  }
}

// C = alpha * (sum over the S split partials, in split order) + beta * C
__global__ void k_dgemm_splitk_sum(const double* __restrict__ ws, int S, int gx, int gy, int m,
                                   int n, double alpha, double beta, double* __restrict__ C,
                                   int64_t ldc, int lower) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * n) return;
  const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
  const int bi = i / DG_T, bj = j / DG_T;
  if (lower && bi < bj) return;
  const int64_t tile = (int64_t)bi * gx + bj, off = (i - bi * DG_T) * DG_T + (j - bj * DG_T);
  double v = 0.0;
  for (int z = 0; z < S; ++z) v += ws[((int64_t)z * gy * gx + tile) * DG_T * DG_T + off];
  double* c = C + (int64_t)i * ldc + j;
  *c = beta == 0.0 ? alpha * v : fma(alpha, v, beta * *c);
}

// One CTA per SM (the 101 KB ring and 64 fp64 accumulators per thread) and ~70 fp64 FMA
// per clock per SM: a product with few output tiles (the narrow panels of the recursion)
// splits its K range over more CTAs, partial tiles to a workspace summed in a fixed order.
template <bool TA, bool TB>
static msb_status gemm(msb_ctx ctx, int m, int n, int K, double alpha, const double* A, int64_t lda,
                       const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                       bool lower = false, int kmode = 0) {
  if (m <= 0 || n <= 0) return MSB_OK;
  static bool attr = false;
  if (!attr) {
    MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_dgemm<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)DG_SMEM));
    attr = true;
  }
  const int gx = (n + DG_T - 1) / DG_T, gy = (m + DG_T - 1) / DG_T;
  const int tiles = lower ? (gx * (gx + 1)) / 2 + (gy - gx) * gx : gx * gy;
  int S = 1;
  if (kmode == 0 && K >= 8 * DG_K && tiles < 2 * ctx->sm_count) {
    S = std::min((2 * ctx->sm_count + tiles - 1) / tiles, K / (4 * DG_K));
    S = std::max(1, std::min(S, 32));
  }
  double* ws = nullptr;
  if (S > 1) {
    const size_t need = (size_t)S * gx * gy * DG_T * DG_T;
    if (ctx->gemm_ws_cap < need) {
      dfree(ctx, ctx->gemm_ws);
      ctx->gemm_ws = dalloc_n<double>(ctx, need);
      ctx->gemm_ws_cap = ctx->gemm_ws ? need : 0;
    }
    ws = ctx->gemm_ws;
    if (!ws) S = 1;
  }
  dim3 g(gx, gy, S);
  k_dgemm<TA, TB><<<g, 256, DG_SMEM, ctx->stream>>>(m, n, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                     lower ? 1 : 0, kmode, S > 1 ? ws : nullptr);
  MSB_LAUNCH_CHECK(ctx);
  if (S > 1) {
    k_dgemm_splitk_sum<<<grid_for((int64_t)m * n, 256), 256, 0, ctx->stream>>>(
        ws, S, gx, gy, m, n, alpha, beta, C, ldc, lower ? 1 : 0);
    MSB_LAUNCH_CHECK(ctx);
  }
  return MSB_OK;
}

msb_status dgemm(msb_ctx ctx, bool ta, bool tb, int m, int n, int K, double alpha, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (ta && tb) return gemm<true, true>(ctx, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc);
  if (ta) return gemm<true, false>(ctx, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc);
  if (tb) return gemm<false, true>(ctx, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc);
  return gemm<false, false>(ctx, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

// Leaf: the Cholesky factor L of the n x n (n <= LEAF) block at A (ld), in place (lower;
// upper zeroed), and its triangular inverse W = L^{-1} into W (ld, lower), from an LDL^T
// elimination in blocks of 4 pivots (3 barriers per 4 pivots instead of 3 per pivot) with
// the square roots deferred to a final parallel pass (L = L' D^{1/2}, W = D^{-1/2} L'^{-1}):
// the critical path per pivot is one reciprocal and a few FMAs.  W' = L'^{-1} is built
// alongside (the forward substitution of each finished block of L' into the rows below).
// Pivot test on d_j = l_jj^2 <= 1e-14 max|A_c|.  1024 threads, 64 x 64 leaves.
constexpr int LB = 4;
__global__ void __launch_bounds__(1024) k_ldl_inv_leaf(double* __restrict__ A, int64_t ld, int n,
                                                       double* __restrict__ W,
                                                       const unsigned long long* amax_bits,
                                                       int* __restrict__ singular) {
  static_assert(LEAF == 64, "thread-element map assumes 64 x 64 leaves and 1024 threads");
  extern __shared__ double lsm[];
  double (*a)[LEAF + 1] = reinterpret_cast<double (*)[LEAF + 1]>(lsm);
  double (*w)[LEAF + 1] = reinterpret_cast<double (*)[LEAF + 1]>(lsm + LEAF * (LEAF + 1));
  __shared__ double u[LEAF][LB];  // u_it = L'_it d_t of the current block's columns
  __shared__ double dinv[LEAF], dd[LEAF];
  const int tid = threadIdx.x;
  for (int e = tid; e < LEAF * LEAF; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    a[r][c] = (r < n && c < n) ? A[(int64_t)r * ld + c] : 0.0;
    w[r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double tol = 1e-14 * __longlong_as_double((long long)*amax_bits);
  for (int jb = 0; jb < n; jb += LB) {
    const int je = min(jb + LB, n);
    // 1. the diagonal block: unit L' and d (one thread; <= 4 pivots)
    if (tid == 0) {
      for (int j = jb; j < je; ++j) {
        double d = a[j][j];
        if (!(d > tol)) {
          atomicExch(singular, 1);
          d = 1.0;
        }
        dd[j] = d;
        const double r = 1.0 / d;
        dinv[j] = r;
        for (int i = j + 1; i < je; ++i) {
          const double uij = a[i][j];
          a[i][j] = uij * r;  // L'_ij
          for (int k = j + 1; k <= i; ++k) a[i][k] -= uij * (a[k][j]);  // a[k][j] = L'_kj (k > j)
        }
      }
    }
    __syncthreads();
    // 2. rows below the block: u_it and L'_it (forward substitution with the unit block);
    //    W' rows of the block (unit lower inverse within the block)
    if (tid < LEAF) {
      const int i = tid;
      if (i >= je && i < n) {
        double v[LB];
#pragma unroll
        for (int t = 0; t < LB; ++t) {
          const int j = jb + t;
          if (j < je) {
            double x = a[i][j];
            for (int q = 0; q < t; ++q) x -= v[q] * a[j][jb + q];
            v[t] = x;
          } else {
            v[t] = 0.0;
          }
        }
#pragma unroll
        for (int t = 0; t < LB; ++t) {
          u[i][t] = v[t];
          if (jb + t < je) a[i][jb + t] = v[t] * dinv[jb + t];
        }
      }
    } else if (tid < 2 * LEAF) {
      const int c = tid - LEAF;
      for (int j = jb + 1; j < je; ++j) {
        double x = w[j][c];
        for (int q = jb; q < j; ++q) x -= a[j][q] * w[q][c];
        w[j][c] = x;
      }
    }
    __syncthreads();
    // 3. rank-(je - jb) updates of the trailing matrix and of the W' rows below the block
#pragma unroll
    for (int e4 = 0; e4 < (LEAF * LEAF) / 1024; ++e4) {
      const int e = tid + 1024 * e4, r = e >> 6, c = e & 63;
      if (r >= je && r < n) {
        if (c >= je) {
          if (c <= r) {
            double x = a[r][c];
            for (int t = 0; t < je - jb; ++t) x -= u[r][t] * a[c][jb + t];
            a[r][c] = x;
          }
        } else if (c < je) {
          double x = w[r][c];
          for (int t = 0; t < je - jb; ++t) x -= a[r][jb + t] * w[jb + t][c];
          w[r][c] = x;
        }
      }
    }
    __syncthreads();
  }
  // L = L' D^{1/2}, W = D^{-1/2} W'
  if (tid < n) {
    const double sq = sqrt(dd[tid]);
    dd[tid] = sq;
    dinv[tid] = 1.0 / sq;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    A[(int64_t)r * ld + c] = c < r ? a[r][c] * dd[c] : (c == r ? dd[r] : 0.0);
    W[(int64_t)r * ld + c] = c <= r ? w[r][c] * dinv[r] : 0.0;
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

// Split rule shared by chol_inv and rtrsm, so that rtrsm's leaves are diagonal blocks
// whose inverses chol_inv stored in W (the inverse factor of every recursion node is
// complete when rtrsm runs: W_aa = (L_aa)^{-1} for a diagonal block of a lower-triangular
// factor).  rtrsm stops at RT_LEAF: blocked TRSM with explicit inverses of <= 256-wide
// diagonal blocks (LAPACK's dtrtri applies inverse blocks the same way), one product
// per 256 columns instead of a recursion down to the 64-wide leaves.
constexpr int RT_LEAF = 256;
static inline int split1(int n) { return ((n / 2 + LEAF - 1) / LEAF) * LEAF; }

// X = B L^{-T} (solve X L^T = B) for B: m x n (ld), L: n x n lower (ld), recursively:
//   X_a = B_a L_a^{-T};  B_c -= X_a L_b^T;  X_c = B_c L_c^{-T}
// with leaves X = B W_leaf^T using the leaf inverses W (= L^{-1} diagonal blocks).
// B is overwritten (scratch).  This is the blocked TRSM of LAPACK dpotrf (backward
// stable up to the conditioning of the 64 x 64 leaf blocks), not a product with the
// full inverse of L11.
static msb_status rtrsm(msb_ctx ctx, double* B, double* X, int m, int n, const double* L,
                        const double* W, int64_t ld) {
  if (n <= RT_LEAF) return gemm<false, true>(ctx, m, n, n, 1.0, B, ld, W, ld, 0.0, X, ld);
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
      MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_ldl_inv_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
      attr = true;
    }
    k_ldl_inv_leaf<<<1, 1024, smem, ctx->stream>>>(F, ld, n, Wb, amax, sing);
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
  if ((rc = gemm<false, true>(ctx, n2, n2, n1, -1.0, F21, ld, F21, ld, 1.0, F22, ld, true)))
    return rc;
  if ((rc = chol_inv(ctx, F22, W22, ld, n2, amax, sing))) return rc;
  // triangular inverse (LAPACK dtrtri): T^T = W11^T L21^T (n1 x n2) into the free upper
  // block F12;  W21 = -W22 T
  if ((rc = gemm<true, true>(ctx, n1, n2, n1, 1.0, W11, ld, F21, ld, 0.0, F12, ld))) return rc;
  if ((rc = gemm<false, true>(ctx, n2, n1, n2, -1.0, W22, ld, F12, ld, 0.0, W21, ld))) return rc;
  return MSB_OK;
}

__global__ void k_absmax2(const double* __restrict__ A, int64_t n, unsigned long long* out,
                          const int* Md = nullptr) {
  if (Md) n = (int64_t)*Md * *Md;  // an M x M matrix, M from the device
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Lower triangle of F = W^T W for lower-triangular W (LAPACK dlauum, recursive):
//   [W11 0; W21 W22]: F11 = W11^T W11 + W21^T W21, F21 = W22^T W21, F22 = W22^T W22
// — M^3/3 flops instead of the M^3 of one SYRK over the full (half-zero) W.  Leaves
// (n <= 512) are one triangular-K product (kmode 2).
static msb_status lauum(msb_ctx ctx, const double* W, double* F, int n, int64_t ld) {
  if (n <= 512) return gemm<true, false>(ctx, n, n, n, 1.0, W, ld, W, ld, 0.0, F, ld, true, 2);
  const int n1 = split1(n), n2 = n - n1;
  const double* W21 = W + (int64_t)n1 * ld;
  const double* W22 = W21 + n1;
  double* F21 = F + (int64_t)n1 * ld;
  double* F22 = F21 + n1;
  msb_status rc;
  if ((rc = lauum(ctx, W, F, n1, ld))) return rc;
  if ((rc = gemm<true, false>(ctx, n1, n1, n2, 1.0, W21, ld, W21, ld, 1.0, F, ld, true))) return rc;
  if ((rc = gemm<true, false>(ctx, n2, n1, n2, 1.0, W22, ld, W21, ld, 0.0, F21, ld, false, 1)))
    return rc;
  return lauum(ctx, W22, F22, n2, ld);
}

// ---------------------------------------------------------------- small SPD systems
// One CTA: LDL^T of the M x M (M <= SMALL_CHOL_M) matrix A (row-major) in shared memory,
// packed lower rows a[i (i+1)/2 + j], in blocks of SB pivots (3 barriers per block): the
// diagonal block by one thread, the rows below it by one thread each (forward substitution
// with the unit block), then the rank-SB update of the trailing matrix.  Output: the unit
// L' packed (diagonal slots unused) followed by the M reciprocal pivots 1/d_j.  Pivot test
// as the recursive path (d_j <= 1e-14 max|A_c| -> singular).  The same matrix as the
// Cholesky factor L = L' D^{1/2}.
constexpr int SC_T = 512, SB = 8;
__global__ void __launch_bounds__(SC_T) k_chol_small(const double* __restrict__ A, int M,
                                                     double* __restrict__ Lp,
                                                     const unsigned long long* amax_bits,
                                                     int* __restrict__ singular, const int* Md) {
  if (Md) {  // M from the device (graph-captured small path; 0 = skip)
    M = *Md;
    if (M == 0) return;
  }
  extern __shared__ double sm[];
  const int np = M * (M + 1) / 2;
  double* a = sm;
  double* dd = sm + np;      // d_j
  double* di = dd + M;       // 1 / d_j
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < M; i += SC_T / 32)
    for (int j = lane; j <= i; j += 32) a[i * (i + 1) / 2 + j] = A[(int64_t)i * M + j];
  __syncthreads();
  const double tol = 1e-14 * __longlong_as_double((long long)*amax_bits);
  for (int jb = 0; jb < M; jb += SB) {
    const int je = min(jb + SB, M);
    if (tid == 0) {
      for (int j = jb; j < je; ++j) {
        double d = a[j * (j + 1) / 2 + j];
        if (!(d > tol)) {
          *singular = 1;
          d = 1.0;
        }
        const double r = 1.0 / d;
        dd[j] = d;
        di[j] = r;
        for (int i = j + 1; i < je; ++i) {
          const int ri = i * (i + 1) / 2;
          const double uij = a[ri + j];
          a[ri + j] = uij * r;
          for (int k = j + 1; k <= i; ++k) a[ri + k] -= uij * a[k * (k + 1) / 2 + j];
        }
      }
    }
    __syncthreads();
    for (int i = je + tid; i < M; i += SC_T) {  // L'_it for the rows below the block
      const int ri = i * (i + 1) / 2;
      double v[SB];
#pragma unroll
      for (int t = 0; t < SB; ++t) {
        const int j = jb + t;
        v[t] = 0.0;
        if (j < je) {
          double x = a[ri + j];
          const int rj = j * (j + 1) / 2;
          for (int q = 0; q < t; ++q) x -= v[q] * a[rj + jb + q];
          v[t] = x;
        }
      }
#pragma unroll
      for (int t = 0; t < SB; ++t)
        if (jb + t < je) a[ri + jb + t] = v[t] * di[jb + t];
    }
    __syncthreads();
    for (int i = je + warp; i < M; i += SC_T / 32) {  // rank-(je - jb) trailing update
      const int ri = i * (i + 1) / 2;
      double ui[SB];
#pragma unroll
      for (int t = 0; t < SB; ++t) ui[t] = jb + t < je ? a[ri + jb + t] * dd[jb + t] : 0.0;
      for (int k = je + lane; k <= i; k += 32) {
        const int rk = k * (k + 1) / 2;
        double x = a[ri + k];
#pragma unroll
        for (int t = 0; t < SB; ++t)
          if (jb + t < je) x -= ui[t] * a[rk + jb + t];
        a[ri + k] = x;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < np; e += SC_T) Lp[e] = a[e];
  for (int j = tid; j < M; j += SC_T) Lp[np + j] = di[j];
}

// x = L'^{-T} D^{-1} L'^{-1} r with k_chol_small's output, one warp (forward substitution
// with the unit L', the pivot scaling, backward substitution with L'^T)
constexpr int SS_T = 256;  // the whole CTA stages the factor into shared memory, warp 0 solves
__global__ void __launch_bounds__(SS_T) k_chol_small_solve(const double* __restrict__ Lp, int M,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ x, const int* done,
                                                           const int* Md) {
  if (Md) {
    M = *Md;
    if (M == 0) return;
  }
  extern __shared__ double sm[];
  double* L = sm;
  const int np = M * (M + 1) / 2;
  const double* dinv = L + np;
  double* y = sm + np + M;
  for (int e = threadIdx.x; e < np + M; e += SS_T) L[e] = Lp[e];
  for (int i = threadIdx.x; i < M; i += SS_T) y[i] = r[i];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int j = 0; j < M; ++j) {  // L' y = r, column-oriented
    const double yj = y[j];
    for (int i = j + 1 + lane; i < M; i += 32) y[i] -= L[i * (i + 1) / 2 + j] * yj;
    __syncwarp();
  }
  for (int i = lane; i < M; i += 32) y[i] *= dinv[i];
  __syncwarp();
  for (int j = M - 1; j >= 0; --j) {  // L'^T x = y, row j of L' holds column j of L'^T
    const int rj = j * (j + 1) / 2;
    const double xj = y[j];
    for (int i = lane; i < j; i += 32) y[i] -= L[rj + i] * xj;
    __syncwarp();
  }
  const bool skip = done && *(volatile const int*)done;
  if (!skip)
    for (int i = lane; i < M; i += 32) x[i] = y[i];
}

void coarse_solve_small(msb_ctx ctx, const Coarse& co, const double* rc, double* xc,
                        const int* done) {
  const int M = co.M;
  const size_t smem = ((size_t)M * (M + 1) / 2 + 2 * M) * sizeof(double);
  k_chol_small_solve<<<1, SS_T, smem, ctx->stream>>>(co.L, M, rc, xc, done, nullptr);
  count_launch();
}

// ---------------------------------------------------------------- mid-size SPD systems
// M_dyn in (SMALL_CHOL_M, 1024] (the dynamic stage's larger partitions, factored for one
// solve): a blocked right-looking LDL^T in ONE cooperative launch of persistent CTAs with
// grid barriers between its phases, instead of the recursion's ~50 dependent launches.
// Per panel of 32 columns: (1) one warp factors the 32 x 32 diagonal block in registers
// (lane i owns row i; the pivot rows reach the other lanes by shuffles); (2) every row below
// is forward-substituted with the unit block (u_i = the row's panel entries, L'_i = u_i D^-1;
// u kept in a scratch); (3) the trailing lower triangle is updated by 32 x 32 tiles,
// A_ik -= u_i . L'_k.  A (row-major, ld M) is overwritten by L' (strictly lower) and d (the
// diagonal); dinv = 1/d.  Pivot test as the other factorisations.
constexpr int CP_B = 32, CP_T2 = 256;

__device__ __forceinline__ void coop_grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// the 32 x 32 diagonal block at (p, p) (nb rows valid): unit L' and d in place, 1/d to dinv
__device__ __forceinline__ void coop_diag_block(double* __restrict__ A, int M, int p, int nb,
                                                double* __restrict__ dinv, double tol,
                                                int* __restrict__ singular) {
  const int i = threadIdx.x;  // one warp
  double row[CP_B];
#pragma unroll
  for (int k = 0; k < CP_B; ++k)
    row[k] = (i < nb && k <= i) ? A[(int64_t)(p + i) * M + p + k] : (k == i ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < CP_B; ++j) {
    double dj = __shfl_sync(0xffffffffu, row[j], j);
    if (j < nb && !(dj > tol)) {
      if (i == 0) *singular = 1;
      dj = 1.0;
      if (i == j) row[j] = 1.0;
    }
    const double rj = 1.0 / dj;
    const double u = i > j ? row[j] : 0.0;
    const double l = u * rj;
#pragma unroll
    for (int k = j + 1; k < CP_B; ++k) {
      const double lk = __shfl_sync(0xffffffffu, l, k);
      if (i >= k) row[k] -= u * lk;
    }
    if (i > j) row[j] = l;
  }
  if (i < nb) {
#pragma unroll
    for (int k = 0; k < CP_B; ++k)
      if (k <= i) A[(int64_t)(p + i) * M + p + k] = row[k];
    dinv[p + i] = 1.0 / row[i];
  }
}

__global__ void __launch_bounds__(CP_T2) k_ldl_coop(double* __restrict__ A, int M, double* __restrict__ U,
                                                    double* __restrict__ dinv,
                                                    const unsigned long long* amax_bits,
                                                    int* __restrict__ singular, unsigned* bar) {
  __shared__ double lb[CP_B][CP_B + 1];
  __shared__ double us[CP_B][CP_B + 1];
  __shared__ double di[CP_B];
  const double tol = 1e-14 * __longlong_as_double((long long)*amax_bits);
  unsigned phase = 0;
  if (blockIdx.x == 0 && threadIdx.x < 32) coop_diag_block(A, M, 0, min(CP_B, M), dinv, tol, singular);
  coop_grid_sync(bar, ++phase * gridDim.x);
  for (int p = 0; p < M; p += CP_B) {
    const int pe = min(p + CP_B, M), nb = pe - p;
    // (2) the rows below the block: forward substitution with the unit block, the inner
    // products split over four accumulators (independent FMA chains)
    for (int e = threadIdx.x; e < CP_B * CP_B; e += CP_T2) {
      const int r = e / CP_B, c = e % CP_B;
      lb[r][c] = (r < nb && c < r) ? A[(int64_t)(p + r) * M + p + c] : 0.0;
    }
    if (threadIdx.x < CP_B) di[threadIdx.x] = threadIdx.x < nb ? dinv[p + threadIdx.x] : 0.0;
    __syncthreads();
    for (int i = pe + blockIdx.x * CP_T2 + threadIdx.x; i < M; i += gridDim.x * CP_T2) {
      double v[CP_B];
#pragma unroll
      for (int t = 0; t < CP_B; ++t) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int q = 0; q + 3 < t; q += 4) {
          s0 += v[q] * lb[t][q];
          s1 += v[q + 1] * lb[t][q + 1];
          s2 += v[q + 2] * lb[t][q + 2];
          s3 += v[q + 3] * lb[t][q + 3];
        }
#pragma unroll
        for (int q = t & ~3; q < t; ++q) s0 += v[q] * lb[t][q];
        const double a = t < nb ? A[(int64_t)i * M + p + t] : 0.0;
        v[t] = a - ((s0 + s1) + (s2 + s3));
      }
#pragma unroll
      for (int t = 0; t < CP_B; ++t)
        if (t < nb) {
          U[(int64_t)i * CP_B + t] = v[t];
          A[(int64_t)i * M + p + t] = v[t] * di[t];
        }
    }
    coop_grid_sync(bar, ++phase * gridDim.x);
    // (3) the trailing lower triangle, 32 x 32 tiles; tile 0 (the next panel's diagonal
    // block) is CTA 0's first, which then factors that block at once (look-ahead: the next
    // panel's first phase overlaps the other CTAs' tiles, one barrier fewer per panel)
    const int nbk = (M - pe + CP_B - 1) / CP_B;
    const int ntile = nbk * (nbk + 1) / 2;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
      int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      while (I * (I + 1) / 2 > t) --I;
      const int K = t - I * (I + 1) / 2;
      const int i0 = pe + I * CP_B, k0 = pe + K * CP_B;
      __syncthreads();
      for (int e = threadIdx.x; e < CP_B * CP_B; e += CP_T2) {
        const int r = e / CP_B, c = e % CP_B;
        us[r][c] = (i0 + r < M && c < nb) ? U[(int64_t)(i0 + r) * CP_B + c] : 0.0;
        lb[r][c] = (k0 + r < M && c < nb) ? A[(int64_t)(k0 + r) * M + p + c] : 0.0;
      }
      __syncthreads();
      const int r = threadIdx.x / 8, c0 = threadIdx.x % 8;
      const int gi = i0 + r;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + 8 * q, gk = k0 + c;
        if (gi < M && gk < M && gk <= gi) {
          double x = A[(int64_t)gi * M + gk];
#pragma unroll
          for (int tt = 0; tt < CP_B; ++tt) x -= us[r][tt] * lb[c][tt];
          A[(int64_t)gi * M + gk] = x;
        }
      }
      if (t == 0) {  // CTA 0: the next diagonal block is final
        __syncthreads();
        if (threadIdx.x < 32) coop_diag_block(A, M, pe, min(CP_B, M - pe), dinv, tol, singular);
      }
    }
    coop_grid_sync(bar, ++phase * gridDim.x);
  }
}

// x = L'^{-T} D^{-1} L'^{-1} r with k_ldl_coop's output, one CTA of 1024 threads in panels of
// 32: the panel's triangle by one warp (shuffles), the rest of the vector by all threads
constexpr int CS_T = 1024;
__global__ void __launch_bounds__(CS_T) k_ldl_coop_solve(const double* __restrict__ A, int M,
                                                         const double* __restrict__ dinv,
                                                         const double* __restrict__ r,
                                                         double* __restrict__ x, const int* done) {
  __shared__ double y[1024];
  __shared__ double lb[CP_B][CP_B + 1];
  const int tid = threadIdx.x;
  if (tid < M) y[tid] = r[tid];
  for (int p = 0; p < M; p += CP_B) {  // L' y = r
    const int pe = min(p + CP_B, M), nb = pe - p;
    {
      const int rr = tid / CP_B, c = tid % CP_B;
      lb[rr][c] = (rr < nb && c < rr) ? A[(int64_t)(p + rr) * M + p + c] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double yl = tid < nb ? y[p + tid] : 0.0;
#pragma unroll
      for (int j = 0; j < CP_B; ++j) {
        const double yj = __shfl_sync(0xffffffffu, yl, j);
        if (tid > j) yl -= lb[tid][j] * yj;
      }
      if (tid < nb) y[p + tid] = yl;
    }
    __syncthreads();
    const int i = pe + tid;
    if (i < M) {
      double s = y[i];
#pragma unroll 8
      for (int t = 0; t < nb; ++t) s -= A[(int64_t)i * M + p + t] * y[p + t];
      y[i] = s;
    }
    __syncthreads();
  }
  if (tid < M) y[tid] *= dinv[tid];
  __syncthreads();
  for (int p = ((M - 1) / CP_B) * CP_B; p >= 0; p -= CP_B) {  // L'^T x = y
    const int pe = min(p + CP_B, M), nb = pe - p;
    {
      const int rr = tid / CP_B, c = tid % CP_B;
      lb[rr][c] = (rr < nb && c < rr) ? A[(int64_t)(p + rr) * M + p + c] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double yl = tid < nb ? y[p + tid] : 0.0;
#pragma unroll
      for (int j = CP_B - 1; j >= 0; --j) {
        const double xj = __shfl_sync(0xffffffffu, yl, j);
        if (tid < j) yl -= lb[j][tid] * xj;
      }
      if (tid < nb) y[p + tid] = yl;
    }
    __syncthreads();
    if (tid < p) {
      double s = y[tid];
#pragma unroll 8
      for (int t = 0; t < nb; ++t) s -= A[(int64_t)(p + t) * M + tid] * y[p + t];
      y[tid] = s;
    }
    __syncthreads();
  }
  const bool skip = done && *(volatile const int*)done;
  if (!skip && tid < M) x[tid] = y[tid];
}

void coarse_solve_coop(msb_ctx ctx, const Coarse& co, const double* rc, double* xc, const int* done) {
  k_ldl_coop_solve<<<1, CS_T, 0, ctx->stream>>>(co.L, co.M, co.tri_y, rc, xc, done);
  count_launch();
}

// The dynamic loop's graph-captured small path: the one-CTA factorisation of an M x M
// system (M <= SMALL_CHOL_M) with M read from the device (*Md; 0 = nothing to do), and its
// solve.  Launch shapes are those of M = SMALL_CHOL_M.
msb_status coarse_factor_small_gated(msb_ctx ctx, Coarse& co, const int* Md) {
  cudaStream_t s = ctx->stream;
  unsigned long long* amax = co.flags;
  int* sing = reinterpret_cast<int*>(co.flags + 1);
  static bool attr = false;
  const int mx = (int)(((size_t)SMALL_CHOL_M * (SMALL_CHOL_M + 1) / 2 + 2 * SMALL_CHOL_M) * sizeof(double));
  if (!attr) {
    MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_chol_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    attr = true;
  }
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.flags, 0, 16, s));
  k_absmax2<<<std::min<int64_t>(grid_for((int64_t)SMALL_CHOL_M * SMALL_CHOL_M, 256), 4 * ctx->sm_count),
              256, 0, s>>>(co.Ac, 0, amax, Md);
  MSB_LAUNCH_CHECK(ctx);
  k_chol_small<<<1, SC_T, mx, s>>>(co.Ac, 0, co.L, amax, sing, Md);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

void coarse_solve_small_gated(msb_ctx ctx, const Coarse& co, const double* rc, double* xc,
                              const int* done, const int* Md) {
  const size_t smem = ((size_t)SMALL_CHOL_M * (SMALL_CHOL_M + 1) / 2 + 2 * SMALL_CHOL_M) * sizeof(double);
  k_chol_small_solve<<<1, SS_T, smem, ctx->stream>>>(co.L, 0, rc, xc, done, Md);
  count_launch();
}

msb_status coarse_factor_dense(msb_ctx ctx, Coarse& co) {
  const int M = co.M;
  cudaStream_t s = ctx->stream;
  if (!co.flags) MSB_ALLOC(ctx, co.flags, unsigned long long, 2);
  unsigned long long* amax = co.flags;
  int* sing = reinterpret_cast<int*>(co.flags + 1);
  co.small = co.tri && M <= SMALL_CHOL_M;
  co.coop = co.tri && !co.small && M <= 1024;
  if (co.coop) {
    if (!co.L || !co.Ainv || !co.tri_y || co.cap < M)
      return set_error(ctx, MSB_EINVAL, "coarse_factor_dense: mid-size buffers");
    unsigned* bar = reinterpret_cast<unsigned*>(co.flags) + 3;  // flags[1] high word
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.flags, 0, 16, s));
    k_absmax2<<<std::min<int64_t>(grid_for((int64_t)M * M, 256), 4 * ctx->sm_count), 256, 0, s>>>(
        co.Ac, (int64_t)M * M, amax);
    MSB_LAUNCH_CHECK(ctx);
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(co.L, co.Ac, (size_t)M * M * sizeof(double), cudaMemcpyDeviceToDevice, s));
    const int G = std::min(ctx->sm_count, 128);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(CP_T2);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MSB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k_ldl_coop, co.L, M, co.Ainv, co.tri_y,
                                         (const unsigned long long*)amax, sing, bar));
    count_launch();
    int hs = 0;
    if (!co.defer_check) {
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, sing, 4, cudaMemcpyDeviceToHost, s));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    if (hs) {
      co.ready = false;
      return set_error(ctx, MSB_ESINGULAR, "singular coarse matrix: pivot <= 1e-14 max|A_c| (M=%d)", M);
    }
    co.ready = true;
    return MSB_OK;
  }
  if (co.small) {
    if (!co.L) MSB_ALLOC(ctx, co.L, double, (int64_t)co.cap * co.cap + co.cap);
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.flags, 0, 16, s));
    k_absmax2<<<std::min<int64_t>(grid_for((int64_t)M * M, 256), 4 * ctx->sm_count), 256, 0, s>>>(
        co.Ac, (int64_t)M * M, amax);
    MSB_LAUNCH_CHECK(ctx);
    static bool attr = false;
    if (!attr) {
      const int mx = (int)(((size_t)SMALL_CHOL_M * (SMALL_CHOL_M + 1) / 2 + 2 * SMALL_CHOL_M) * sizeof(double));
      MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      MSB_CUDA_TRY(ctx, cudaFuncSetAttribute(k_chol_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      attr = true;
    }
    k_chol_small<<<1, SC_T, ((size_t)M * (M + 1) / 2 + 2 * M) * sizeof(double), s>>>(co.Ac, M, co.L,
                                                                                   amax, sing, nullptr);
    MSB_LAUNCH_CHECK(ctx);
    int hs = 0;
    if (!co.defer_check) {
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, sing, 4, cudaMemcpyDeviceToHost, s));
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    if (hs) {
      co.ready = false;
      return set_error(ctx, MSB_ESINGULAR, "singular coarse matrix: pivot <= 1e-14 max|A_c| (M=%d)", M);
    }
    co.ready = true;
    return MSB_OK;
  }
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
  if (co.tri) {  // a single solve per factorisation: keep W = L^{-1} (co.Ainv), x = W^T (W r)
    co.ready = true;
    return MSB_OK;
  }
  // A_c^{-1} = W^T W: lower tiles with the K range restricted to the nonzeros of W,
  // written over the factor buffer (L is no longer needed), then mirrored; swap so
  // that co.Ainv holds the inverse and co.L the inverse factor W.
  if ((rc = lauum(ctx, Wb, F, M, M))) return rc;
  dim3 g((M + 31) / 32, (M + 31) / 32);
  k_mirror_lower<<<g, dim3(32, 32), 0, s>>>(F, M);
  MSB_LAUNCH_CHECK(ctx);
  std::swap(co.L, co.Ainv);
  if ((rc = coarse_pack_symmetric(ctx, co))) return rc;
  co.ready = true;
  return MSB_OK;
}

}  // namespace msb
