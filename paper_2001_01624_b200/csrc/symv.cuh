// Symmetric GEMV over the packed lower triangle of A_c^{-1} (coarse.cu): the per-tile
// and per-output-block device bodies, shared by the standalone kernels and the
// persistent cycle kernel (cycle.cu).  256 threads per CTA.  CG: read r_c and the tile
// partials with ld.global.cg (they are rewritten every iteration inside one persistent
// launch, where no kernel boundary invalidates L1).
#pragma once

namespace msb {

constexpr int ST = 64;

template <bool CG>
__device__ __forceinline__ double ld_mut(const double* p) {
  return CG ? __ldcg(p) : *p;
}

__device__ __forceinline__ void symv_tile_rc(int64_t t, int& bi, int& bj) {
  bi = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while ((int64_t)bi * (bi + 1) / 2 > t) --bi;
  bj = (int)(t - (int64_t)bi * (bi + 1) / 2);
}

// tile t: row contribution X_t r_bj and (off-diagonal) column contribution X_t^T r_bi
// into part[t][0..63], part[t][64..127].  Uses 8.5 KB of static shared memory.
// map / roff (batched solves, coarse_schur.cu): matrix row r reads rc[map[roff + r]]
// (map NULL: rc[roff + r]).
template <bool CG>
__device__ __forceinline__ void symv_tile_body(const double* __restrict__ Xp, int M,
                                               const double* rc, double* __restrict__ part,
                                               int64_t t, const int32_t* __restrict__ map = nullptr,
                                               int roff = 0) {
  int bi, bj;
  symv_tile_rc(t, bi, bj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // columns 2tx, 2tx+1; rows ty + 8u
  const double2* tile = reinterpret_cast<const double2*>(Xp + t * ST * ST);
  double2 a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = __ldcs(tile + (ty + 8 * u) * (ST / 2) + tx);
  pdl_wait();  // the tile is an input: loaded while the restriction drains; r_c after the wait
  pdl_trigger();
  auto at = [&](int r) -> int { return map ? map[roff + r] : roff + r; };
  const int cj = bj * ST + 2 * tx;
  const double r0 = cj < M ? ld_mut<CG>(rc + at(cj)) : 0.0;
  const double r1 = cj + 1 < M ? ld_mut<CG>(rc + at(cj + 1)) : 0.0;
  double ri[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int row = bi * ST + ty + 8 * u;
    ri[u] = row < M ? ld_mut<CG>(rc + at(row)) : 0.0;
  }
  __shared__ double rows_sh[ST];
  __shared__ double cols_sh[8][ST];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double v = a[u].x * r0 + a[u].y * r1;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (tx == 0) rows_sh[ty + 8 * u] = v;
  }
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    c0 += a[u].x * ri[u];
    c1 += a[u].y * ri[u];
  }
  cols_sh[ty][2 * tx] = c0;
  cols_sh[ty][2 * tx + 1] = c1;
  __syncthreads();
  double* pt = part + t * 2 * ST;
  if (threadIdx.x < ST) {
    pt[threadIdx.x] = rows_sh[threadIdx.x];
  } else if (threadIdx.x < 2 * ST) {
    const int c = threadIdx.x - ST;
    double v = 0.0;
    if (bi != bj)
      for (int g = 0; g < 8; ++g) v += cols_sh[g][c];
    pt[ST + c] = v;
  }
  __syncthreads();  // shared arrays are reused by the next unit of a persistent CTA
}

// output block b: xc[b] = sum_{j <= b} row part of (b, j) + sum_{k > b} column part of (k, b),
// G = blockDim / 64 thread groups of 64 taking every G-th contribution (the persistent
// kernel runs 4 groups, k_symv_reduce 16: a 4-deep instead of 14-deep chain of dependent
// L2 loads per thread at M = 3,400), then a fixed-order combine of the groups
// omap / roff: output row r goes to xc[omap[roff + r]] (omap NULL: xc[roff + r])
template <bool CG>
__device__ __forceinline__ void symv_reduce_body(const double* part, int M, int ntb,
                                                 double* __restrict__ xc, int b, bool skip,
                                                 const int32_t* __restrict__ omap = nullptr,
                                                 int roff = 0) {
  const int i = threadIdx.x & (ST - 1), g = threadIdx.x / ST, G = blockDim.x / ST;
  const int64_t rowbase = (int64_t)b * (b + 1) / 2;
  double v = 0.0;
  // batches of 8 independent loads in flight, then summed in order (the same order as one
  // load at a time: deterministic, identical result)
  for (int e0 = g; e0 < ntb; e0 += 8 * G) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * G;
      const int64_t off = e <= b ? (rowbase + e) * 2 * ST + i
                                 : ((int64_t)e * (e + 1) / 2 + b) * 2 * ST + ST + i;
      t[u] = e < ntb ? ld_mut<CG>(part + off) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * G < ntb) v += t[u];
  }
  __shared__ double sh[16][ST];
  sh[g][i] = v;
  __syncthreads();
  if (g == 0) {
    double tot = 0.0;
    for (int q = 0; q < G; ++q) tot += sh[q][i];
    const int row = b * ST + i;
    if (row < M && !skip) xc[omap ? omap[roff + row] : roff + row] = tot;
  }
  __syncthreads();
}

}  // namespace msb
