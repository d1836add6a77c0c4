// Rows a4 (Galerkin A_c = P^T A P, G6) and a5 (coarse factor + solve, G7).
//
// RAP: A = Σ_f T_f (e_i - e_l)(e_i - e_l)^T + A^T_00 e_0 e_0^T, so
//   A_c = Σ_f T_f g_f g_f^T + A^T_00 (P_0.)^T P_0.,   g_f = (P_i. - P_l.)^T,
// one thread per cell (its +x/+y/+z faces), g over the union of the two rows'
// columns (<= 2W entries), fp64 atomics into the dense row-major A_c.
//
// Factor + explicit inverse: coarse_factor.cu.  Every coarse solve in the cycle is a
// single bandwidth-bound GEMV (M^2 doubles) instead of two latency-bound triangular
// solves.
#include <algorithm>
#include <cstdlib>

#include <climits>
#include <vector>

#include "internal.cuh"
#include "symv.cuh"
#include "fx.cuh"

namespace msb {


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

// ---------------------------------------------------------------- deterministic constant-basis RAP
// For a constant basis (explicit level, one slot: the dynamic, indicator-halo-0 and
// constant levels) A_c = sum over faces between blocks J != K of T (e_J - e_K)(e_J - e_K)^T
// (+ the gauge term).  The entries are accumulated EXACTLY in 128-bit fixed point with
// 64-bit integer atomics (carry into the high word), so the result does not depend on the
// order in which the atomics land: the same inputs give the same A_c bits on every run
// (the dynamic stage is rebuilt every iteration and its Δp bins amplify any run-to-run
// rounding noise).  Scale 2^F with F = 90 - ilogb(max T): every entry sum stays below
// 2^126, contributions are exact down to 2^-50 relative to max T.
__global__ void k_absmax_t(const double* __restrict__ T, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(T[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Constant basis (W = 1): A_c = P^T A P has (A_c)_JK = -sum of T_f over the faces between
// blocks J != K, and (A_c)_JJ = sum over J's outer faces (+ the gauge term of cell 0).
// Only the magnitude sum of each unordered pair {J, K} is accumulated, into the lower entry
// (max, min); the conversion (k_fx_const_to_double) negates it into both off-diagonal
// entries and forms each diagonal as its row's pair sums — exact integer sums, so the
// result is the same as accumulating all four entries per face, and order-independent.
// Faces along a block boundary hit the same pair from consecutive lanes: runs of equal
// pairs within a warp are summed first (segmented shuffle scan, exact 128-bit adds) and the
// run's last lane issues the two atomics.  The gauge term goes to the diagonal slot.
__global__ void __launch_bounds__(256) k_rap_const_det(const int32_t* __restrict__ col, Grid3 g, int M,
                                                       const double* __restrict__ Tx,
                                                       const double* __restrict__ Ty,
                                                       const double* __restrict__ Tz,
                                                       const unsigned long long* __restrict__ tmax_bits,
                                                       unsigned long long* __restrict__ acc,
                                                       const int* Md) {
  if (Md) {  // M from the device (the dynamic loop's graph-captured small path; 0 = skip)
    M = *Md;
    if (M == 0) return;
  }
  const unsigned FULL = 0xffffffffu, NONE = 0xffffffffu;
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool in = c < N;
  int i = 0, j = 0, k = 0;
  if (in) g3_coords(g, c, i, j, k);
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  const int J = in ? col[c] : -1;
  double Tf[3] = {0.0, 0.0, 0.0};
  if (in) {
    Tf[0] = i < g.nx - 1 ? Tx[c] : 0.0;
    Tf[1] = j < g.ny - 1 ? Ty[c] : 0.0;
    Tf[2] = k < g.nz - 1 ? Tz[c] : 0.0;
  }
  const int nb[3] = {c + 1, c + g.nx, c + g.nxy};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    unsigned key = NONE;
    unsigned long long lo = 0, hi = 0;
    if (in && Tf[d] != 0.0) {
      const int K = col[nb[d]];
      if (K != J) {
        key = (unsigned)(J > K ? J * M + K : K * M + J);
        fx_split(Tf[d], F, lo, hi);
      }
    }
    const unsigned prev = __shfl_up_sync(FULL, key, 1);
    const unsigned next = __shfl_down_sync(FULL, key, 1);
    const unsigned heads = __ballot_sync(FULL, lane == 0 || prev != key);
    const int start = 31 - __clz(heads & (FULL >> (31 - lane)));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long ylo = __shfl_up_sync(FULL, lo, o);
      const unsigned long long yhi = __shfl_up_sync(FULL, hi, o);
      if (lane - o >= start) add128(lo, hi, ylo, yhi);
    }
    if (key != NONE && (lane == 31 || next != key)) {
      unsigned long long* e = acc + 2 * (size_t)key;
      const unsigned long long old = atomicAdd(e, lo);
      atomicAdd(e + 1, hi + (old + lo < old ? 1ull : 0ull));
    }
  }
  if (c == 0) fx_add(acc + 2 * ((size_t)J * M + J), Tf[0] + 0.0 + Tf[1] + 0.0 + Tf[2] + 0.0, F);
}

// One CTA per row a of the constant-basis A_c: off-diagonal entries from the pair sums,
// the diagonal as their exact 128-bit total plus the gauge slot.
__global__ void __launch_bounds__(256) k_fx_const_to_double(const unsigned long long* __restrict__ acc,
                                                            int M,
                                                            const unsigned long long* __restrict__ tmax_bits,
                                                            double* __restrict__ Ac, const int* Md) {
  if (Md) M = *Md;
  const int a = blockIdx.x;
  if (a >= M) return;
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  unsigned long long slo = 0, shi = 0;
  for (int b = threadIdx.x; b < M; b += blockDim.x) {
    if (b == a) continue;
    const size_t e = a > b ? (size_t)a * M + b : (size_t)b * M + a;
    const unsigned long long lo = acc[2 * e], hi = acc[2 * e + 1];
    Ac[(size_t)a * M + b] = -fx_value(lo, hi, F);
    add128(slo, shi, lo, hi);
  }
  if (threadIdx.x == 0) add128(slo, shi, acc[2 * ((size_t)a * M + a)], acc[2 * ((size_t)a * M + a) + 1]);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ylo = __shfl_xor_sync(0xffffffffu, slo, o);
    const unsigned long long yhi = __shfl_xor_sync(0xffffffffu, shi, o);
    add128(slo, shi, ylo, yhi);
  }
  __shared__ unsigned long long wl[8], wh[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wl[w] = slo;
    wh[w] = shi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long lo = wl[0], hi = wh[0];
    for (int v = 1; v < (int)(blockDim.x >> 5); ++v) add128(lo, hi, wl[v], wh[v]);
    Ac[(size_t)a * M + a] = fx_value(lo, hi, F);
  }
}

__global__ void k_fx_to_double(const unsigned long long* __restrict__ acc, int64_t n,
                               const unsigned long long* __restrict__ tmax_bits,
                               double* __restrict__ Ac) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  // the 128-bit integer hi 2^64 + lo, rounded to double (deterministic), scaled back
  Ac[e] = fx_value(acc[2 * e], acc[2 * e + 1], F);
}

// Rows of P summing to one (MsRSB's partition of unity) make sum_b (A_c)_ab over the face
// terms vanish, so k_rap<true, true> accumulates only the lower off-diagonal entries (half
// the atomics, and none on the diagonal — the entries every face of a support hits) and
// the diagonal is minus the row's off-diagonal total plus the diagonal slot (the gauge
// term's correction).  Equal to the direct sum up to the rounding of P's row sums.
__global__ void __launch_bounds__(256) k_fx_sym_to_double(const unsigned long long* __restrict__ acc,
                                                          int M,
                                                          const unsigned long long* __restrict__ tmax_bits,
                                                          double* __restrict__ Ac) {
  const int a = blockIdx.x;
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  unsigned long long slo = 0, shi = 0;
  for (int b = threadIdx.x; b < M; b += blockDim.x) {
    if (b == a) continue;
    const size_t e = a > b ? (size_t)a * M + b : (size_t)b * M + a;
    const unsigned long long lo = acc[2 * e], hi = acc[2 * e + 1];
    Ac[(size_t)a * M + b] = fx_value(lo, hi, F);
    add128(slo, shi, lo, hi);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ylo = __shfl_xor_sync(0xffffffffu, slo, o);
    const unsigned long long yhi = __shfl_xor_sync(0xffffffffu, shi, o);
    add128(slo, shi, ylo, yhi);
  }
  __shared__ unsigned long long wl[8], wh[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wl[w] = slo;
    wh[w] = shi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long lo = wl[0], hi = wh[0];
    for (int v = 1; v < (int)(blockDim.x >> 5); ++v) add128(lo, hi, wl[v], wh[v]);
    // diagonal = slot(a, a) - row total (two's complement)
    const unsigned long long nlo = ~lo + 1ull, nhi = ~hi + (nlo == 0ull ? 1ull : 0ull);
    unsigned long long dlo = acc[2 * ((size_t)a * M + a)], dhi = acc[2 * ((size_t)a * M + a) + 1];
    add128(dlo, dhi, nlo, nhi);
    Ac[(size_t)a * M + a] = fx_value(dlo, dhi, F);
  }
}

// FX: accumulate into the 128-bit fixed-point buffer (deterministic, see above) instead of
// fp64 atomics; |T g_a g_b| <= max T because P entries lie in [0, 1]
constexpr int ELLW = 125, ELLC = 62;  // box-stencil slots per row, centre slot

// ELL conversions, one warp per row a of the box stencil (Cartesian levels).  The
// neighbour b of slot d is a + offset(d) when its block coordinates stay in range.
__device__ __forceinline__ int ell_nb(int a, int d, int n0, int n1, int n2) {
  const int ax = a % n0, ay = (a / n0) % n1, az = a / (n0 * n1);
  const int bx = ax + d % 5 - 2, by = ay + (d / 5) % 5 - 2, bz = az + d / 25 - 2;
  if (bx < 0 || bx >= n0 || by < 0 || by >= n1 || bz < 0 || bz >= n2) return -1;
  return bx + n0 * (by + n1 * bz);
}

// SYM (partition-of-unity rows): off-diagonal (a, b) lives in the lower entry — row
// max(a, b) at the slot of min(a, b) — and the diagonal is the centre slot minus the row's
// exact off-diagonal total (as k_fx_sym_to_double).
__global__ void __launch_bounds__(256) k_fx_ell_sym(const unsigned long long* __restrict__ acc,
                                                    int M, int n0, int n1, int n2,
                                                    const unsigned long long* __restrict__ tmax_bits,
                                                    double* __restrict__ Aell) {
  const int a = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= M) return;  // warp-uniform
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  unsigned long long slo = 0, shi = 0;
  for (int d = lane; d < ELLW; d += 32) {
    double v = 0.0;
    const int b = d == ELLC ? -1 : ell_nb(a, d, n0, n1, n2);
    if (b >= 0) {
      const size_t e = b < a ? (size_t)a * ELLW + d : (size_t)b * ELLW + (ELLW - 1 - d);
      const unsigned long long lo = acc[2 * e], hi = acc[2 * e + 1];
      v = fx_value(lo, hi, F);
      add128(slo, shi, lo, hi);
    }
    if (d != ELLC) Aell[(size_t)a * ELLW + d] = v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ylo = __shfl_xor_sync(0xffffffffu, slo, o);
    const unsigned long long yhi = __shfl_xor_sync(0xffffffffu, shi, o);
    add128(slo, shi, ylo, yhi);
  }
  if (lane == 0) {
    const unsigned long long nlo = ~slo + 1ull, nhi = ~shi + (nlo == 0ull ? 1ull : 0ull);
    unsigned long long dlo = acc[2 * ((size_t)a * ELLW + ELLC)],
                       dhi = acc[2 * ((size_t)a * ELLW + ELLC) + 1];
    add128(dlo, dhi, nlo, nhi);
    Aell[(size_t)a * ELLW + ELLC] = fx_value(dlo, dhi, F);
  }
}

// full accumulation (imported P): every entry (a, b) was summed at row a
__global__ void k_fx_ell_full(const unsigned long long* __restrict__ acc, int M, int n0, int n1,
                              int n2, const unsigned long long* __restrict__ tmax_bits,
                              double* __restrict__ Aell) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * ELLW) return;
  const int a = (int)(e / ELLW), d = (int)(e - (int64_t)a * ELLW);
  const int F = 90 - ilogb(__longlong_as_double((long long)*tmax_bits));
  const bool ok = d == ELLC || ell_nb(a, d, n0, n1, n2) >= 0;
  Aell[e] = ok ? fx_value(acc[2 * e], acc[2 * e + 1], F) : 0.0;
}

// dense row-major A_c (M x M, zero-filled beforehand) from the box stencil
__global__ void k_ell_to_dense(const double* __restrict__ Aell, int M, int n0, int n1, int n2,
                               double* __restrict__ Ac) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * ELLW) return;
  const int a = (int)(e / ELLW), d = (int)(e - (int64_t)a * ELLW);
  const int b = d == ELLC ? a : ell_nb(a, d, n0, n1, n2);
  if (b >= 0) Ac[(int64_t)a * M + b] = Aell[e];
}

// ELL (Cartesian levels): the accumulator is the 125-slot box stencil of each row,
// entry (a, b) at acc[a * 125 + ell_slot(a, b)] (|b_x - a_x|, |b_y - a_y|, |b_z - a_z| <= 2:
// open-box supports reach at most the second neighbour block, coarse.cu header); an entry
// outside the box sets bad[0] (never expected).
__device__ __forceinline__ int64_t ell_at(const msb_level_s& L, int a, int b, int* bad) {
  const int n0 = L.nb[0], n1 = L.nb[1];
  const int ax = a % n0, ay = (a / n0) % n1, az = a / (n0 * n1);
  const int bx = b % n0, by = (b / n0) % n1, bz = b / (n0 * n1);
  const int dx = bx - ax + 2, dy = by - ay + 2, dz = bz - az + 2;
  if ((unsigned)dx > 4u || (unsigned)dy > 4u || (unsigned)dz > 4u) {
    atomicOr(bad, 1);
    return (int64_t)a * ELLW + ELLC;
  }
  return (int64_t)a * ELLW + dx + 5 * dy + 25 * dz;
}

template <bool FX, bool SYM, bool ELL = false>
__global__ void k_rap(const msb_level_s L, const double* __restrict__ P, const double* __restrict__ Tx,
                      const double* __restrict__ Ty, const double* __restrict__ Tz,
                      double* __restrict__ Ac, unsigned long long* __restrict__ acc,
                      const unsigned long long* __restrict__ tmax_bits, int* bad = nullptr) {
  const int F = FX ? 90 - ilogb(__longlong_as_double((long long)*tmax_bits)) : 0;
  int64_t N = L.N;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int M = L.M;
  int64_t sxy = (int64_t)L.nx * L.ny;
  // 32-bit coordinates (msb_build_tpfa bounds 3N < 2^31): 64-bit division is an
  // emulated ~100-instruction sequence and dominated this kernel (362 us per dynamic-stage
  // assembly on config 3)
  const int c32 = (int)c, nxy32 = L.nx * L.ny;
  const int k = c32 / nxy32, rem = c32 - k * nxy32;
  const int j = rem / L.nx, i = rem - j * L.nx;
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
        if (FX && SYM) {
          // symmetric and row-sum-free: one add per unordered pair into its lower entry;
          // the diagonal is formed from the row in k_fx_sym_to_double
          if (gc[a] > gc[b])
            fx_add(acc + 2 * (ELL ? ell_at(L, gc[a], gc[b], bad) : (int64_t)gc[a] * M + gc[b]),
                   ta * gv[b], F);
        } else if (FX) {
          fx_add(acc + 2 * (ELL ? ell_at(L, gc[a], gc[b], bad) : (int64_t)gc[a] * M + gc[b]),
                 ta * gv[b], F);
        } else {
          atomicAdd(Ac + (int64_t)gc[a] * M + gc[b], ta * gv[b]);
        }
      }
    }
  }
  if (c == 0) {  // gauge: A_00 doubled adds A^T_00 (P_0.)^T P_0.
    double d0 = Tf[0] + 0.0 + Tf[1] + 0.0 + Tf[2] + 0.0;
    for (int a = 0; a < nc; ++a) {
      if (FX && SYM) {
        // off-diagonal gauge terms join the pair sums; the diagonal slot takes the gauge
        // diagonal plus the row's gauge off-diagonals (same integers), which the
        // conversion's row sum removes again
        unsigned long long dlo, dhi;
        fx_of(d0 * cv[a] * cv[a], F, dlo, dhi);
        for (int b = 0; b < nc; ++b) {
          if (b == a) continue;
          unsigned long long lo, hi;
          fx_of(d0 * cv[a] * cv[b], F, lo, hi);
          const unsigned long long s2 = dlo + lo;
          dhi += hi + (s2 < dlo ? 1ull : 0ull);
          dlo = s2;
          if (cc[a] > cc[b])
            fx_add_raw(acc + 2 * (ELL ? ell_at(L, cc[a], cc[b], bad) : (int64_t)cc[a] * M + cc[b]),
                       lo, hi);
        }
        fx_add_raw(acc + 2 * (ELL ? (int64_t)cc[a] * ELLW + ELLC : (int64_t)cc[a] * M + cc[a]), dlo,
                   dhi);
      } else {
        for (int b = 0; b < nc; ++b) {
          if (FX)
            fx_add(acc + 2 * (ELL ? ell_at(L, cc[a], cc[b], bad) : (int64_t)cc[a] * M + cc[b]),
                   d0 * cv[a] * cv[b], F);
          else atomicAdd(Ac + (int64_t)cc[a] * M + cc[b], d0 * cv[a] * cv[b]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- symmetric GEMV (SYMV)
// A_c^{-1} is symmetric, so the coarse solve reads only its lower triangle: 64 x 64
// tiles (bi >= bj) packed contiguously, tile t = bi(bi+1)/2 + bj, zero-padded at the
// edge.  k_symv_tiles: one CTA per tile loads the whole tile at once (8 double2 per
// thread) and produces both its row contribution X_t r_bj (for output block bi) and,
// off the diagonal, its column contribution X_t^T r_bi (for block bj) into per-tile
// partial slots; k_symv_reduce sums each output block's slots in a fixed order
// (deterministic).  HBM bytes per solve: 4 M (M + 64) instead of 8 M^2.

__global__ void k_pack_lower(const double* __restrict__ X, int M, int ntb, double* __restrict__ Xp) {
  const int64_t t = blockIdx.x;  // tile index
  // invert t = bi(bi+1)/2 + bj
  int bi = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while ((int64_t)bi * (bi + 1) / 2 > t) --bi;
  const int bj = (int)(t - (int64_t)bi * (bi + 1) / 2);
  double* dst = Xp + t * ST * ST;
  for (int e = threadIdx.x; e < ST * ST; e += blockDim.x) {
    const int r = bi * ST + e / ST, c = bj * ST + e % ST;
    dst[e] = (r < M && c < M) ? X[(int64_t)r * M + c] : 0.0;
  }
}

constexpr int SYMV_T = 256;  // threads per tile: 8 double2 of the tile per thread

// 5 CTAs per SM (48 registers): config 2's 1,485 tiles are two resident waves instead of 2.5
__global__ void __launch_bounds__(SYMV_T, 5) k_symv_tiles(const double* __restrict__ Xp, int M,
                                                       const double* __restrict__ rc,
                                                       double* __restrict__ part) {
  symv_tile_body<false>(Xp, M, rc, part, blockIdx.x);
}

__global__ void __launch_bounds__(16 * ST) k_symv_reduce(const double* __restrict__ part, int M,
                                                        int ntb, double* __restrict__ xc,
                                                        const int* done) {
  pdl_wait();
  pdl_trigger();
  const bool skip = done && *(volatile const int*)done;
  symv_reduce_body<false>(part, M, ntb, xc, blockIdx.x, skip);
}

// batched form (several packed matrices, vector rows through an optional index map):
// one CTA per tile descriptor, one CTA per output-block descriptor
__global__ void __launch_bounds__(SYMV_T) k_symv_tiles_b(const SymvTile* __restrict__ td,
                                                         const double* __restrict__ Xp,
                                                         const double* __restrict__ vec,
                                                         const int32_t* __restrict__ map,
                                                         double* __restrict__ part) {
  const SymvTile d = td[blockIdx.x];
  symv_tile_body<false>(Xp + d.tile_base * ST * ST, d.M, vec, part + d.tile_base * 2 * ST, d.t,
                        map, d.roff);
}

__global__ void __launch_bounds__(16 * ST) k_symv_reduce_b(const SymvRow* __restrict__ rd,
                                                          const double* __restrict__ part,
                                                          double* __restrict__ out,
                                                          const int32_t* __restrict__ omap,
                                                          const int* done) {
  pdl_wait();
  pdl_trigger();
  const bool skip = done && *(volatile const int*)done;
  const SymvRow d = rd[blockIdx.x];
  symv_reduce_body<false>(part + d.tile_base * 2 * ST, d.M, d.ntb, out, d.b, skip, omap, d.roff);
}

void symv_batched(msb_ctx ctx, const SymvTile* td, int ntile, const SymvRow* rd, int nrow,
                  const double* Xp, const double* vec, const int32_t* map, double* part,
                  double* out, const int32_t* omap, const int* done) {
  launch_ex(k_symv_tiles_b, dim3(ntile), dim3(SYMV_T), 0, ctx->stream, kPDL, 1, td, Xp, vec, map,
            part);
  launch_ex(k_symv_reduce_b, dim3(nrow), dim3(16 * ST), 0, ctx->stream, kPDL, 1, rd, part, out, omap,
            done);
  count_launch();
  count_launch();
}

// x = W^T (W r) with the lower-triangular inverse factor W (row-major, ld M): one warp
// per row of W r, one warp per column of W^T y (lane-strided, fixed shuffle tree)
__global__ void __launch_bounds__(256) k_trmv_lower(const double* __restrict__ W, int M,
                                                    const double* __restrict__ r,
                                                    double* __restrict__ y) {
  const int i = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= M) return;
  double v = 0.0;
  for (int j = lane; j <= i; j += 32) v = fma(W[(int64_t)i * M + j], r[j], v);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) y[i] = v;
}

__global__ void __launch_bounds__(256) k_trmv_lower_t(const double* __restrict__ W, int M,
                                                      const double* __restrict__ y,
                                                      double* __restrict__ x, const int* done) {
  const int j = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= M) return;
  const bool skip = done && *(volatile const int*)done;
  double v = 0.0;
  for (int i = j + lane; i < M; i += 32) v = fma(W[(int64_t)i * M + j], y[i], v);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0 && !skip) x[j] = v;
}

void coarse_solve(msb_ctx ctx, const Coarse& co, const double* rc, double* xc, const int* done) {
  if (co.tri && co.small) {
    coarse_solve_small(ctx, co, rc, xc, done);
    return;
  }
  if (co.tri && co.coop) {
    coarse_solve_coop(ctx, co, rc, xc, done);
    return;
  }
  if (co.tri) {
    const unsigned g = grid_for((int64_t)co.M * 32, 256);
    k_trmv_lower<<<g, 256, 0, ctx->stream>>>(co.Ainv, co.M, rc, co.tri_y);
    k_trmv_lower_t<<<g, 256, 0, ctx->stream>>>(co.Ainv, co.M, co.tri_y, xc, done);
    count_launch();
    count_launch();
    return;
  }
  if (co.kind == 1) {
    coarse_schur_solve(ctx, co, rc, xc, done);
    return;
  }
  coarse_solve_dense(ctx, co, rc, xc, done);
}

msb_status coarse_pack_symmetric(msb_ctx ctx, Coarse& co) {
  const int M = co.M;
  const int ntb = (M + ST - 1) / ST;
  const int64_t nt = (int64_t)ntb * (ntb + 1) / 2;
  if (co.xp_cap < nt) {
    dfree(ctx, co.Xp);
    dfree(ctx, co.part);
    MSB_ALLOC(ctx, co.Xp, double, nt * ST * ST);
    MSB_ALLOC(ctx, co.part, double, nt * 2 * ST);
    co.xp_cap = nt;
  }
  co.ntb = ntb;
  k_pack_lower<<<(unsigned)nt, 256, 0, ctx->stream>>>(co.Ainv, M, ntb, co.Xp);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

void coarse_solve_dense(msb_ctx ctx, const Coarse& co, const double* rc, double* xc,
                        const int* done) {
  const int64_t nt = (int64_t)co.ntb * (co.ntb + 1) / 2;
  launch_ex(k_symv_tiles, dim3((unsigned)nt), dim3(SYMV_T), 0, ctx->stream, kPDL, 1, co.Xp, co.M,
            rc, co.part);
  launch_ex(k_symv_reduce, dim3(co.ntb), dim3(16 * ST), 0, ctx->stream, kPDL, 1, co.part, co.M,
            co.ntb, xc, done);
  count_launch();
  count_launch();
}

// Cartesian levels: exact 128-bit fixed-point accumulation into the box stencil (16 B x 125
// per row: 40 MB at M = 20,000), converted to co.Aell; then the dense explicit inverse for
// M <= SCHUR_MIN_M, else the Schur-complement solver (coarse_schur.cu).
constexpr int SCHUR_MIN_M = 4096;

static msb_status ensure_dense(msb_ctx ctx, Coarse& co, int M) {
  if (co.cap >= M) return MSB_OK;
  dfree(ctx, co.Ac);
  dfree(ctx, co.L);
  dfree(ctx, co.Ainv);
  co.Ac = co.L = co.Ainv = nullptr;
  co.cap = 0;
  MSB_ALLOC(ctx, co.Ac, double, (int64_t)M * M);
  MSB_ALLOC(ctx, co.L, double, (int64_t)M * M + M);  // + the small path's pivot reciprocals
  MSB_ALLOC(ctx, co.Ainv, double, (int64_t)M * M);
  if (co.tri) {
    dfree(ctx, co.tri_y);
    co.tri_y = nullptr;
    MSB_ALLOC(ctx, co.tri_y, double, M);
  }
  co.cap = M;
  return MSB_OK;
}

static msb_status coarse_assemble_cart(msb_ctx ctx, msb_level L, msb_op op) {
  const int M = L->M;
  Coarse& co = L->co;
  cudaStream_t st = ctx->stream;
  co.M = M;
  co.ready = false;
  for (int a = 0; a < 3; ++a) co.nb[a] = L->nb[a];
  const size_t n = (size_t)M * ELLW;
  if (co.acc_cap < n) {
    dfree(ctx, co.acc);
    co.acc = nullptr;
    co.acc_cap = 0;
    MSB_ALLOC(ctx, co.acc, unsigned long long, 2 * n + 2);
    co.acc_cap = n;
  }
  if (co.ell_cap < M) {
    dfree(ctx, co.Aell);
    co.Aell = nullptr;
    co.ell_cap = 0;
    MSB_ALLOC(ctx, co.Aell, double, n);
    co.ell_cap = M;
  }
  int* bad = reinterpret_cast<int*>(co.acc + 2 * n + 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.acc, 0, (2 * n + 2) * sizeof(unsigned long long), st));
  const unsigned long long* tmax_c = nullptr;
  if (msb_status r0 = op_tmax(ctx, op, &tmax_c)) return r0;
  unsigned long long* tmax = const_cast<unsigned long long*>(tmax_c);
  if (L->unity)
    k_rap<true, true, true><<<grid_for(L->N, 128), 128, 0, st>>>(*L, L->P[L->cur], op->Tx, op->Ty,
                                                                op->Tz, nullptr, co.acc, tmax, bad);
  else
    k_rap<true, false, true><<<grid_for(L->N, 128), 128, 0, st>>>(*L, L->P[L->cur], op->Tx, op->Ty,
                                                                 op->Tz, nullptr, co.acc, tmax, bad);
  MSB_LAUNCH_CHECK(ctx);
  if (L->unity)
    k_fx_ell_sym<<<grid_for((int64_t)M * 32, 256), 256, 0, st>>>(co.acc, M, L->nb[0], L->nb[1],
                                                                 L->nb[2], tmax, co.Aell);
  else
    k_fx_ell_full<<<grid_for((int64_t)n, 256), 256, 0, st>>>(co.acc, M, L->nb[0], L->nb[1],
                                                             L->nb[2], tmax, co.Aell);
  MSB_LAUNCH_CHECK(ctx);
  int hbad = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (hbad)
    return set_error(ctx, MSB_EINVAL, "coarse coupling beyond the second neighbour block");
  if (M > SCHUR_MIN_M) {
    coarse_schur_free(ctx, co);
    msb_status rc = coarse_schur_setup(ctx, co, *L);
    if (rc == MSB_OK) {
      co.kind = 1;
      co.ready = true;
      return MSB_OK;
    }
    if (rc != MSB_EINVAL) return rc;  // EINVAL: no useful split of this coarse grid
    ctx->err[0] = 0;
  }
  co.kind = 0;
  msb_status rc = ensure_dense(ctx, co, M);
  if (rc) return rc;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.Ac, 0, (size_t)M * M * sizeof(double), st));
  k_ell_to_dense<<<grid_for((int64_t)n, 256), 256, 0, st>>>(co.Aell, M, L->nb[0], L->nb[1],
                                                           L->nb[2], co.Ac);
  MSB_LAUNCH_CHECK(ctx);
  return coarse_factor_dense(ctx, co);
}

msb_status coarse_assemble(msb_ctx ctx, msb_level L, msb_op op) {
  if (L->kind == 0) return coarse_assemble_cart(ctx, L, op);
  return coarse_assemble_dense(ctx, L, op);
}

msb_status op_tmax(msb_ctx ctx, msb_op op, const unsigned long long** out) {
  if (!op->tmax) MSB_ALLOC(ctx, op->tmax, unsigned long long, 1);
  if (!op->tmax_valid) {
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(op->tmax, 0, 8, ctx->stream));
    k_absmax_t<<<std::min<int64_t>(grid_for(3 * op->N, 256), 4 * ctx->sm_count), 256, 0, ctx->stream>>>(
        op->Tx, 3 * op->N, op->tmax);
    MSB_LAUNCH_CHECK(ctx);
    op->tmax_valid = true;
  }
  *out = op->tmax;
  return MSB_OK;
}

msb_status coarse_assemble_const_gated(msb_ctx ctx, msb_level L, msb_op op, const int* Md, int Mcap) {
  Coarse& co = L->co;
  cudaStream_t st = ctx->stream;
  if (!co.acc || co.acc_cap < (size_t)Mcap * Mcap)
    return set_error(ctx, MSB_EINVAL, "coarse_assemble_const_gated: accumulator not reserved");
  if (!op->tmax_valid) return set_error(ctx, MSB_EINVAL, "coarse_assemble_const_gated: max|T| not cached");
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.acc, 0, (size_t)2 * Mcap * Mcap * sizeof(unsigned long long), st));
  k_rap_const_det<<<grid_for(op->N, 256), 256, 0, st>>>(L->col, make_grid3(op->nx, op->ny, op->nz), 0,
                                                        op->Tx, op->Ty, op->Tz, op->tmax, co.acc, Md);
  MSB_LAUNCH_CHECK(ctx);
  k_fx_const_to_double<<<Mcap, 256, 0, st>>>(co.acc, 0, op->tmax, co.Ac, Md);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

msb_status coarse_assemble_dense(msb_ctx ctx, msb_level L, msb_op op) {
  int M = L->M;
  Coarse& co = L->co;
  if (co.cap < M) {
    coarse_free(ctx, co);
    msb_status rc = ensure_dense(ctx, co, M);
    if (rc) return rc;
  }
  co.M = M;
  co.kind = 0;
  // explicit levels: deterministic exact accumulation (128-bit fixed point) whenever its
  // 16 B per entry fit comfortably (M <= 8192: 1 GiB); beyond, fp64 atomics
  cudaStream_t st = ctx->stream;
  // constant basis (W = 1, every P entry exactly 1): only the faces between blocks; an
  // imported W = 1 level (rows no longer known to sum to one) takes the general path
  const bool constant = L->kind == 1 && L->W == 1 && L->unity;
  if (M <= 8192) {
    const size_t n = (size_t)M * M;
    if (co.acc_cap < n) {  // sized for the buffers' capacity: a growing M_dyn reallocates once
      const size_t ncap = std::max(n, (size_t)co.cap * co.cap);
      dfree(ctx, co.acc);
      co.acc = nullptr;
      co.acc_cap = 0;
      MSB_ALLOC(ctx, co.acc, unsigned long long, 2 * ncap + 1);
      co.acc_cap = ncap;
    }
    unsigned long long* tmax = co.acc + 2 * n;
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.acc, 0, (2 * n + 1) * sizeof(unsigned long long), st));
    const unsigned long long* tmax_c = nullptr;
    if (msb_status r0 = op_tmax(ctx, op, &tmax_c)) return r0;
    tmax = const_cast<unsigned long long*>(tmax_c);
    if (constant) {
      k_rap_const_det<<<grid_for(op->N, 256), 256, 0, st>>>(
          L->col, make_grid3(op->nx, op->ny, op->nz), M, op->Tx, op->Ty, op->Tz, tmax, co.acc,
          nullptr);
    } else {
      if (L->unity)
        k_rap<true, true><<<grid_for(L->N, 128), 128, 0, st>>>(*L, L->P[L->cur], op->Tx, op->Ty,
                                                              op->Tz, co.Ac, co.acc, tmax);
      else
        k_rap<true, false><<<grid_for(L->N, 128), 128, 0, st>>>(*L, L->P[L->cur], op->Tx, op->Ty,
                                                               op->Tz, co.Ac, co.acc, tmax);
    }
    MSB_LAUNCH_CHECK(ctx);
    if (constant)
      k_fx_const_to_double<<<M, 256, 0, st>>>(co.acc, M, tmax, co.Ac, nullptr);
    else if (L->unity)
      k_fx_sym_to_double<<<M, 256, 0, st>>>(co.acc, M, tmax, co.Ac);
    else
      k_fx_to_double<<<grid_for((int64_t)n, 256), 256, 0, st>>>(co.acc, (int64_t)n, tmax, co.Ac);
    MSB_LAUNCH_CHECK(ctx);
    return coarse_factor_dense(ctx, co);
  }
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(co.Ac, 0, (size_t)M * M * sizeof(double), st));
  k_rap<false, false><<<grid_for(L->N, 128), 128, 0, st>>>(*L, L->P[L->cur], op->Tx, op->Ty, op->Tz,
                                                    co.Ac, nullptr, nullptr);
  MSB_LAUNCH_CHECK(ctx);
  return coarse_factor_dense(ctx, co);
}

void coarse_free(msb_ctx ctx, Coarse& co) {
  coarse_schur_free(ctx, co);
  dfree(ctx, co.tri_y);
  co.tri_y = nullptr;
  dfree(ctx, co.Aell);
  co.Aell = nullptr;
  co.ell_cap = 0;
  co.kind = 0;
  dfree(ctx, co.Ac);
  dfree(ctx, co.Ainv);
  dfree(ctx, co.L);
  dfree(ctx, co.Xp);
  dfree(ctx, co.part);
  dfree(ctx, co.acc);
  dfree(ctx, co.flags);
  co.flags = nullptr;
  co.acc = nullptr;
  co.acc_cap = 0;
  co.Xp = co.part = nullptr;
  co.xp_cap = 0;
  co.Ac = co.Ainv = co.L = nullptr;
  co.ready = false;
  co.cap = 0;
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_coarse_assemble(msb_ctx ctx, msb_level L, msb_op op) {
  MSB_NVTX("msb_coarse_assemble");
  if (!ctx || !L || !op) return set_error(ctx, MSB_EINVAL, "msb_coarse_assemble: null");
  if (L->N != op->N) return set_error(ctx, MSB_EDIM, "level/operator size mismatch");
  if (L->kind != 0 && (int64_t)L->M * L->M > (int64_t)1 << 31)
    return set_error(ctx, MSB_EINVAL, "dense coarse operator too large (M=%d)", L->M);
  {  // A_c = P^T A P inherits A's singularity on a compartment without the gauge cell
    bool conn = false;
    msb_status rc = op_connected(ctx, op, &conn);
    if (rc) return rc;
    if (!conn)
      return set_error(ctx, MSB_EINCONSISTENT,
                       "the faces with T > 0 split the grid into several compartments: A is "
                       "singular on every compartment without the gauge cell 0");
  }
  return coarse_assemble(ctx, L, op);
}

// COO dump of a Cartesian level's assembled A_c (every in-range box-stencil slot, zeros
// included): nnz_out host; rows/cols int32, vals double (host|dev, each may be NULL).
__global__ void k_ell_coo(const double* __restrict__ Aell, int M, int n0, int n1, int n2,
                          const int64_t* __restrict__ pos, int32_t* __restrict__ r,
                          int32_t* __restrict__ c, double* __restrict__ v) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * ELLW) return;
  const int a = (int)(e / ELLW), d = (int)(e - (int64_t)a * ELLW);
  const int b = d == ELLC ? a : ell_nb(a, d, n0, n1, n2);
  if (b < 0) return;
  const int64_t k = pos[e];
  r[k] = a;
  c[k] = b;
  v[k] = Aell[e];
}

__global__ void k_ell_valid(int M, int n0, int n1, int n2, int64_t* __restrict__ flag) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * ELLW) return;
  const int a = (int)(e / ELLW), d = (int)(e - (int64_t)a * ELLW);
  flag[e] = (d == ELLC || ell_nb(a, d, n0, n1, n2) >= 0) ? 1 : 0;
}

extern "C" msb_status msb_level_export_coarse(msb_ctx ctx, msb_level L, int64_t* nnz_out,
                                              int32_t* rows, int32_t* cols, double* vals) {
  if (!ctx || !L || !nnz_out) return set_error(ctx, MSB_EINVAL, "msb_level_export_coarse: null");
  const Coarse& co = L->co;
  if (L->kind != 0 || !co.Aell || !co.ready)
    return set_error(ctx, MSB_EINVAL, "no assembled Cartesian coarse operator");
  const int M = L->M;
  const int64_t n = (int64_t)M * ELLW;
  cudaStream_t st = ctx->stream;
  std::vector<int64_t> flag(n);
  int64_t* dflag = dalloc_n<int64_t>(ctx, n);
  if (!dflag) return set_error(ctx, MSB_ENOMEM, "export scratch");
  k_ell_valid<<<grid_for(n, 256), 256, 0, st>>>(M, co.nb[0], co.nb[1], co.nb[2], dflag);
  count_launch();
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(flag.data(), dflag, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  int64_t nnz = 0;
  for (int64_t e = 0; e < n; ++e) {  // exclusive positions (row-major, slot order)
    const int64_t f = flag[e];
    flag[e] = nnz;
    nnz += f;
  }
  *nnz_out = nnz;
  if (rows || cols || vals) {
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(dflag, flag.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    int32_t* dr = dalloc_n<int32_t>(ctx, nnz);
    int32_t* dc = dalloc_n<int32_t>(ctx, nnz);
    double* dv = dalloc_n<double>(ctx, nnz);
    if (!dr || !dc || !dv) return set_error(ctx, MSB_ENOMEM, "export scratch");
    k_ell_coo<<<grid_for(n, 256), 256, 0, st>>>(co.Aell, M, co.nb[0], co.nb[1], co.nb[2], dflag, dr,
                                                dc, dv);
    count_launch();
    if (rows) MSB_CUDA_TRY(ctx, copy_out(ctx, rows, dr, nnz * sizeof(int32_t)));
    if (cols) MSB_CUDA_TRY(ctx, copy_out(ctx, cols, dc, nnz * sizeof(int32_t)));
    if (vals) MSB_CUDA_TRY(ctx, copy_out(ctx, vals, dv, nnz * sizeof(double)));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, dr);
    dfree(ctx, dc);
    dfree(ctx, dv);
  }
  dfree(ctx, dflag);
  return MSB_OK;
}
