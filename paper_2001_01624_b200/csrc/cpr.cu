// §8 NEXT-4 — CPR two-stage preconditioner for the compressible two-phase system
// (PAPER.md:122-203 §4, :287-292; readings C1-C6).
//
//   k_cpr_linearize   F = (F_w | F_o) and the block 7-point Jacobian, one thread per
//                     cell: accumulation, the six face fluxes with
//                     single-point upstream ρλ recomputed by both cells
//                     of a face (no atomics), wells; analytic derivatives
//   k_cpr_decouple    per-cell IMPES / quasi-IMPES weights (the 2 x 2 system of
//                     PAPER.md:180-186) fused with the premultiplication J* = W J, F* = W F
//   predictor         n_cycles Eq.-(8) cycles on J*_pp: damped Jacobi (k_cpr_jacobi_pp),
//                     residual (k_cpr_residual_pp), the Cartesian level's restriction and
//                     prolongation (cycle.cu), x_c = A_c^{-1} r_c (k_gemv_rows)
//   coarse setup      A_c = P^T J*_pp P (k_cpr_rap: exact 128-bit fixed point, fx.cuh),
//                     explicit inverse by blocked Gauss–Jordan (pivot blocks of 64 inverted
//                     in one CTA, rank-64 updates on the fp64 tensor-core GEMM)
//   corrector         ILU(0) of the full J* with 2 x 2 cell blocks in red-black cell order:
//                     red pivots D_r, black pivots D̃_b = D_b − Σ A_br D_r^{-1} A_rb
//                     (k_cpr_ilu_setup), solve in three passes (k_cpr_ilu_{red1,black,red2})
#include <algorithm>
#include <cmath>
#include <vector>

#include "fx.cuh"
#include "internal.cuh"

struct msb_cpr_s {
  msb_ctx ctx = nullptr;
  msb_op op = nullptr;
  msb_level lev = nullptr;
  msb_fluid fl{};
  int n_cycles = 1;
  double omega_s = 2.0 / 3.0;
  int64_t N = 0;
  double* J = nullptr;    // 28 N: plane (2b + v) * 7 + d
  double* F = nullptr;    // 2 N
  double* mA = nullptr;   // 2 N: ∂A_w/∂S, ∂A_o/∂S (IMPES)
  double* w = nullptr;    // 2 N
  double* Js = nullptr;   // 14 N: J*'s first block row, pp slots 0..6 | ps slots 0..6
  double* Fs = nullptr;   // N: F*'s first block
  double* ilu = nullptr;  // 4 N: inverse pivot block per cell (row-major 2 x 2)
  int M = 0;
  unsigned long long* acc = nullptr;  // 2 M^2 fixed-point accumulator
  double* Ac = nullptr;               // M^2
  double* Ainv = nullptr;             // M^2
  double* gj = nullptr;               // Gauss–Jordan panels: Cp (M x 64), R (64 x M), P (64^2)
  double* xp = nullptr;   // N: predictor iterate Δp
  double* rp = nullptr;   // N: predictor residual
  double* x1 = nullptr;   // N: Jacobi output
  double* rc = nullptr;   // M
  double* xc = nullptr;   // M
  double* r2 = nullptr;   // 2N: updated residual
  int* zero = nullptr;    // device int 0 (the cycle kernels' stop flag)
  unsigned long long* flags = nullptr;  // [0] max|J*_pp| bits, [1] singular, [2] max|A_c| bits
  bool linearized = false, decoupled = false;
};

namespace msb {

constexpr int CP_T = 256;

struct CprDev {
  Grid3 g;
  const double* Tx;  // base transmissibility planes (cell-padded, face (c, c + e_a))
  const double* Ty;
  const double* Tz;
  double mu_w, mu_o, rho_w, rho_o, c_w, c_o, c_r, phi, p_ref, s;  // s = Δt / |Ω|
  int nrel;
};

__device__ __forceinline__ double cp_rho(const CprDev& D, double p, int ph) {
  return ph == 0 ? D.rho_w * exp(D.c_w * (p - D.p_ref)) : D.rho_o * exp(D.c_o * (p - D.p_ref));
}
// λ and dλ/dS
__device__ __forceinline__ void cp_lam(const CprDev& D, double S, int ph, double& l, double& dl) {
  const double s = ph == 0 ? S : 1.0 - S;
  const double mu = ph == 0 ? D.mu_w : D.mu_o;
  const double sg = ph == 0 ? 1.0 : -1.0;
  if (D.nrel == 2) {
    l = (s * s) / mu;
    dl = sg * 2.0 * s / mu;
  } else {
    l = s / mu;
    dl = sg / mu;
  }
}

// neighbour of c in stencil slot d (1 -x, 2 +x, 3 -y, 4 +y, 5 -z, 6 +z) or -1
__device__ __forceinline__ int cp_nb(const Grid3& g, int c, int i, int j, int k, int d) {
  switch (d) {
    case 0: return c;
    case 1: return i > 0 ? c - 1 : -1;
    case 2: return i < g.nx - 1 ? c + 1 : -1;
    case 3: return j > 0 ? c - g.nx : -1;
    case 4: return j < g.ny - 1 ? c + g.nx : -1;
    case 5: return k > 0 ? c - g.nxy : -1;
    default: return k < g.nz - 1 ? c + g.nxy : -1;
  }
}

__device__ __forceinline__ int cp_opp(int d) { return d == 0 ? 0 : (d & 1 ? d + 1 : d - 1); }

// F and J at cell c.  The residual's terms are added in the oracle's order: accumulation,
// then per axis the face where c is the left cell and the face where it is the right cell,
// then the well.
__global__ void __launch_bounds__(CP_T) k_cpr_linearize(CprDev D, const double* __restrict__ p,
                                                        const double* __restrict__ S,
                                                        const double* __restrict__ pn,
                                                        const double* __restrict__ Sn,
                                                        const double* __restrict__ q,
                                                        double* __restrict__ F,
                                                        double* __restrict__ J,
                                                        double* __restrict__ mA) {
  const int N = D.g.nxy * D.g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(D.g, c, i, j, k);
  const double pc = p[c], Sc = S[c];
  double jac[2][2][7];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int d = 0; d < 7; ++d) jac[b][v][d] = 0.0;
  // accumulation
  const double phi = D.phi * exp(D.c_r * (pc - D.p_ref));
  const double phin = D.phi * exp(D.c_r * (pn[c] - D.p_ref));
  const double rw = cp_rho(D, pc, 0), ro = cp_rho(D, pc, 1);
  const double rwn = cp_rho(D, pn[c], 0), ron = cp_rho(D, pn[c], 1);
  double Fw = phi * rw * Sc - phin * rwn * Sn[c];
  double Fo = phi * ro * (1.0 - Sc) - phin * ron * (1.0 - Sn[c]);
  jac[0][0][0] = (D.c_r + D.c_w) * (phi * rw * Sc);
  jac[0][1][0] = phi * rw;
  jac[1][0][0] = (D.c_r + D.c_o) * (phi * ro * (1.0 - Sc));
  jac[1][1][0] = -(phi * ro);
  mA[c] = phi * rw;
  mA[N + c] = -(phi * ro);
  // faces: slot order (+x as left, -x as right, +y, -y, +z, -z)
  const int order[6] = {2, 1, 4, 3, 6, 5};
#pragma unroll
  for (int o = 0; o < 6; ++o) {
    const int d = order[o];
    const int n = cp_nb(D.g, c, i, j, k, d);
    if (n < 0) continue;
    const bool plus = (d & 1) == 0;  // c is the face's left cell
    const double T = d <= 2 ? (plus ? D.Tx[c] : D.Tx[n]) : d <= 4 ? (plus ? D.Ty[c] : D.Ty[n])
                                                               : (plus ? D.Tz[c] : D.Tz[n]);
    const int l = plus ? c : n, r = plus ? n : c;
    const double pl = p[l], pr = p[r];
    const double dp = pl - pr;
    const bool upl = pl >= pr;  // ties to the left cell (reading A17)
    const int u = upl ? l : r;
    const double pu = p[u], Su = S[u];
    const double sg = plus ? 1.0 : -1.0;  // row c gets +flux as the left cell, -flux as right
    const bool uc = (u == c);
    const double sT = D.s * T;
#pragma unroll
    for (int ph = 0; ph < 2; ++ph) {
      const double rho = cp_rho(D, pu, ph);
      double lam, dlam;
      cp_lam(D, Su, ph, lam, dlam);
      const double m = rho * lam;
      const double flux = sT * m * dp;
      if (ph == 0) Fw += sg * flux;
      else Fo += sg * flux;
      const double cph = ph == 0 ? D.c_w : D.c_o;
      const double dm_dp = cph * m, dm_dS = rho * dlam;
      // ∂flux/∂p_c and ∂flux/∂p_n (c is l or r)
      const double dpc = sT * ((plus ? m : -m) + (uc ? dp * dm_dp : 0.0));
      const double dpn = sT * ((plus ? -m : m) + (uc ? 0.0 : dp * dm_dp));
      const double dSc = uc ? sT * dp * dm_dS : 0.0;
      const double dSn = uc ? 0.0 : sT * dp * dm_dS;
      jac[ph][0][0] += sg * dpc;
      jac[ph][0][d] += sg * dpn;
      jac[ph][1][0] += sg * dSc;
      jac[ph][1][d] += sg * dSn;
    }
  }
  // well
  const double Q = q ? q[c] : 0.0;
  if (Q > 0.0) {
    Fw -= D.s * rw * Q;
    jac[0][0][0] -= D.s * D.c_w * rw * Q;
  } else if (Q < 0.0) {
    double lw, dlw, lo, dlo;
    cp_lam(D, Sc, 0, lw, dlw);
    cp_lam(D, Sc, 1, lo, dlo);
    const double lt = lw + lo;
    const double fw = lw / lt, fo = lo / lt;
    const double dfw = (dlw * lo - lw * dlo) / (lt * lt);
    Fw -= D.s * rw * fw * Q;
    Fo -= D.s * ro * fo * Q;
    jac[0][0][0] -= D.s * D.c_w * rw * fw * Q;
    jac[1][0][0] -= D.s * D.c_o * ro * fo * Q;
    jac[0][1][0] -= D.s * rw * dfw * Q;
    jac[1][1][0] -= D.s * ro * (-dfw) * Q;
  }
  F[c] = Fw;
  F[N + c] = Fo;
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int d = 0; d < 7; ++d) J[(size_t)((2 * b + v) * 7 + d) * N + c] = jac[b][v][d];
}

// weights (method 0 none, 1 IMPES, 2 quasi-IMPES) and J* = W J, F* = W F; max|J*_pp| bits
__global__ void __launch_bounds__(CP_T) k_cpr_decouple(int N, int method,
                                                       const double* __restrict__ J,
                                                       const double* __restrict__ F,
                                                       const double* __restrict__ mA,
                                                       double* __restrict__ w,
                                                       double* __restrict__ Js,
                                                       double* __restrict__ Fs,
                                                       unsigned long long* flags) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double amax = 0.0;
  if (c < N) {
    double m1 = 0.0, m2 = 0.0;
    if (method == 1) {
      m1 = mA[c];
      m2 = mA[N + c];
    } else if (method == 2) {
      m1 = J[(size_t)(1 * 7 + 0) * N + c];  // ∂F_w/∂S_c
      m2 = J[(size_t)(3 * 7 + 0) * N + c];  // ∂F_o/∂S_c
    }
    double w1 = 1.0, w2 = 0.0;
    if (!(m1 == 0.0 && m2 == 0.0)) {
      const double det = m1 - m2;  // det [m1 m2; 1 1]
      if (det == 0.0) {
        atomicOr(flags + 1, 1ull);
      } else {
        w1 = -m2 / det;
        w2 = m1 / det;
      }
    }
    w[c] = w1;
    w[N + c] = w2;
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int d = 0; d < 7; ++d) {
        const double a = J[(size_t)(v * 7 + d) * N + c];        // row w
        const double b = J[(size_t)((2 + v) * 7 + d) * N + c];  // row o
        const double js = __dadd_rn(__dmul_rn(w1, a), __dmul_rn(w2, b));
        Js[(size_t)(v * 7 + d) * N + c] = js;
        if (v == 0) amax = fmax(amax, fabs(js));
      }
    Fs[c] = __dadd_rn(__dmul_rn(w1, F[c]), __dmul_rn(w2, F[N + c]));
  }
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) atomicMax(flags, (unsigned long long)__double_as_longlong(amax));
}

// ---------------------------------------------------------------- coupled ILU(0)
// 2 x 2 block of row c at stencil slot d: [[J*pp, J*ps], [J_sp, J_ss]]
__device__ __forceinline__ void cp_block(const double* __restrict__ Js, const double* __restrict__ J,
                                         int N, int c, int d, double (&a)[4]) {
  a[0] = Js[(size_t)(0 * 7 + d) * N + c];
  a[1] = Js[(size_t)(1 * 7 + d) * N + c];
  a[2] = J[(size_t)(2 * 7 + d) * N + c];
  a[3] = J[(size_t)(3 * 7 + d) * N + c];
}

__device__ __forceinline__ bool cp_inv2(const double (&a)[4], double (&o)[4]) {
  const double det = a[0] * a[3] - a[1] * a[2];
  if (det == 0.0 || !isfinite(det)) return false;
  const double id = 1.0 / det;
  o[0] = a[3] * id;
  o[1] = -a[1] * id;
  o[2] = -a[2] * id;
  o[3] = a[0] * id;
  return true;
}

// red cells ((i+j+k) even): inverse of D_r; black: inverse of D_b − Σ_r A_br D_r^{-1} A_rb
// with the red neighbours taken in ascending cell order (-z, -y, -x, +x, +y, +z)
__global__ void __launch_bounds__(CP_T) k_cpr_ilu_setup(Grid3 g, const double* __restrict__ Js,
                                                        const double* __restrict__ J,
                                                        double* __restrict__ ilu,
                                                        unsigned long long* flags) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  double D[4];
  cp_block(Js, J, N, c, 0, D);
  if (((i + j + k) & 1) == 1) {
    const int asc[6] = {5, 3, 1, 2, 4, 6};
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      const int d = asc[o];
      const int n = cp_nb(g, c, i, j, k, d);
      if (n < 0) continue;
      double Abr[4], Dr[4], Dri[4], Arb[4];
      cp_block(Js, J, N, c, d, Abr);
      cp_block(Js, J, N, n, 0, Dr);
      cp_block(Js, J, N, n, cp_opp(d), Arb);
      if (!cp_inv2(Dr, Dri)) {
        atomicOr(flags + 1, 2ull);
        continue;
      }
      // T = D_r^{-1} A_rb, D -= A_br T
      const double t0 = Dri[0] * Arb[0] + Dri[1] * Arb[2], t1 = Dri[0] * Arb[1] + Dri[1] * Arb[3];
      const double t2 = Dri[2] * Arb[0] + Dri[3] * Arb[2], t3 = Dri[2] * Arb[1] + Dri[3] * Arb[3];
      D[0] -= Abr[0] * t0 + Abr[1] * t2;
      D[1] -= Abr[0] * t1 + Abr[1] * t3;
      D[2] -= Abr[2] * t0 + Abr[3] * t2;
      D[3] -= Abr[2] * t1 + Abr[3] * t3;
    }
  }
  double Di[4];
  if (!cp_inv2(D, Di)) {
    atomicOr(flags + 1, 2ull);
    Di[0] = Di[1] = Di[2] = Di[3] = 0.0;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) ilu[(size_t)e * N + c] = Di[e];
}

// pass 1 (red): t_r = D_r^{-1} r_r into x;  pass 3 (red): x_r = D_r^{-1}(r_r − Σ A_rb x_b)
// pass 2 (black): x_b = D̃_b^{-1}(r_b − Σ A_br t_r)
template <int PASS>
__global__ void __launch_bounds__(CP_T) k_cpr_ilu_pass(Grid3 g, const double* __restrict__ Js,
                                                       const double* __restrict__ J,
                                                       const double* __restrict__ ilu,
                                                       const double* __restrict__ r,
                                                       double* __restrict__ x) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const bool black = ((i + j + k) & 1) == 1;
  if ((PASS == 2) != black) return;
  double y0 = r[c], y1 = r[N + c];
  if (PASS != 1) {
    const int asc[6] = {5, 3, 1, 2, 4, 6};
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      const int d = asc[o];
      const int n = cp_nb(g, c, i, j, k, d);
      if (n < 0) continue;
      double A[4];
      cp_block(Js, J, N, c, d, A);
      const double u0 = x[n], u1 = x[N + n];
      y0 -= A[0] * u0 + A[1] * u1;
      y1 -= A[2] * u0 + A[3] * u1;
    }
  }
  const double a = ilu[c], b = ilu[(size_t)N + c], cc = ilu[(size_t)2 * N + c],
               dd = ilu[(size_t)3 * N + c];
  x[c] = a * y0 + b * y1;
  x[N + c] = cc * y0 + dd * y1;
}

// ---------------------------------------------------------------- operators on J*
// J*_pp x at cell c, neighbours in ascending cell order (scipy's CSR row order)
__device__ __forceinline__ double cp_pp_row(const Grid3& g, const double* __restrict__ A, int N,
                                            int c, int i, int j, int k,
                                            const double* __restrict__ x) {
  const int asc[7] = {5, 3, 1, 0, 2, 4, 6};
  double s = 0.0;
#pragma unroll
  for (int o = 0; o < 7; ++o) {
    const int d = asc[o];
    const int n = cp_nb(g, c, i, j, k, d);
    if (n >= 0) s += A[(size_t)d * N + c] * x[n];
  }
  return s;
}

// r = b − J*_pp x
__global__ void __launch_bounds__(CP_T) k_cpr_residual_pp(Grid3 g, const double* __restrict__ A,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ r) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  r[c] = b[c] - cp_pp_row(g, A, N, c, i, j, k, x);
}

// xo = x + ω (b − J*_pp x) / J*_pp,cc   (x may be NULL: x = 0)
__global__ void __launch_bounds__(CP_T) k_cpr_jacobi_pp(Grid3 g, const double* __restrict__ A,
                                                        const double* __restrict__ b,
                                                        const double* __restrict__ x,
                                                        double omega, double* __restrict__ xo) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const double xc = x ? x[c] : 0.0;
  const double r = x ? b[c] - cp_pp_row(g, A, N, c, i, j, k, x) : b[c] - 0.0;
  xo[c] = xc + omega * (r / A[c]);
}

// r2 = r − J*[:, p] Δp: p rows with J*_pp, S rows with J_sp
__global__ void __launch_bounds__(CP_T) k_cpr_update(Grid3 g, const double* __restrict__ Js,
                                                     const double* __restrict__ J,
                                                     const double* __restrict__ r,
                                                     const double* __restrict__ dp,
                                                     double* __restrict__ r2) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  r2[c] = r[c] - cp_pp_row(g, Js, N, c, i, j, k, dp);
  r2[N + c] = r[N + c] - cp_pp_row(g, J + (size_t)(2 * 7) * N, N, c, i, j, k, dp);
}

// y = J* x (both block rows)
__global__ void __launch_bounds__(CP_T) k_cpr_apply_sys(Grid3 g, const double* __restrict__ Js,
                                                        const double* __restrict__ J,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  y[c] = cp_pp_row(g, Js, N, c, i, j, k, x) +
         cp_pp_row(g, Js + (size_t)7 * N, N, c, i, j, k, x + N);
  y[N + c] = cp_pp_row(g, J + (size_t)(2 * 7) * N, N, c, i, j, k, x) +
             cp_pp_row(g, J + (size_t)(3 * 7) * N, N, c, i, j, k, x + N);
}

// b = -F* (the Newton right-hand side of the decoupled system)
__global__ void k_cpr_negrhs(int64_t N, const double* __restrict__ Fs, const double* __restrict__ F,
                             double* __restrict__ b) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  b[t] = -Fs[t];
  b[N + t] = -F[N + t];
}

__global__ void k_cpr_axpy(int64_t n, const double* __restrict__ a, double* __restrict__ y) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) y[t] += a[t];
}

// ---------------------------------------------------------------- coarse operator
// A_c(I, J) += P_iI · a_{i,d} · P_{n_d, J} over the Cartesian level's parity slots: per
// slot s the neighbours whose slot-s column equals cell i's are summed first (u_s), the
// others are scattered on their own; exact fixed-point atomics (fx.cuh)
struct CartP {
  Grid3 g;
  const int32_t* tab;
  const double* P;
  int nb0, nb1;
};

__device__ __forceinline__ int cart_col(const CartP& L, int i, int j, int k, int s) {
  const int jx = L.tab[2 * i + (s & 1)], jy = L.tab[2 * (L.g.nx + j) + ((s >> 1) & 1)],
            jz = L.tab[2 * (L.g.nx + L.g.ny + k) + (s >> 2)];
  if (jx < 0 || jy < 0 || jz < 0) return -1;
  return jx + L.nb0 * (jy + L.nb1 * jz);
}

__global__ void __launch_bounds__(128) k_cpr_rap(CartP L, const double* __restrict__ A, int M,
                                                 const unsigned long long* __restrict__ amax_bits,
                                                 unsigned long long* __restrict__ acc) {
  const int N = L.g.nxy * L.g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(L.g, c, i, j, k);
  const int F = 90 - ilogb(__longlong_as_double((long long)*amax_bits));
  int I[8];
  double pI[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    I[t] = cart_col(L, i, j, k, t);
    pI[t] = I[t] >= 0 ? L.P[(size_t)t * N + c] : 0.0;
  }
  int nn[7], ni[7], nj[7], nk[7];
  double a[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) {
    nn[d] = cp_nb(L.g, c, i, j, k, d);
    a[d] = nn[d] >= 0 ? A[(size_t)d * N + c] : 0.0;
    ni[d] = i + (d == 1 ? -1 : d == 2 ? 1 : 0);
    nj[d] = j + (d == 3 ? -1 : d == 4 ? 1 : 0);
    nk[d] = k + (d == 5 ? -1 : d == 6 ? 1 : 0);
  }
  for (int s = 0; s < 8; ++s) {
    const int J0 = I[s];
    double u = 0.0;
    for (int d = 0; d < 7; ++d) {
      if (nn[d] < 0 || a[d] == 0.0) continue;
      const int Jd = cart_col(L, ni[d], nj[d], nk[d], s);
      if (Jd < 0) continue;
      const double v = a[d] * L.P[(size_t)s * N + nn[d]];
      if (v == 0.0) continue;
      if (Jd == J0) {
        u += v;
      } else {
        for (int t = 0; t < 8; ++t)
          if (I[t] >= 0 && pI[t] != 0.0) fx_add(acc + 2 * ((size_t)I[t] * M + Jd), pI[t] * v, F);
      }
    }
    if (J0 >= 0 && u != 0.0)
      for (int t = 0; t < 8; ++t)
        if (I[t] >= 0 && pI[t] != 0.0) fx_add(acc + 2 * ((size_t)I[t] * M + J0), pI[t] * u, F);
  }
}

__global__ void k_cpr_fx_dense(const unsigned long long* __restrict__ acc, int64_t n,
                               const unsigned long long* __restrict__ amax_bits,
                               double* __restrict__ Ac, unsigned long long* __restrict__ cmax) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (t < n) {
    const int F = 90 - ilogb(__longlong_as_double((long long)*amax_bits));
    const double v = fx_value(acc[2 * t], acc[2 * t + 1], F);
    Ac[t] = v;
    m = fabs(v);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(cmax, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------------------- Gauss–Jordan inverse
constexpr int GJB = 64;

// invert the w x w pivot block A(k0.., k0..) (ld M) without pivoting into P (ld 64)
__global__ void __launch_bounds__(1024) k_gj_pivot(const double* __restrict__ A, int64_t ld,
                                                   int k0, int w, double* __restrict__ P,
                                                   const unsigned long long* cmax_bits,
                                                   unsigned long long* flags) {
  __shared__ double a[GJB][GJB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < GJB * GJB; e += blockDim.x) {
    const int r = e / GJB, c = e % GJB;
    a[r][c] = (r < w && c < w) ? A[(int64_t)(k0 + r) * ld + k0 + c] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const double amax = __longlong_as_double((long long)*cmax_bits);
  // in-place Gauss–Jordan: after step q, column q holds the inverse's column
  for (int q = 0; q < GJB; ++q) {
    const double piv = a[q][q];
    if (q < w && !(fabs(piv) > 1e-14 * amax)) {
      if (tid == 0) atomicOr(flags + 1, 4ull);
    }
    const double ip = 1.0 / piv;
    __syncthreads();
    // update rows r != q: a[r][c] -= a[r][q] * a[q][c] * ip (c != q); a[r][q] = -a[r][q] ip
    for (int e = tid; e < GJB * GJB; e += blockDim.x) {
      const int r = e / GJB, c = e % GJB;
      if (r != q && c != q) a[r][c] -= a[r][q] * (a[q][c] * ip);
    }
    __syncthreads();
    for (int e = tid; e < GJB; e += blockDim.x) {
      if (e != q) {
        a[e][q] = -a[e][q] * ip;
        a[q][e] = a[q][e] * ip;
      }
    }
    __syncthreads();
    if (tid == 0) a[q][q] = ip;
    __syncthreads();
  }
  for (int e = tid; e < GJB * GJB; e += blockDim.x) P[e] = a[e / GJB][e % GJB];
}

// Cp = A(:, k0..k0+w) with the pivot rows zeroed (ld 64)
__global__ void k_gj_copycol(const double* __restrict__ A, int64_t ld, int M, int k0, int w,
                             double* __restrict__ Cp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)M * GJB) return;
  const int r = (int)(t / GJB), c = (int)(t % GJB);
  Cp[t] = (c < w && (r < k0 || r >= k0 + w)) ? A[(int64_t)r * ld + k0 + c] : 0.0;
}

// A(k0.., :) = R; A(k0.., k0..) = P
__global__ void k_gj_rowfix(double* __restrict__ A, int64_t ld, int M, int k0, int w,
                            const double* __restrict__ R, const double* __restrict__ P) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)w * M) return;
  const int r = (int)(t / M), c = (int)(t % M);
  A[(int64_t)(k0 + r) * ld + c] =
      (c >= k0 && c < k0 + w) ? P[r * GJB + (c - k0)] : R[(int64_t)r * M + c];
}

// x_c = A^{-1} r_c, one warp per row (lane-strided, fixed shuffle tree)
__global__ void __launch_bounds__(256) k_gemv_rows(const double* __restrict__ A, int M,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y) {
  const int row = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const double* a = A + (int64_t)row * M;
  double v = 0.0;
  for (int c = lane; c < M; c += 32) v = fma(a[c], x[c], v);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) y[row] = v;
}

static CprDev dev_of(msb_cpr c) {
  msb_op op = c->op;
  CprDev D;
  D.g = make_grid3(op->nx, op->ny, op->nz);
  D.Tx = op->Tb;
  D.Ty = op->Tb + op->N;
  D.Tz = op->Tb + 2 * op->N;
  D.mu_w = c->fl.mu_w;
  D.mu_o = c->fl.mu_o;
  D.rho_w = c->fl.rho_w;
  D.rho_o = c->fl.rho_o;
  D.c_w = c->fl.c_w;
  D.c_o = c->fl.c_o;
  D.c_r = c->fl.c_r;
  D.phi = c->fl.phi;
  D.p_ref = c->fl.p_ref;
  D.s = c->fl.dt / (op->dx * op->dy * op->dz);
  D.nrel = c->fl.nrel;
  return D;
}

static msb_status cpr_inverse(msb_ctx ctx, msb_cpr c) {
  const int M = c->M;
  cudaStream_t st = ctx->stream;
  double* A = c->Ainv;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(A, c->Ac, (size_t)M * M * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
  double* Cp = c->gj;
  double* R = Cp + (size_t)M * GJB;
  double* P = R + (size_t)GJB * M;
  for (int k0 = 0; k0 < M; k0 += GJB) {
    const int w = std::min(GJB, M - k0);
    k_gj_pivot<<<1, 1024, 0, st>>>(A, M, k0, w, P, c->flags + 2, c->flags);
    MSB_LAUNCH_CHECK(ctx);
    // R = P A(k0.., :)
    msb_status rc = dgemm(ctx, false, false, w, M, w, 1.0, P, GJB, A + (size_t)k0 * M, M, 0.0, R, M);
    if (rc) return rc;
    k_gj_copycol<<<grid_for((int64_t)M * GJB, 256), 256, 0, st>>>(A, M, M, k0, w, Cp);
    MSB_LAUNCH_CHECK(ctx);
    // A -= Cp R (pivot rows untouched: their Cp rows are zero)
    if ((rc = dgemm(ctx, false, false, M, M, w, -1.0, Cp, GJB, R, M, 1.0, A, M))) return rc;
    // A(:, k0..) = -Cp P (pivot rows get 0, overwritten next)
    if ((rc = dgemm(ctx, false, false, M, w, w, -1.0, Cp, GJB, P, GJB, 0.0, A + k0, M))) return rc;
    k_gj_rowfix<<<grid_for((int64_t)w * M, 256), 256, 0, st>>>(A, M, M, k0, w, R, P);
    MSB_LAUNCH_CHECK(ctx);
  }
  return MSB_OK;
}

static msb_status cpr_predictor(msb_ctx ctx, msb_cpr c, const double* rp_in) {
  cudaStream_t st = ctx->stream;
  const Grid3 g = make_grid3(c->op->nx, c->op->ny, c->op->nz);
  const unsigned gr = grid_for(c->N, CP_T);
  for (int cyc = 0; cyc < c->n_cycles; ++cyc) {
    // pre-smoothing: x1 = x + ω D^{-1}(b − A x)   (x = 0 on the first cycle)
    k_cpr_jacobi_pp<<<gr, CP_T, 0, st>>>(g, c->Js, rp_in, cyc ? c->xp : nullptr, c->omega_s,
                                         c->x1);
    MSB_LAUNCH_CHECK(ctx);
    k_cpr_residual_pp<<<gr, CP_T, 0, st>>>(g, c->Js, rp_in, c->x1, c->rp);
    MSB_LAUNCH_CHECK(ctx);
    msb_status rc = level_restrict(ctx, c->lev, c->rp, c->rc, c->zero);
    if (rc) return rc;
    k_gemv_rows<<<grid_for((int64_t)c->M * 32, 256), 256, 0, st>>>(c->Ainv, c->M, c->rc, c->xc);
    MSB_LAUNCH_CHECK(ctx);
    if ((rc = level_prolong_add(ctx, c->lev, c->x1, c->xc, c->zero))) return rc;
    std::swap(c->x1, c->xp);  // xp = the cycle's result
  }
  return MSB_OK;
}

static msb_status cpr_ilu_solve(msb_ctx ctx, msb_cpr c, const double* r, double* x) {
  cudaStream_t st = ctx->stream;
  const Grid3 g = make_grid3(c->op->nx, c->op->ny, c->op->nz);
  const unsigned gr = grid_for(c->N, CP_T);
  k_cpr_ilu_pass<1><<<gr, CP_T, 0, st>>>(g, c->Js, c->J, c->ilu, r, x);
  MSB_LAUNCH_CHECK(ctx);
  k_cpr_ilu_pass<2><<<gr, CP_T, 0, st>>>(g, c->Js, c->J, c->ilu, r, x);
  MSB_LAUNCH_CHECK(ctx);
  k_cpr_ilu_pass<3><<<gr, CP_T, 0, st>>>(g, c->Js, c->J, c->ilu, r, x);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

static msb_status cpr_apply_dev(msb_ctx ctx, msb_cpr c, const double* r, double* dx) {
  msb_status rc = cpr_predictor(ctx, c, r);
  if (rc) return rc;
  cudaStream_t st = ctx->stream;
  const Grid3 g = make_grid3(c->op->nx, c->op->ny, c->op->nz);
  const unsigned gr = grid_for(c->N, CP_T);
  k_cpr_update<<<gr, CP_T, 0, st>>>(g, c->Js, c->J, r, c->xp, c->r2);
  MSB_LAUNCH_CHECK(ctx);
  if ((rc = cpr_ilu_solve(ctx, c, c->r2, dx))) return rc;
  k_cpr_axpy<<<gr, CP_T, 0, st>>>(c->N, c->xp, dx);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

static msb_status cpr_apply_sys_dev(msb_ctx ctx, msb_cpr c, const double* x, double* y) {
  const Grid3 g = make_grid3(c->op->nx, c->op->ny, c->op->nz);
  k_cpr_apply_sys<<<grid_for(c->N, CP_T), CP_T, 0, ctx->stream>>>(g, c->Js, c->J, x, y);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

}  // namespace msb

using namespace msb;

extern "C" {

msb_status msb_cpr_destroy(msb_cpr c) {
  if (!c) return MSB_OK;
  msb_ctx ctx = c->ctx;
  cudaStreamSynchronize(ctx->stream);
  for (void* p : {(void*)c->J, (void*)c->F, (void*)c->mA, (void*)c->w, (void*)c->Js,
                  (void*)c->Fs, (void*)c->ilu, (void*)c->acc, (void*)c->Ac, (void*)c->Ainv,
                  (void*)c->gj, (void*)c->xp, (void*)c->rp, (void*)c->x1, (void*)c->rc,
                  (void*)c->xc, (void*)c->r2, (void*)c->zero, (void*)c->flags})
    dfree(ctx, p);
  delete c;
  return MSB_OK;
}

msb_status msb_cpr_create(msb_ctx ctx, msb_op op, msb_level lev, const msb_fluid* fl,
                          int32_t n_cycles, double omega_s, msb_cpr* out) {
  if (!ctx || !op || !lev || !fl || !out) return set_error(ctx, MSB_EINVAL, "msb_cpr_create: null");
  *out = nullptr;
  if (fl->nrel != 1 && fl->nrel != 2) return set_error(ctx, MSB_EINVAL, "msb_cpr_create: nrel must be 1 or 2");
  if (n_cycles < 1) return set_error(ctx, MSB_EINVAL, "msb_cpr_create: n_cycles < 1");
  if (lev->kind != 0) return set_error(ctx, MSB_EINVAL, "msb_cpr_create: Cartesian level required");
  if (lev->nx != op->nx || lev->ny != op->ny || lev->nz != op->nz)
    return set_error(ctx, MSB_EDIM, "msb_cpr_create: level of another grid");
  if (lev->M > 8192)
    return set_error(ctx, MSB_EINVAL, "msb_cpr_create: the predictor's dense coarse inverse "
                     "supports M <= 8192 (M=%d)", lev->M);
  if (!(fl->dt > 0.0) || !(fl->mu_w > 0.0) || !(fl->mu_o > 0.0))
    return set_error(ctx, MSB_EINVAL, "msb_cpr_create: dt and viscosities must be > 0");
  msb_cpr c = new msb_cpr_s();
  c->ctx = ctx;
  c->op = op;
  c->lev = lev;
  c->fl = *fl;
  c->n_cycles = n_cycles;
  c->omega_s = omega_s;
  c->N = op->N;
  c->M = lev->M;
  const int64_t N = op->N;
  const int64_t M = lev->M;
  auto fail = [&](msb_status s) {
    msb_cpr_destroy(c);
    return s;
  };
#define CPR_ALLOC(ptr, type, n)                                                              \
  do {                                                                                       \
    (ptr) = dalloc_n<type>(ctx, (size_t)(n));                                                \
    if (!(ptr)) return fail(set_error(ctx, MSB_ENOMEM, "msb_cpr_create: allocation of %zu bytes", \
                                      (size_t)(n) * sizeof(type)));                          \
  } while (0)
  CPR_ALLOC(c->J, double, 28 * N);
  CPR_ALLOC(c->F, double, 2 * N);
  CPR_ALLOC(c->mA, double, 2 * N);
  CPR_ALLOC(c->w, double, 2 * N);
  CPR_ALLOC(c->Js, double, 14 * N);
  CPR_ALLOC(c->Fs, double, N);
  CPR_ALLOC(c->ilu, double, 4 * N);
  CPR_ALLOC(c->acc, unsigned long long, 2 * M * M);
  CPR_ALLOC(c->Ac, double, M * M);
  CPR_ALLOC(c->Ainv, double, M * M);
  CPR_ALLOC(c->gj, double, 2 * M * GJB + GJB * GJB);
  CPR_ALLOC(c->xp, double, N);
  CPR_ALLOC(c->rp, double, N);
  CPR_ALLOC(c->x1, double, N);
  CPR_ALLOC(c->rc, double, M);
  CPR_ALLOC(c->xc, double, M);
  CPR_ALLOC(c->r2, double, 2 * N);
  CPR_ALLOC(c->zero, int, 4);
  CPR_ALLOC(c->flags, unsigned long long, 4);
#undef CPR_ALLOC
  cudaError_t e = cudaMemsetAsync(c->zero, 0, 4 * sizeof(int), ctx->stream);
  if (e != cudaSuccess) return fail(set_error(ctx, MSB_ECUDA, "memset: %s", cudaGetErrorString(e)));
  *out = c;
  return MSB_OK;
}

msb_status msb_cpr_linearize(msb_ctx ctx, msb_cpr c, const double* p, const double* S,
                             const double* p_n, const double* S_n, const double* q) {
  MSB_NVTX("msb_cpr_linearize");
  if (!ctx || !c || !p || !S || !p_n || !S_n) return set_error(ctx, MSB_EINVAL, "msb_cpr_linearize: null");
  const int64_t N = c->N;
  const size_t B = N * sizeof(double);
  struct Staged {
    msb_ctx ctx;
    void* o[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    ~Staged() {
      cudaStreamSynchronize(ctx->stream);
      for (void* x : o) dfree(ctx, x);
    }
  } sg{ctx};
  const double* dp = (const double*)stage_in(ctx, p, B, &sg.o[0]);
  const double* dS = (const double*)stage_in(ctx, S, B, &sg.o[1]);
  const double* dpn = (const double*)stage_in(ctx, p_n, B, &sg.o[2]);
  const double* dSn = (const double*)stage_in(ctx, S_n, B, &sg.o[3]);
  const double* dq = q ? (const double*)stage_in(ctx, q, B, &sg.o[4]) : nullptr;
  if (!dp || !dS || !dpn || !dSn || (q && !dq)) return set_error(ctx, MSB_ENOMEM, "msb_cpr_linearize: staging");
  k_cpr_linearize<<<grid_for(N, CP_T), CP_T, 0, ctx->stream>>>(dev_of(c), dp, dS, dpn, dSn, dq, c->F,
                                                               c->J, c->mA);
  MSB_LAUNCH_CHECK(ctx);
  c->linearized = true;
  c->decoupled = false;
  return MSB_OK;
}

msb_status msb_cpr_decouple(msb_ctx ctx, msb_cpr c, int32_t method) {
  MSB_NVTX("msb_cpr_decouple");
  if (!ctx || !c) return set_error(ctx, MSB_EINVAL, "msb_cpr_decouple: null");
  if (method < 0 || method > 2) return set_error(ctx, MSB_EINVAL, "msb_cpr_decouple: method");
  if (!c->linearized) return set_error(ctx, MSB_EINVAL, "msb_cpr_decouple: linearize first");
  const int64_t N = c->N;
  const int M = c->M;
  cudaStream_t st = ctx->stream;
  c->decoupled = false;
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(c->flags, 0, 4 * sizeof(unsigned long long), st));
  k_cpr_decouple<<<grid_for(N, CP_T), CP_T, 0, st>>>((int)N, method, c->J, c->F, c->mA, c->w, c->Js,
                                                      c->Fs, c->flags);
  MSB_LAUNCH_CHECK(ctx);
  // predictor: A_c = P^T J*_pp P, exact, then the explicit inverse
  msb_level L = c->lev;
  CartP cp{make_grid3(L->nx, L->ny, L->nz), L->tab, L->P[L->cur], L->nb[0], L->nb[1]};
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(c->acc, 0, (size_t)2 * M * M * sizeof(unsigned long long), st));
  k_cpr_rap<<<grid_for(N, 128), 128, 0, st>>>(cp, c->Js, M, c->flags, c->acc);
  MSB_LAUNCH_CHECK(ctx);
  k_cpr_fx_dense<<<grid_for((int64_t)M * M, 256), 256, 0, st>>>(c->acc, (int64_t)M * M, c->flags,
                                                                c->Ac, c->flags + 2);
  MSB_LAUNCH_CHECK(ctx);
  msb_status rc = cpr_inverse(ctx, c);
  if (rc) return rc;
  // corrector: block red-black ILU(0) pivots
  k_cpr_ilu_setup<<<grid_for(N, CP_T), CP_T, 0, st>>>(make_grid3(c->op->nx, c->op->ny, c->op->nz),
                                                      c->Js, c->J, c->ilu, c->flags);
  MSB_LAUNCH_CHECK(ctx);
  unsigned long long fl[4];
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (fl[1] & 1ull) return set_error(ctx, MSB_ESINGULAR, "msb_cpr_decouple: singular weight system");
  if (fl[1] & 4ull) return set_error(ctx, MSB_ESINGULAR, "msb_cpr_decouple: coarse pivot <= 1e-14 max|A_c|");
  if (fl[1] & 2ull) return set_error(ctx, MSB_ESINGULAR, "msb_cpr_decouple: singular ILU(0) pivot block");
  c->decoupled = true;
  return MSB_OK;
}

msb_status msb_cpr_apply(msb_ctx ctx, msb_cpr c, const double* r, double* dx) {
  MSB_NVTX("msb_cpr_apply");
  if (!ctx || !c || !r || !dx || r == dx) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply: args");
  if (!c->decoupled) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply: decouple first");
  if (!is_device_ptr(r) || !is_device_ptr(dx)) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply: device vectors");
  return cpr_apply_dev(ctx, c, r, dx);
}

msb_status msb_cpr_apply_system(msb_ctx ctx, msb_cpr c, const double* x, double* y) {
  if (!ctx || !c || !x || !y) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply_system: args");
  if (!c->decoupled) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply_system: decouple first");
  if (!is_device_ptr(x) || !is_device_ptr(y)) return set_error(ctx, MSB_EINVAL, "msb_cpr_apply_system: device vectors");
  return cpr_apply_sys_dev(ctx, c, x, y);
}

msb_status msb_cpr_export(msb_ctx ctx, msb_cpr c, double* F, double* J, double* w, double* Fs,
                          double* Js_row0) {
  if (!ctx || !c) return set_error(ctx, MSB_EINVAL, "msb_cpr_export: null");
  if (!c->linearized) return set_error(ctx, MSB_EINVAL, "msb_cpr_export: linearize first");
  if ((w || Fs || Js_row0) && !c->decoupled)
    return set_error(ctx, MSB_EINVAL, "msb_cpr_export: decouple first");
  const int64_t N = c->N;
  const size_t B = N * sizeof(double);
  if (F) MSB_CUDA_TRY(ctx, copy_out(ctx, F, c->F, 2 * B));
  if (J) MSB_CUDA_TRY(ctx, copy_out(ctx, J, c->J, 28 * B));
  if (w) MSB_CUDA_TRY(ctx, copy_out(ctx, w, c->w, 2 * B));
  if (Fs) {
    MSB_CUDA_TRY(ctx, copy_out(ctx, Fs, c->Fs, B));
    MSB_CUDA_TRY(ctx, copy_out(ctx, Fs + N, c->F + N, B));
  }
  if (Js_row0) MSB_CUDA_TRY(ctx, copy_out(ctx, Js_row0, c->Js, 14 * B));
  return sync(ctx);
}

msb_status msb_cpr_export_coarse(msb_ctx ctx, msb_cpr c, double* Ac, int32_t* M_out) {
  if (!ctx || !c) return set_error(ctx, MSB_EINVAL, "msb_cpr_export_coarse: null");
  if (M_out) *M_out = c->M;
  if (!Ac) return MSB_OK;
  if (!c->decoupled) return set_error(ctx, MSB_EINVAL, "msb_cpr_export_coarse: decouple first");
  MSB_CUDA_TRY(ctx, copy_out(ctx, Ac, c->Ac, (size_t)c->M * c->M * sizeof(double)));
  return sync(ctx);
}

msb_status msb_cpr_fgmres(msb_ctx ctx, msb_cpr c, const double* b, double* x, double tol,
                          int32_t restart, int32_t max_iter, int32_t fixed_iters, int32_t precond,
                          int32_t* iters_out, double* res_hist) {
  MSB_NVTX("msb_cpr_fgmres");
  if (!ctx || !c || !x) return set_error(ctx, MSB_EINVAL, "msb_cpr_fgmres: null");
  if (precond != 1 && precond != 2) return set_error(ctx, MSB_EINVAL, "msb_cpr_fgmres: precond must be 1 or 2");
  if (!c->decoupled) return set_error(ctx, MSB_EINVAL, "msb_cpr_fgmres: decouple first");
  const int64_t N2 = 2 * c->N;
  struct Staged {
    msb_ctx ctx;
    double* d = nullptr;
    void* o = nullptr;
    ~Staged() {
      cudaStreamSynchronize(ctx->stream);
      dfree(ctx, d);
      dfree(ctx, o);
    }
  } sb{ctx};
  const double* db;
  if (b) {
    db = (const double*)stage_in(ctx, b, N2 * sizeof(double), &sb.o);
    if (!db) return set_error(ctx, MSB_ENOMEM, "rhs staging");
  } else {  // -F*
    sb.d = dalloc_n<double>(ctx, N2);
    if (!sb.d) return set_error(ctx, MSB_ENOMEM, "rhs");
    k_cpr_negrhs<<<grid_for(c->N, CP_T), CP_T, 0, ctx->stream>>>(c->N, c->Fs, c->F, sb.d);
    MSB_LAUNCH_CHECK(ctx);
    db = sb.d;
  }
  FgOps ops;
  ops.A = [&](const double* xv, double* yv) { return cpr_apply_sys_dev(ctx, c, xv, yv); };
  if (precond == 1) ops.M = [&](const double* v, double* z) { return cpr_apply_dev(ctx, c, v, z); };
  else ops.M = [&](const double* v, double* z) { return cpr_ilu_solve(ctx, c, v, z); };
  return fgmres_core(ctx, N2, ops, db, x, tol, restart, max_iter, fixed_iters, iters_out, res_hist);
}

}  // extern "C"
