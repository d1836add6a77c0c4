// Row a3 — MsRSB restricted-smoothing sweep (G2 Cartesian parity slots, G3 ELL).
//
//   P^_ij = (1-ω) P_ij + (ω/D_i) Σ_{l~i} T_il P_lj   on the pattern (positive form, A5)
//   P_ij <- P^_ij / Σ_k P^_ik                         every row (A6)
//   δ_n  = max |P^{n+1} - P^n|                         (A16)
//
// One thread per cell, all slots of the cell in registers (so the row sum and the
// renormalisation are free), coalesced fp64 loads of each slot plane and of the
// cell-padded transmissibilities.  Sweep n reads buffer n&1 and writes buffer
// (n+1)&1.  δ_n is folded per block into one of DSLOTS atomicMax slots (spreading
// the atomic traffic over DSLOTS L2 lines); sweep n+1 starts by reading sweep n's
// slots and returns at once when δ_n <= tol, so a chunk of sweeps is enqueued
// without host round trips and without any grid-wide fence.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.cuh"
#include "tma.cuh"

namespace msb {

constexpr int DSLOTS = 16;
constexpr int SWEEP_BLOCK = 256;

__device__ __forceinline__ double nmax(double a, double b) { return (b > a || b != b) ? b : a; }

// true if the previous sweep already met the tolerance (block-uniform)
__device__ __forceinline__ bool sweep_skip(const unsigned long long* __restrict__ dslots, int n,
                                           double tol) {
  __shared__ int skip;
  if (threadIdx.x < 32) {
    double d = 0.0;
    if (n > 0 && tol >= 0.0 && threadIdx.x < DSLOTS)  // L2 read: written by the previous grid
      d = __longlong_as_double((long long)__ldcg(dslots + (n - 1) * DSLOTS + threadIdx.x));
    for (int o = 16; o > 0; o >>= 1) d = nmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (threadIdx.x == 0) skip = (n > 0 && tol >= 0.0 && d <= tol) ? 1 : 0;
  }
  __syncthreads();
  return skip != 0;
}

__device__ __forceinline__ void sweep_fold(double v, unsigned long long* __restrict__ dslots,
                                           int n) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w = nmax(w, __shfl_xor_sync(0xffffffffu, w, o));
    if (threadIdx.x == 0)
      atomicMax(dslots + n * DSLOTS + (blockIdx.x % DSLOTS),
                (unsigned long long)__double_as_longlong(w));
  }
}

// ---------------------------------------------------------------- G2: Cartesian sweep
// Per-axis coordinate masks (built once per level from the parity table):
//   bit p      slot parity p is a support of this coordinate
//   bit 2+p    the -1 neighbour holds the same column in parity p
//   bit 4+p    the +1 neighbour holds the same column in parity p
// so the sweep needs three byte loads per cell and no column arithmetic.
__global__ void k_axis_mask(const int32_t* __restrict__ tab, int n, int off,
                            uint8_t* __restrict__ mask) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int32_t* t = tab + 2 * (off + x);
  uint8_t m = 0;
  for (int p = 0; p < 2; ++p) {
    if (t[p] < 0) continue;
    m |= 1u << p;
    if (x > 0 && tab[2 * (off + x - 1) + p] == t[p]) m |= 1u << (2 + p);
    if (x < n - 1 && tab[2 * (off + x + 1) + p] == t[p]) m |= 1u << (4 + p);
  }
  mask[off + x] = m;
}

// Two threads per cell: lanes 0-15 of a warp take 16 consecutive cells for the four
// slots with z-parity 0, lanes 16-31 the same cells for z-parity 1, so every slot plane
// is read as 128-byte half-warp segments.  All loads are predicated selects (no
// branches), so the compiler issues a slot's seven loads back to back; inactive
// (cell, slot) pairs and masked neighbours fetch nothing.  The row sum (A6) is the two
// halves' partial sums joined by one shuffle.
__global__ void __launch_bounds__(SWEEP_BLOCK, 4) k_sweep_cart(
    double* __restrict__ P0, double* __restrict__ P1, const double* __restrict__ Tx,
    const double* __restrict__ Ty, const double* __restrict__ Tz, const uint8_t* __restrict__ amask,
    Grid3 g, double omega, int n, double tol, unsigned long long* __restrict__ dslots) {
  if (sweep_skip(dslots, n, tol)) return;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int N = g.nxy * g.nz;
  const int nx = g.nx, sxy = g.nxy;
  const int lane = threadIdx.x & 31, h = lane >> 4;
  const int c0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 16 + (lane & 15);
  const bool in = c0 < N;
  const int c = in ? c0 : N - 1;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const unsigned mx = amask[i], my = amask[nx + j], mz = amask[nx + g.ny + k];
  const double txp = Tx[c], typ = Ty[c], tzp = Tz[c];
  const double txm = i > 0 ? Tx[c - 1] : 0.0;
  const double tym = j > 0 ? Ty[c - nx] : 0.0;
  const double tzm = k > 0 ? Tz[c - sxy] : 0.0;
  const double D = txp + txm + typ + tym + tzp + tzm;
  const double wD = omega / D;
  const double om1 = 1.0 - omega;
  const bool zin = in && ((mz >> h) & 1u);
  const bool zm = (mz >> (2 + h)) & 1u, zp = (mz >> (4 + h)) & 1u;
  const double* __restrict__ base = Pin + (size_t)(4 * h) * N + c;
  double* __restrict__ obase = Pout + (size_t)(4 * h) * N + c;
  double po[4], ph[4];
  double sum = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int px = q & 1, py = q >> 1;
    const bool act = zin && ((mx >> px) & (my >> py) & 1u);
    const double* __restrict__ b = base + (size_t)q * N;
    const double vzm = (act && zm) ? b[-sxy] : 0.0;
    const double vym = (act && ((my >> (2 + py)) & 1u)) ? b[-nx] : 0.0;
    const double vxm = (act && ((mx >> (2 + px)) & 1u)) ? b[-1] : 0.0;
    const double vxp = (act && ((mx >> (4 + px)) & 1u)) ? b[1] : 0.0;
    const double vyp = (act && ((my >> (4 + py)) & 1u)) ? b[nx] : 0.0;
    const double vzp = (act && zp) ? b[sxy] : 0.0;
    const double p = act ? b[0] : 0.0;
    double acc = tzm * vzm;
    acc += tym * vym;
    acc += txm * vxm;
    acc += txp * vxp;
    acc += typ * vyp;
    acc += tzp * vzp;
    po[q] = p;
    ph[q] = act ? om1 * p + wD * acc : 0.0;
    sum += ph[q];
  }
  sum += __shfl_xor_sync(0xffffffffu, sum, 16);
  double dloc = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int px = q & 1, py = q >> 1;
    const bool act = zin && ((mx >> px) & (my >> py) & 1u);
    if (act) {
      const double pn = ph[q] / sum;
      obase[(size_t)q * N] = pn;
      dloc = nmax(dloc, fabs(pn - po[q]));
    }
  }
  sweep_fold(dloc, dslots, n);
}

// ---------------------------------------------------------------- G2': TMA-staged z-marching sweep
// The B200 path for grids whose x extent is even (TMA needs 16-byte global strides).
// A CTA owns a 32 x 4 column tile and marches it along z.  Each z plane of the tile
// plus its halo — all 8 slot planes of P and the three T planes — arrives in shared
// memory as two 4D TMA boxes (OOB halo zero-filled by the hardware) in a ring of
// TT_S stages signalled by mbarriers and prefetched TT_S-2 planes ahead.  Two threads
// per cell (lanes 0-15: slots with z-parity 0, lanes 16-31: z-parity 1, as in
// k_sweep_cart) read every neighbour from shared memory — the z neighbours are the
// ring's previous/next stage — so each P value crosses HBM once per sweep and the
// 28 neighbour reads per thread are LDS, not LDG.  Persistent CTAs take (x-tile,
// y-tile, z-chunk) items round-robin; the z-chunk length is chosen on the host to
// balance the items over the resident CTAs.  Same arithmetic as k_sweep_cart
// (masked transmissibilities multiply zero-filled values; the renormalisation is a
// reciprocal with one residual correction, i.e. the correctly rounded quotient).
// TMA requires the innermost box start to be 16-byte aligned, so the x halo is two
// cells wide on each side (box x range [x0-2, x0+34), x0 a multiple of 32).
constexpr int TT_X = 32, TT_Y = 4;

struct SweepTiles {
  int ntx, nty, kz, items;
};

// v if bit else +0.0, without a predicate (bit in {0, 1})
__device__ __forceinline__ double mask_d(double v, unsigned bit) {
  return __longlong_as_double(__double_as_longlong(v) & -(long long)bit);
}


// One thread per cell owns all 8 slots: the per-cell work (five T reads, D, 1/D, the
// twelve masked weights, the row sum, 1/sum, the store address) is done once (a
// two-threads-per-cell variant was issue-bound: profiles/r01_v9).  The TMA issue cursor
// runs ahead across items, so the next item's first planes load during the current
// item's last steps (no ring drain at item boundaries).
template <int TY>
struct SweepBox {
  static constexpr int BX = TT_X + 4;           // 2-cell x halo (16-byte TMA start)
  static constexpr int PPL = (TY + 2) * BX;     // one slot plane of the P box
  static constexpr int TPL = (TY + 1) * BX;     // one face-direction plane of the T box
  static constexpr int P_DBL = 8 * PPL;
  static constexpr int T_DBL = 3 * TPL;
  static constexpr int STAGE = ((P_DBL + T_DBL) * 8 + 127) / 128 * 128 / 8;
  static constexpr uint32_t TX = (uint32_t)(P_DBL + T_DBL) * 8u;
  static constexpr size_t smem(int S) { return (size_t)S * STAGE * 8 + 64; }
};

// v & m on both 32-bit halves (m all-ones or zero)
__device__ __forceinline__ double and_mask32(double v, unsigned m) {
  return __hiloint2double(__double2hiint(v) & (int)m, __double2loint(v) & (int)m);
}

__device__ __forceinline__ double and_mask(double v, unsigned long long m) {
  return __longlong_as_double((long long)((unsigned long long)__double_as_longlong(v) & m));
}


// Grid-wide barrier for the persistent multi-sweep launch (all CTAs co-resident: the
// launch is cooperative).  The fences order this CTA's generic-proxy stores before the
// arrive and the other CTAs' stores before this CTA's next TMA (async-proxy) loads.
__device__ __forceinline__ void sweep_grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
}

// ---------------------------------------------------------------- G2-ws: warp-specialised ring
// k_sweep_tma8's arithmetic with a producer/consumer ring instead of CTA barriers: one
// producer warp (lane 0) streams the planes of all of this CTA's items through S stages,
// waiting on per-stage "empty" mbarriers; each of the TY consumer warps (one tile row
// of 32 cells) waits on the stage's "full" mbarrier, computes, and releases the plane
// with one arrive.  Warps never wait for each other, only for data, so a warp can run
// up to S-2 planes ahead of the slowest.  One launch runs `cnt` sweeps n0 .. n0+cnt-1
// with a grid barrier between them (persistent, cooperative launch), so the per-launch
// ramp and drain are paid once per chunk instead of once per sweep; the ring's phase
// counters run on across sweeps.  Every sweep first tests δ of the previous one and the
// whole grid stops at the same sweep (δ is final after the barrier).
template <int TY, int S>
__global__ void __launch_bounds__(32 * (TY + 1)) k_sweep_ws(
    const __grid_constant__ CUtensorMap mP0, const __grid_constant__ CUtensorMap mP1,
    const __grid_constant__ CUtensorMap mT, double* __restrict__ P0, double* __restrict__ P1,
    const uint8_t* __restrict__ amask, Grid3 g, SweepTiles tl, double omega, int n0, int cnt,
    double tol, unsigned long long* __restrict__ dslots, unsigned* __restrict__ gbar) {
  using B = SweepBox<TY>;
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * B::STAGE);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = g.nx, ny = g.ny, nz = g.nz, nxy = g.nxy, N = g.nxy * g.nz;
  const int tiles = tl.ntx * tl.nty;
  if (tid == 0) {
    if (smem_u32(sm) & 127u) __trap();  // TMA destinations must be 128-byte aligned
    for (int t = 0; t < S; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&empty[t], TY);
    }
    mbar_fence_init();
  }
  uint32_t q = 0, seq = 0;  // ring sequence: producer issue count / consumer item base
  // T (3 N doubles: 27 MB on config 2) is re-read by every sweep while both P buffers stream
  // through L2: its boxes are loaded with an evict-last priority so they stay resident across
  // the sweeps (35.2 -> 33.6 us per config-2 sweep; profiles/r02i/t_evict_last_ab.txt).  An
  // evict-first hint on the P boxes measured slower (the halo rows shared by neighbouring
  // CTAs are dropped before their second reader; profiles/r02i/sweep_tma_hint_ab.txt).
  const unsigned long long pol_t = l2_policy_evict_last();
  for (int j = 0; j < cnt; ++j) {
    const int n = n0 + j;
    if (j > 0) sweep_grid_sync(gbar, (unsigned)j * gridDim.x);
    if (sweep_skip(dslots, n, tol)) break;  // uniform: δ_{n-1} is final (its __syncthreads
                                            // also publishes the barrier init)
    double dloc = 0.0;
    if (warp == TY) {  // producer
      if (lane == 0) {
        const CUtensorMap* mIn = (n & 1) ? &mP1 : &mP0;
        for (int item = blockIdx.x; item < tl.items; item += gridDim.x) {
          const int xt = item % tl.ntx, yt = (item / tl.ntx) % tl.nty, zc = item / tiles;
          const int k0 = zc * tl.kz, np = min(k0 + tl.kz, nz) - k0 + 2;
          for (int p = 0; p < np; ++p, ++q) {
            const int slot = q % S;
            if (q >= (uint32_t)S) mbar_wait(&empty[slot], ((q / S) - 1) & 1u);
            double* st = sm + slot * B::STAGE;
            mbar_expect_tx(&full[slot], B::TX);
            tma_load_4d(st, mIn, &full[slot], xt * TT_X - 2, yt * TY - 1, k0 - 1 + p, 0);
            tma_load_4d_hint(st + B::P_DBL, &mT, &full[slot], xt * TT_X - 2, yt * TY - 1, k0 - 1 + p, 0, pol_t);
          }
        }
      }
    } else {  // consumers: warp = tile row
      double* __restrict__ Pout = (n & 1) ? P0 : P1;
      const double om1 = 1.0 - omega;
      const int tx = lane, ty = warp;
      const int loc = (ty + 1) * B::BX + (tx + 2);
      for (int item = blockIdx.x; item < tl.items; item += gridDim.x) {
        const int xt = item % tl.ntx, yt = (item / tl.ntx) % tl.nty, zc = item / tiles;
        const int x0 = xt * TT_X, y0 = yt * TY, k0 = zc * tl.kz, k1 = min(k0 + tl.kz, nz);
        const int np = k1 - k0 + 2;
        auto wait_full = [&](int p) {
          const uint32_t sq = seq + p;
          mbar_wait(&full[sq % S], (sq / S) & 1u);
        };
        auto release = [&](int p) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[(seq + p) % S]);
        };
        const int x = x0 + tx, y = y0 + ty;
        const bool inxy = x < nx && y < ny;
        const unsigned mx = inxy ? amask[x] : 0u, my = inxy ? amask[nx + y] : 0u;
        // loop-invariant x/y neighbour masks, one 32-bit word applied to both halves
        const unsigned mxm0 = 0u - ((mx >> 2) & 1u), mxm1 = 0u - ((mx >> 3) & 1u);
        const unsigned mxp0 = 0u - ((mx >> 4) & 1u), mxp1 = 0u - ((mx >> 5) & 1u);
        const unsigned mym0 = 0u - ((my >> 2) & 1u), mym1 = 0u - ((my >> 3) & 1u);
        const unsigned myp0 = 0u - ((my >> 4) & 1u), myp1 = 0u - ((my >> 5) & 1u);
        // active slots of this column: bit s set iff x parity s&1 and y parity (s>>1)&1
        // are supports here (the z parity is folded in per plane)
        const unsigned axy = ((mx & 1u) ? 0x55u : 0u) | ((mx & 2u) ? 0xAAu : 0u);
        const unsigned act_xy =
            axy & (((my & 1u) ? 0x33u : 0u) | ((my & 2u) ? 0xCCu : 0u)) & (inxy ? 0xFFu : 0u);
        unsigned mz_next = amask[nx + ny + k0];
        double pzm[8], tzm;
        wait_full(0);
        {
          const double* s0 = sm + (seq % S) * B::STAGE;
#pragma unroll
          for (int s = 0; s < 8; ++s) pzm[s] = s0[loc + s * B::PPL];
          tzm = s0[B::P_DBL + 2 * B::TPL + loc];
        }
        release(0);
        wait_full(1);
        double* __restrict__ pout = Pout + (size_t)(x + nx * y) + (size_t)k0 * nxy;
        for (int k = k0; k < k1; ++k) {
          const int pc = k - k0 + 1;
          const unsigned mz = mz_next;
          if (k + 1 < k1) mz_next = amask[nx + ny + k + 1];
          wait_full(pc + 1);
          const double* __restrict__ sC = sm + ((seq + pc) % S) * B::STAGE;
          const double* __restrict__ sP = sm + ((seq + pc + 1) % S) * B::STAGE;
          const double* __restrict__ tC = sC + B::P_DBL;
          const double txp = tC[loc], txm = tC[loc - 1];
          const double typ = tC[B::TPL + loc], tym = tC[B::TPL + loc - B::BX];
          const double tzp = tC[2 * B::TPL + loc];
          const double D = txp + txm + typ + tym + tzp + tzm;
          const double wD = inxy ? omega * rcp_fast(D) : 0.0;
          const double wxm0 = and_mask32(txm, mxm0), wxm1 = and_mask32(txm, mxm1);
          const double wxp0 = and_mask32(txp, mxp0), wxp1 = and_mask32(txp, mxp1);
          const double wym0 = and_mask32(tym, mym0), wym1 = and_mask32(tym, mym1);
          const double wyp0 = and_mask32(typ, myp0), wyp1 = and_mask32(typ, myp1);
          const double wzm0 = and_mask32(tzm, 0u - ((mz >> 2) & 1u));
          const double wzm1 = and_mask32(tzm, 0u - ((mz >> 3) & 1u));
          const double wzp0 = and_mask32(tzp, 0u - ((mz >> 4) & 1u));
          const double wzp1 = and_mask32(tzp, 0u - ((mz >> 5) & 1u));
          double ph[8], po[8];
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
            const int o = loc + s * B::PPL;
            double acc = (pz ? wzm1 : wzm0) * pzm[s];
            acc += (py ? wym1 : wym0) * sC[o - B::BX];
            acc += (px ? wxm1 : wxm0) * sC[o - 1];
            acc += (px ? wxp1 : wxp0) * sC[o + 1];
            acc += (py ? wyp1 : wyp0) * sC[o + B::BX];
            acc += (pz ? wzp1 : wzp0) * sP[o];
            po[s] = sC[o];
            ph[s] = om1 * po[s] + wD * acc;
          }
          release(pc);  // plane pc is read for the last time above
          double slo = 0.0, shi = 0.0;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            slo += ph[s];
            shi += ph[4 + s];
          }
          const double sum = slo + shi;
          // inactive (cell, slot) entries have ph = po = 0 exactly, so they add 0 to δ
          // and only their stores need the activity predicate
          const unsigned act = act_xy & (((mz & 1u) ? 0x0Fu : 0u) | ((mz & 2u) ? 0xF0u : 0u));
          if (inxy) {
            const double rs = rcp_fast(sum);
            double* __restrict__ qo = pout;
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              const double pn = div_rn(ph[s], sum, rs);
              if ((act >> s) & 1u) *qo = pn;
              qo += N;
              const double d = fabs(pn - po[s]);
              dloc = d > dloc ? d : dloc;
            }
          }
#pragma unroll
          for (int s = 0; s < 8; ++s) pzm[s] = po[s];
          tzm = tzp;
          pout += nxy;
        }
        release(np - 1);
        seq += np;
      }
    }
    sweep_fold(dloc, dslots, n);
  }
}

// Zero diagonal of A_T: a cell with no open face (D_T = 0) has no
// smoothing update.  Checked once per msb_smooth_basis call, so the sweep kernels need
// no per-step NaN bookkeeping.
__global__ void k_zero_diag(const double* __restrict__ Tx, const double* __restrict__ Ty,
                            const double* __restrict__ Tz, Grid3 g, int* __restrict__ flag) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  const double D = Tx[c] + (i > 0 ? Tx[c - 1] : 0.0) + Ty[c] + (j > 0 ? Ty[c - g.nx] : 0.0) +
                   Tz[c] + (k > 0 ? Tz[c - g.nxy] : 0.0);
  if (!(D > 0.0)) atomicExch(flag, 1);
}

// ---------------------------------------------------------------- G3: explicit (ELL) sweep
constexpr int ELL_MAXW = 16;

__global__ void __launch_bounds__(SWEEP_BLOCK) k_sweep_ell(
    double* __restrict__ P0, double* __restrict__ P1, const double* __restrict__ Tx,
    const double* __restrict__ Ty, const double* __restrict__ Tz, const int32_t* __restrict__ col,
    const int8_t* __restrict__ nbs, int W, Grid3 g, double omega, int n, double tol,
    unsigned long long* __restrict__ dslots) {
  if (sweep_skip(dslots, n, tol)) return;
  const double* __restrict__ Pin = (n & 1) ? P1 : P0;
  double* __restrict__ Pout = (n & 1) ? P0 : P1;
  const int N = g.nxy * g.nz;
  const int nx = g.nx, sxy = g.nxy;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double dloc = 0.0;
  if (c < N) {
    int i, j, k;
    g3_coords(g, c, i, j, k);
    double t[6];
    int nb[6];
    t[0] = k > 0 ? Tz[c - sxy] : 0.0;       nb[0] = c - sxy;
    t[1] = j > 0 ? Ty[c - nx] : 0.0;        nb[1] = c - nx;
    t[2] = i > 0 ? Tx[c - 1] : 0.0;         nb[2] = c - 1;
    t[3] = Tx[c];                           nb[3] = c + 1;
    t[4] = Ty[c];                           nb[4] = c + nx;
    t[5] = Tz[c];                           nb[5] = c + sxy;
    double D = t[3] + t[2] + t[4] + t[1] + t[5] + t[0];
    double wD = omega / D;
    double om1 = 1.0 - omega;
    double ph[ELL_MAXW], po[ELL_MAXW];
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < ELL_MAXW; ++s) {
      ph[s] = 0.0;
      po[s] = 0.0;
      if (s < W && col[(size_t)s * N + c] >= 0) {
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          int sl = nbs[((size_t)d * W + s) * N + c];
          if (sl >= 0) acc += t[d] * Pin[(size_t)sl * N + nb[d]];
        }
        double p = Pin[(size_t)s * N + c];
        po[s] = p;
        ph[s] = om1 * p + wD * acc;
        sum += ph[s];
      }
    }
#pragma unroll
    for (int s = 0; s < ELL_MAXW; ++s) {
      if (s < W && col[(size_t)s * N + c] >= 0) {
        double pn = ph[s] / sum;
        Pout[(size_t)s * N + c] = pn;
        dloc = nmax(dloc, fabs(pn - po[s]));
      }
    }
  }
  sweep_fold(dloc, dslots, n);
}

using SweepKernMulti = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, double*,
                                double*, const uint8_t*, Grid3, SweepTiles, double, int, int,
                                double, unsigned long long*, unsigned*);
struct SweepLaunch {
  SweepKernMulti multi = nullptr;  // a chunk of sweeps per (cooperative) launch
  int threads = 0, ty = 0, occ = 0;
  size_t smem = 0;
};

template <typename K>
static cudaError_t sweep_setup_common(SweepLaunch* out, K kern, int threads, int ty, size_t smem) {
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (err != cudaSuccess) return err;
  out->threads = threads;
  out->ty = ty;
  out->occ = occ < 1 ? 1 : occ;
  out->smem = smem;
  return cudaSuccess;
}
static cudaError_t sweep_setup(SweepLaunch* out, SweepKernMulti kern, int threads, int ty,
                               size_t smem) {
  out->multi = kern;
  return sweep_setup_common(out, kern, threads, ty, smem);
}

// The sweep kernel: warp-specialised TMA ring, persistent over a chunk of sweeps
// (4 consumer warps, 3 ring stages; DESIGN.md §4.1 lists the variants measured).
static cudaError_t sweep_variant(SweepLaunch* out) {
  return sweep_setup(out, k_sweep_ws<4, 3>, 160, 4, SweepBox<4>::smem(3) + 64);
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_smooth_basis(msb_ctx ctx, msb_level L, msb_op op, int32_t max_sweeps,
                                       double omega, double tol, int32_t* sweeps_done,
                                       double* last_delta, double* deltas) {
  MSB_NVTX("msb_smooth_basis");
  if (!ctx || !L || !op) return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: null");
  if (max_sweeps < 0 || !(omega > 0.0) || !(omega <= 1.0))
    return set_error(ctx, MSB_EINVAL, "msb_smooth_basis: bad max_sweeps/omega");
  if (L->N != op->N) return set_error(ctx, MSB_EDIM, "level/operator size mismatch");
  if (L->kind == 1 && L->W > ELL_MAXW)
    return set_error(ctx, MSB_EINVAL, "ELL width %d exceeds %d", L->W, ELL_MAXW);
  if (sweeps_done) *sweeps_done = 0;
  if (last_delta) *last_delta = 0.0;
  if (max_sweeps == 0) return MSB_OK;
  cudaStream_t st = ctx->stream;
  // δ slots per sweep, then one 128-byte line for the multi-sweep grid barrier counter
  unsigned long long* dslots =
      dalloc_n<unsigned long long>(ctx, (size_t)max_sweeps * DSLOTS + DSLOTS);
  if (!dslots) return set_error(ctx, MSB_ENOMEM, "sweep state");
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(dslots, 0, ((size_t)max_sweeps * DSLOTS + DSLOTS) * 8, st));
  unsigned* gbar = reinterpret_cast<unsigned*>(dslots + (size_t)max_sweeps * DSLOTS);
  Grid3 g = make_grid3(op->nx, op->ny, op->nz);
  {
    int* zf = dalloc_n<int>(ctx, 1);
    if (!zf) return set_error(ctx, MSB_ENOMEM, "zero-diagonal flag");
    MSB_CUDA_TRY(ctx, cudaMemsetAsync(zf, 0, sizeof(int), st));
    k_zero_diag<<<grid_for(op->N, 256), 256, 0, st>>>(op->Tx, op->Ty, op->Tz, g, zf);
    MSB_LAUNCH_CHECK(ctx);
    int hz = 0;
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hz, zf, sizeof(int), cudaMemcpyDeviceToHost, st));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, zf);
    if (hz) {
      dfree(ctx, dslots);
      return set_error(ctx, MSB_EZERO_DIAG, "zero diagonal in A_T (a cell with no open face)");
    }
  }
  L->unity = true;  // every sweep renormalises the rows of P to sum to one
  if (L->kind == 0 && !L->amask) {
    int tot = op->nx + op->ny + op->nz;
    MSB_ALLOC(ctx, L->amask, uint8_t, tot);
    int dims[3] = {op->nx, op->ny, op->nz};
    int off = 0;
    for (int a = 0; a < 3; ++a) {
      k_axis_mask<<<grid_for(dims[a], 128), 128, 0, st>>>(L->tab, dims[a], off, L->amask);
      MSB_LAUNCH_CHECK(ctx);
      off += dims[a];
    }
  }
  double* Pa = L->P[L->cur];
  double* Pb = L->P[L->cur ^ 1];
  // TMA path: tensor maps over both P buffers and the 3N transmissibility block.
  bool use_tma = false;
  CUtensorMap mP[2], mT;
  SweepTiles tl{};
  unsigned tgrid = 0;
  SweepLaunch sl{};
  if (L->kind == 0 && (op->nx % 2) == 0) {
    static SweepLaunch cached{};
    if (!cached.multi) MSB_CUDA_TRY(ctx, sweep_variant(&cached));
    sl = cached;
    const uint64_t dP[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 8};
    const uint64_t dT[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 3};
    const uint64_t st3[3] = {(uint64_t)op->nx, (uint64_t)op->nx * op->ny, (uint64_t)L->N};
    const uint32_t bP[4] = {TT_X + 4, (uint32_t)sl.ty + 2, 1, 8};
    const uint32_t bT[4] = {TT_X + 4, (uint32_t)sl.ty + 1, 1, 3};
    use_tma = tma_encode_4d(&mP[0], Pa, dP, st3, bP) && tma_encode_4d(&mP[1], Pb, dP, st3, bP) &&
              tma_encode_4d(&mT, op->Tx, dT, st3, bT);
    if (use_tma) {
      tl.ntx = (op->nx + TT_X - 1) / TT_X;
      tl.nty = (op->ny + sl.ty - 1) / sl.ty;
      const int64_t slots = (int64_t)sl.occ * ctx->sm_count;
      const int64_t tiles = (int64_t)tl.ntx * tl.nty;
      // z-chunking: minimise (waves) x (planes per item incl. 2 halo planes)
      int64_t best = INT64_MAX;
      for (int nzc = 1; nzc <= op->nz; ++nzc) {
        int kz = (op->nz + nzc - 1) / nzc;
        int64_t items = tiles * ((op->nz + kz - 1) / kz);
        int64_t waves = (items + slots - 1) / slots;
        int64_t cost = waves * (kz + 2);
        if (cost < best) {
          best = cost;
          tl.kz = kz;
          tl.items = (int)items;
        }
      }
      tgrid = (unsigned)std::min<int64_t>(tl.items, slots);
    }
  }
  const unsigned grid = L->kind == 0 ? grid_for(L->N * 2, SWEEP_BLOCK) : grid_for(L->N, SWEEP_BLOCK);
  const int chunk = 32;
  int issued = 0, n = 0;
  double last = 0.0;
  bool bad = false, done = false;
  // Chunks of up to 32 sweeps are enqueued without host round trips; each chunk's δ slots
  // are copied to pinned memory behind it, and the host reads chunk c while chunk c+1
  // runs (two-deep pipeline).  Sweeps after convergence return at entry (δ_{n-1} <= tol),
  // so the over-issued chunk costs one empty launch.
  unsigned long long* hbuf =
      static_cast<unsigned long long*>(pinned_scratch(ctx, 2 * (size_t)chunk * DSLOTS * 8));
  if (!hbuf) {
    dfree(ctx, dslots);
    return set_error(ctx, MSB_ENOMEM, "pinned readback buffer");
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (auto& e : ev) MSB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int c_first[2] = {0, 0}, c_n[2] = {0, 0};
  auto launch_chunk = [&](int b) -> msb_status {
    const int nl = std::min(chunk, max_sweeps - issued);
    if (use_tma && sl.multi) {
      // the chunk's sweeps in one cooperative launch (grid barrier between sweeps)
      MSB_CUDA_TRY(ctx, cudaMemsetAsync(gbar, 0, sizeof(unsigned), st));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(tgrid);
      cfg.blockDim = dim3(sl.threads);
      cfg.dynamicSmemBytes = sl.smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      MSB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, sl.multi, mP[0], mP[1], mT, Pa, Pb,
                                           (const uint8_t*)L->amask, g, tl, omega, issued, nl, tol,
                                           dslots, gbar));
    } else {
      for (int t = 0; t < nl; ++t) {
        const int idx = issued + t;
        if (L->kind == 0)
          k_sweep_cart<<<grid, SWEEP_BLOCK, 0, st>>>(Pa, Pb, op->Tx, op->Ty, op->Tz, L->amask, g,
                                                     omega, idx, tol, dslots);
        else
          k_sweep_ell<<<grid, SWEEP_BLOCK, 0, st>>>(Pa, Pb, op->Tx, op->Ty, op->Tz, L->col, L->nbs,
                                                    L->W, g, omega, idx, tol, dslots);
        MSB_LAUNCH_CHECK(ctx);
      }
    }
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hbuf + (size_t)b * chunk * DSLOTS,
                                      dslots + (size_t)issued * DSLOTS, (size_t)nl * DSLOTS * 8,
                                      cudaMemcpyDeviceToHost, st));
    MSB_CUDA_TRY(ctx, cudaEventRecord(ev[b], st));
    c_first[b] = issued;
    c_n[b] = nl;
    issued += nl;
    return MSB_OK;
  };
  msb_status lrc = MSB_OK;
  int cb = 0;
  if (max_sweeps > 0) lrc = launch_chunk(0);
  while (!lrc) {
    const bool more = issued < max_sweeps;
    if (more && (lrc = launch_chunk(cb ^ 1))) break;
    if (cudaEventSynchronize(ev[cb]) != cudaSuccess) {
      lrc = set_error(ctx, MSB_ECUDA, "sweep chunk: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    const unsigned long long* hb = hbuf + (size_t)cb * chunk * DSLOTS;
    for (int t = 0; t < c_n[cb] && !done; ++t) {
      double d = 0.0;
      for (int q = 0; q < DSLOTS; ++q) {
        double v;
        memcpy(&v, &hb[(size_t)t * DSLOTS + q], 8);
        d = (v > d || v != v) ? v : d;
      }
      if (!(d == d)) bad = true;
      if (deltas) deltas[c_first[cb] + t] = d;
      last = d;
      n = c_first[cb] + t + 1;
      if (tol >= 0.0 && d <= tol) done = true;
    }
    if (done || !more) break;
    cb ^= 1;
  }
  cudaStreamSynchronize(st);  // an over-issued chunk may still be running
  for (auto& e : ev) cudaEventDestroy(e);
  if (lrc) {
    dfree(ctx, dslots);
    return lrc;
  }
  dfree(ctx, dslots);
  if (n & 1) L->cur ^= 1;
  if (sweeps_done) *sweeps_done = n;
  if (last_delta) *last_delta = last;
  if (bad) return set_error(ctx, MSB_EZERO_DIAG, "non-finite update: zero diagonal in A_T");
  if (tol >= 0.0 && !done) return MSB_NOT_CONVERGED;
  return MSB_OK;
}
