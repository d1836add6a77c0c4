// Rows a6 + a8 fused for the Cartesian level on B200: r = b - A x and r_c = P^T r in
// one TMA-staged z-marching pass (the sweep's tiling, sweep.cu), instead of a residual
// pass that materialises r plus a gather pass that re-reads it.
//
// A CTA owns a 32 x 4 column tile and marches it along z.  Per z plane one mbarrier
// stage receives four TMA boxes: x (tile + 2/1-cell x/y halo, zero-filled outside the
// grid), b (tile), the three T planes (tile + minus-side halo) and the 8 P slot planes
// (tile).  Two threads per cell (z-parity halves of the 8 slots, as the sweep): both
// evaluate r at the cell from shared memory, each accumulates P_s r for its 4 slots in
// registers while the slot's column does not change along z — along a z column the
// column index of slot s changes only where its z block changes — and flushes the
// running sum with one fp64 atomicAdd when it does.  So the restriction costs ~1
// atomic per 2.5 P entries instead of a separate pass over P and r.
//
// The reduction order of r_c is therefore not fixed (atomics): results agree with the
// gather path to rounding (tests/test_gpu_parity.py tolerances), not bitwise.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.cuh"
#include "tma.cuh"

namespace msb {

constexpr int RT_X = 32, RT_Y = 4;
constexpr int RX_X = RT_X + 4, RX_Y = RT_Y + 2;       // x box: [x0-2, x0+34) x [y0-1, y0+5)
constexpr int RQ_Y = RT_Y + 1;                        // T box rows [y0-1, y0+4)
constexpr int RX_DBL = RX_X * RX_Y;                   // 216
constexpr int RB_DBL = RT_X * RT_Y;                   // 128 (b tile)
constexpr int RQ_DBL = 3 * RX_X * RQ_Y;               // 540
constexpr int RP_DBL = 8 * RT_X * RT_Y;               // 1024 (P tile, 8 slot planes)
// every TMA destination 128-byte (16-double) aligned
constexpr int al16(int d) { return (d + 15) / 16 * 16; }
constexpr int R_OFF_B = al16(RX_DBL);
constexpr int R_OFF_T = al16(R_OFF_B + RB_DBL);
constexpr int R_OFF_P = al16(R_OFF_T + RQ_DBL);
constexpr int RSTAGE_DBL = al16(R_OFF_P + RP_DBL);
constexpr uint32_t RSTAGE_TX = (uint32_t)(RX_DBL + RB_DBL + RQ_DBL + RP_DBL) * 8u;
constexpr size_t rr_smem(int S) { return (size_t)S * RSTAGE_DBL * 8 + 64; }
constexpr int RR_THREADS = 2 * RT_X * RT_Y;
constexpr int RR_STAGES_DEFAULT = 4;  // ring depth (MSB_RR_STAGES=4|6|8 to A/B)

struct RRTiles {
  int ntx, nty, kz, items;
};

template <int RT_S>
__global__ void __launch_bounds__(RR_THREADS) k_resrestrict_tma(
    const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mB,
    const __grid_constant__ CUtensorMap mT, const __grid_constant__ CUtensorMap mP,
    const int32_t* __restrict__ tab, int nb0, int nb1, Grid3 g, RRTiles tl,
    double* __restrict__ rc, int first, double* __restrict__ partials, const int* done_flag) {
  const bool done = *(volatile const int*)done_flag != 0;
  extern __shared__ __align__(128) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + RT_S * RSTAGE_DBL);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, h = lane >> 4;
  const int ty = w >> 1, tx = ((w & 1) << 4) + (lane & 15);
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  if (tid == 0) {
    if (smem_u32(sm) & 127u) __trap();
    for (int t = 0; t < RT_S; ++t) mbar_init(&bars[t], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int xl = (ty + 1) * RX_X + (tx + 2);   // cell in the x and T boxes
  const int bl = ty * RT_X + tx;               // cell in the b and P tiles
  uint32_t seq = 0;
  double nrm = 0.0;
  for (int item = blockIdx.x; item < tl.items; item += gridDim.x) {
    const int xt = item % tl.ntx, rest = item / tl.ntx;
    const int yt = rest % tl.nty, zc = rest / tl.nty;
    const int x0 = xt * RT_X, y0 = yt * RT_Y, k0 = zc * tl.kz, k1 = min(k0 + tl.kz, nz);
    const int np = k1 - k0 + 2;  // x planes k0-1 .. k1 (b, T, P are read at the same z)
    auto issue = [&](int p) {
      const uint32_t sq = seq + p;
      const int slot = sq % RT_S;
      double* st = sm + slot * RSTAGE_DBL;
      const int z = k0 - 1 + p;
      mbar_expect_tx(&bars[slot], RSTAGE_TX);
      tma_load_4d(st, &mX, &bars[slot], x0 - 2, y0 - 1, z, 0);  // rank-4 maps, unit 4th extent
      tma_load_4d(st + R_OFF_B, &mB, &bars[slot], x0, y0, z, 0);
      tma_load_4d(st + R_OFF_T, &mT, &bars[slot], x0 - 2, y0 - 1, z, 0);
      tma_load_4d(st + R_OFF_P, &mP, &bars[slot], x0, y0, z, 0);
    };
    auto wait = [&](int p) {
      const uint32_t sq = seq + p;
      mbar_wait(&bars[sq % RT_S], (sq / RT_S) & 1u);
    };
    // ring holds planes pc..pc+RT_S-1 in step pc; the own-column minus-z values (x and
    // Tz at k-1) are carried in registers, so RT_S-2 planes are in flight ahead of need
    if (tid == 0)
      for (int p = 0; p < min(RT_S, np); ++p) issue(p);
    const int x = x0 + tx, y = y0 + ty;
    const bool inxy = x < nx && y < ny;
    const int2 jxp = inxy ? reinterpret_cast<const int2*>(tab)[x] : make_int2(-1, -1);
    const int2 jyp = inxy ? reinterpret_cast<const int2*>(tab)[nx + y] : make_int2(-1, -1);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int jz_run = -1;  // column block along z of this thread's parity for the running sums
    auto flush = [&]() {
      if (jz_run >= 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int jx = (q & 1) ? jxp.y : jxp.x, jy = (q >> 1) ? jyp.y : jyp.x;
          if (jx >= 0 && jy >= 0 && acc[q] != 0.0 && !done)
            atomicAdd(rc + jx + nb0 * (jy + nb1 * jz_run), acc[q]);
          acc[q] = 0.0;
        }
      }
    };
    double xzm, tzm;
    wait(0);
    {
      const double* s0 = sm + (seq % RT_S) * RSTAGE_DBL;
      xzm = s0[xl];
      tzm = s0[R_OFF_T + 2 * RX_X * RQ_Y + xl];
    }
    // z block of this thread's parity per plane, prefetched one plane ahead so the
    // table load's latency never sits at the head of a step
    int jz_next = inxy ? tab[2 * (nx + ny + k0) + h] : -1;
    for (int k = k0; k < k1; ++k) {
      const int pc = k - k0 + 1;
      const int jz = jz_next;
      if (k + 1 < k1) jz_next = inxy ? tab[2 * (nx + ny + k + 1) + h] : -1;
      if (pc == 1) wait(1);
      wait(pc + 1);
      if (jz != jz_run) {
        flush();
        jz_run = jz;
      }
      const double* __restrict__ sC = sm + ((seq + pc) % RT_S) * RSTAGE_DBL;
      const double* __restrict__ sP = sm + ((seq + pc + 1) % RT_S) * RSTAGE_DBL;
      if (inxy) {
        const double* tC = sC + R_OFF_T;
        const double txp = tC[xl], txm = tC[xl - 1];
        const double typ = tC[RX_X * RQ_Y + xl], tym = tC[RX_X * RQ_Y + xl - RX_X];
        const double tzp = tC[2 * RX_X * RQ_Y + xl];
        const double D = txp + txm + typ + tym + tzp + tzm;
        // zero-filled halo x values meet zero transmissibilities at the boundary, in the
        // order of residual_at (cycle.cu)
        double off = tzm * xzm;
        off += tym * sC[xl - RX_X];
        off += txm * sC[xl - 1];
        off += txp * sC[xl + 1];
        off += typ * sC[xl + RX_X];
        off += tzp * sP[xl];
        const int c = x + nx * (y + ny * k);
        const double dA = (c == 0) ? 2.0 * D : D;
        const double r = sC[R_OFF_B + bl] - (dA * sC[xl] - off);
        if (h == 0) nrm += r * r;
        const double* pt = sC + R_OFF_P + 4 * h * RT_X * RT_Y + bl;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(pt[q * RT_X * RT_Y], r, acc[q]);
      }
      xzm = sC[xl];
      tzm = sC[R_OFF_T + 2 * RX_X * RQ_Y + xl];
      __syncthreads();  // plane pc-1's ring slot is free
      if (tid == 0) {
        fence_proxy_async_smem();
        if (pc - 1 + RT_S < np) issue(pc - 1 + RT_S);
      }
    }
    flush();
    jz_run = -1;
    seq += np;
  }
  if (first) {
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) sh[w] = nrm;
    __syncthreads();
    if (tid < 32) {
      double v = tid < (RR_THREADS >> 5) ? sh[tid] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) partials[blockIdx.x] = v;
    }
  }
}

// Host side: tensor maps + tiling; returns false (caller falls back to the two-pass
// path) when TMA cannot describe the layout (odd nx) or the driver refuses.
bool resrestrict_plan(msb_ctx ctx, msb_op op, msb_level L, const double* x, const double* b,
                      RRLaunch* out) {
  if (L->kind != 0 || (op->nx % 2) != 0) return false;
  const uint64_t N = (uint64_t)L->N;
  const uint64_t d3[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 1};
  const uint64_t s3[3] = {(uint64_t)op->nx, (uint64_t)op->nx * op->ny, N};
  const uint64_t dT[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 3};
  const uint64_t dP[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 8};
  const uint32_t bX[4] = {RX_X, RX_Y, 1, 1}, bB[4] = {RT_X, RT_Y, 1, 1};
  const uint32_t bT[4] = {RX_X, RQ_Y, 1, 3}, bP[4] = {RT_X, RT_Y, 1, 8};
  // rank-3 maps are encoded as rank 4 with a unit outer extent
  if (!tma_encode_4d(&out->mX, x, d3, s3, bX) || !tma_encode_4d(&out->mB, b, d3, s3, bB) ||
      !tma_encode_4d(&out->mT, op->Tx, dT, s3, bT) ||
      !tma_encode_4d(&out->mP, L->P[L->cur], dP, s3, bP))
    return false;
  static int occ = 0, stages = 0;
  if (!occ) {
    const char* e = getenv("MSB_RR_STAGES");
    stages = e ? atoi(e) : RR_STAGES_DEFAULT;
    if (stages != 4 && stages != 6 && stages != 8) stages = RR_STAGES_DEFAULT;
    cudaError_t err = cudaSuccess;
    auto setup = [&](auto kern, int S) {
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rr_smem(S));
      if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, RR_THREADS, rr_smem(S));
    };
    if (stages == 4) setup(k_resrestrict_tma<4>, 4);
    else if (stages == 6) setup(k_resrestrict_tma<6>, 6);
    else setup(k_resrestrict_tma<8>, 8);
    if (err != cudaSuccess) {
      cudaGetLastError();
      occ = 0;
      return false;
    }
    if (occ < 1) occ = 1;
  }
  out->stages = stages;
  RRTiles tl{};
  tl.ntx = (op->nx + RT_X - 1) / RT_X;
  tl.nty = (op->ny + RT_Y - 1) / RT_Y;
  const int64_t slots = (int64_t)occ * ctx->sm_count;
  const int64_t tiles = (int64_t)tl.ntx * tl.nty;
  int64_t best = INT64_MAX;
  for (int nzc = 1; nzc <= op->nz; ++nzc) {
    const int kz = (op->nz + nzc - 1) / nzc;
    const int64_t items = tiles * ((op->nz + kz - 1) / kz);
    const int64_t waves = (items + slots - 1) / slots;
    const int64_t cost = waves * (kz + 2);
    if (cost < best) {
      best = cost;
      tl.kz = kz;
      tl.items = (int)items;
    }
  }
  out->ntx = tl.ntx;
  out->nty = tl.nty;
  out->kz = tl.kz;
  out->items = tl.items;
  out->grid = (unsigned)std::min<int64_t>(tl.items, slots);
  return true;
}

msb_status resrestrict_launch(msb_ctx ctx, msb_op op, msb_level L, const RRLaunch& P, double* rc,
                              int first, double* partials, const int* done) {
  RRTiles tl{P.ntx, P.nty, P.kz, P.items};
  const Grid3 g = make_grid3(op->nx, op->ny, op->nz);
#define MSB_RR_LAUNCH(S)                                                                       \
  k_resrestrict_tma<S><<<P.grid, RR_THREADS, rr_smem(S), ctx->stream>>>(                       \
      P.mX, P.mB, P.mT, P.mP, L->tab, L->nb[0], L->nb[1], g, tl, rc, first, partials, done)
  if (P.stages == 4) MSB_RR_LAUNCH(4);
  else if (P.stages == 6) MSB_RR_LAUNCH(6);
  else MSB_RR_LAUNCH(8);
#undef MSB_RR_LAUNCH
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

}  // namespace msb
