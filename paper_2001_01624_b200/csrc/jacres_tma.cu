// Rows a7 + a6 fused for the B200 (Cartesian level, ν = 1, pre-smoothing):
//   x1 = x + ω_s D_A^{-1} (b - A x)      (damped Jacobi; reading A9)
//   r1 = b - A x1                        (the residual the coarse correction restricts)
// in ONE z-marching pass, instead of a Jacobi pass and a residual pass that each read
// x, b and the three transmissibility planes (ncu, config 2: 16.4 + 13.4 us).
//
// A CTA owns a 32 x 4 column tile and a z-chunk.  A producer warp streams, per z plane,
// three TMA boxes into an S-stage mbarrier ring: x over the tile plus a 2-cell x/y halo,
// b over the tile plus 1, and the three T planes over the tile plus [2 below, 1 above]
// in y (OOB zero-filled; T is cell-padded, so boundary faces are 0).  Four consumer
// warps march z: at plane z they evaluate the Jacobi update on the tile plus a 1-cell
// halo (34 x 6 cells) into a 4-plane shared x1 ring, then — one named barrier later —
// the residual of x1 at plane z-1 on the tile, and store x1 and r1 there.  x, b and T
// cross HBM once per iteration; the Jacobi work on the halo (204 vs 128 cells) and the
// 2-plane z halo of each chunk are recomputation/L2 traffic, not HBM.
//
// Arithmetic is term-for-term that of residual_at (cycle.cu): D = Σ T in the same order,
// the off-diagonal sum in the order -z, -y, -x, +x, +y, +z, the gauge A_00 = 2 D at cell
// 0, r = b - (D_A x - off), x1 = x + ω (r / D_A); a missing neighbour contributes
// T = 0 times a zero-filled x, which leaves the sum unchanged.  Cells outside the grid
// get x1 = 0.  The stop-test partial is ||b - A x||² over this CTA's tile cells, one
// per CTA (deterministic for a fixed grid).
//
// Used when the grid's Jacobi/residual working set (x, b, T: 5 N doubles) is well beyond
// the L2 (jacres_fused_wanted: config 5).  On config 2 (1.1M cells) the separate residual
// pass reads x1, b and T from L2 right after the Jacobi pass (ncu: ~0 DRAM bytes), so the
// fusion saves little HBM traffic while its z-march serialises ~26 dependent plane steps
// per CTA (76.6-84 us against 71.8 us per iteration, profiles/r01_v10); at 10M cells both
// passes stream from HBM and the fusion removes the second one.  The quotient is formed
// as in k_jacobi (div_rn), so x1 and r1 are bit-identical to the two-pass path.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.cuh"
#include "tma.cuh"

namespace msb {

constexpr int JQ_TX = 32;
constexpr int JQ_BX = JQ_TX + 4;  // box width: x0-2 .. x0+33 (16-byte start)
constexpr int jq_al16(int d) { return (d + 15) / 16 * 16; }
template <int TY>
struct JQBox {
  static constexpr int XR = TY + 4;  // x box rows y0-2 .. y0+TY+1
  static constexpr int BR = TY + 2;  // b box rows y0-1 .. y0+TY
  static constexpr int TR = TY + 3;  // T box rows y0-2 .. y0+TY
  static constexpr int HX = JQ_TX + 2, HY = TY + 2, HC = HX * HY;  // Jacobi region
  static constexpr int OB = jq_al16(XR * JQ_BX);
  static constexpr int OT = OB + jq_al16(BR * JQ_BX);
  static constexpr int TPL = TR * JQ_BX;  // one face plane of the T box
  static constexpr int STAGE = jq_al16(OT + 3 * TPL);
  static constexpr uint32_t BYTES = (uint32_t)(XR * JQ_BX + BR * JQ_BX + 3 * TPL) * 8u;
  static constexpr int X1 = 4, X1P = jq_al16(HC);  // x1 ring planes
  static constexpr int CONS = 32 * TY;              // consumer threads (one warp per tile row)
  static constexpr size_t smem(int S) { return ((size_t)S * STAGE + X1 * X1P) * 8 + 128; }
};

struct JQTiles {
  int ntx, nty, kz, items;
};

template <int CONS>
__device__ __forceinline__ void jq_consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CONS) : "memory");
}

template <int TY, int S>
__global__ void __launch_bounds__(32 * TY + 32) k_jacres_tma(
    const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mB,
    const __grid_constant__ CUtensorMap mT, double* __restrict__ xo, double* __restrict__ rout,
    Grid3 g, JQTiles tl, double omega, int first, double* __restrict__ partials,
    const int* done_flag) {
  using B = JQBox<TY>;
  if (*(volatile const int*)done_flag) return;  // converged: no stores, no partial
  extern __shared__ __align__(128) double sm[];
  double* x1s = sm + S * B::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(x1s + B::X1 * B::X1P);
  uint64_t* empty = full + S;
  __shared__ double red[TY];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = g.nx, ny = g.ny, nz = g.nz, nxy = g.nxy;
  const int tiles = tl.ntx * tl.nty;
  if (tid == 0) {
    if (smem_u32(sm) & 127u) __trap();  // TMA destinations must be 128-byte aligned
    for (int t = 0; t < S; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&empty[t], TY);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == TY) {  // producer: planes k0-2 .. k1+1 of every item of this CTA
    if (lane == 0) {
      uint32_t q = 0;
      for (int item = blockIdx.x; item < tl.items; item += gridDim.x) {
        const int xt = item % tl.ntx, yt = (item / tl.ntx) % tl.nty, zc = item / tiles;
        const int x0 = xt * JQ_TX, y0 = yt * TY, k0 = zc * tl.kz;
        const int np = min(k0 + tl.kz, nz) - k0 + 4;
        for (int p = 0; p < np; ++p, ++q) {
          const int slot = q % S;
          if (q >= (uint32_t)S) mbar_wait(&empty[slot], ((q / S) - 1) & 1u);
          double* st = sm + slot * B::STAGE;
          const int z = k0 - 2 + p;
          mbar_expect_tx(&full[slot], B::BYTES);
          tma_load_4d(st, &mX, &full[slot], x0 - 2, y0 - 2, z, 0);
          tma_load_4d(st + B::OB, &mB, &full[slot], x0 - 2, y0 - 1, z, 0);
          tma_load_4d(st + B::OT, &mT, &full[slot], x0 - 2, y0 - 2, z, 0);
        }
      }
    }
    return;  // the producer takes no part in the consumers' named barriers
  }
  uint32_t seq = 0;
  double vsum = 0.0;
  for (int item = blockIdx.x; item < tl.items; item += gridDim.x) {
    const int xt = item % tl.ntx, yt = (item / tl.ntx) % tl.nty, zc = item / tiles;
    const int x0 = xt * JQ_TX, y0 = yt * TY, k0 = zc * tl.kz, k1 = min(k0 + tl.kz, nz);
    const int np = k1 - k0 + 4;  // planes k0-2 .. k1+1; plane index p = z - (k0 - 2)
    auto stage = [&](int p) -> const double* { return sm + ((seq + p) % S) * B::STAGE; };
    auto wait_full = [&](int p) {
      const uint32_t sq = seq + p;
      mbar_wait(&full[sq % S], (sq / S) & 1u);
    };
    auto release = [&](int p) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(seq + p) % S]);
    };
    auto x1slot = [&](int z) -> double* { return x1s + ((z - k0 + 1) & (B::X1 - 1)) * B::X1P; };
    wait_full(0);
    wait_full(1);
    for (int jz = k0 - 1; jz <= k1; ++jz) {
      const int pj = jz - k0 + 2;
      wait_full(pj + 1);
      const double* sD = stage(pj - 1);
      const double* sC = stage(pj);
      const double* sU = stage(pj + 1);
      // ---- Jacobi on the tile + 1-cell halo at plane jz
      double* x1w = x1slot(jz);
      const bool zin = jz >= 0 && jz < nz;
#pragma unroll
      for (int u = 0; u < (B::HC + B::CONS - 1) / B::CONS; ++u) {
        const int id = tid + u * B::CONS;
        if (id < B::HC) {
          const int hx = id % B::HX, hy = id / B::HX;
          const int gx = x0 - 1 + hx, gy = y0 - 1 + hy;
          const bool in = zin && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
          const int xi = (hy + 1) * JQ_BX + hx + 1;  // x and T boxes (rows from y0-2)
          const double* T = sC + B::OT;
          const double txp = T[xi], txm = T[xi - 1];
          const double typ = T[B::TPL + xi], tym = T[B::TPL + xi - JQ_BX];
          const double tzp = T[2 * B::TPL + xi], tzm = sD[B::OT + 2 * B::TPL + xi];
          const double D = txp + txm + typ + tym + tzp + tzm;
          double off = tzm * sD[xi];
          off += tym * sC[xi - JQ_BX];
          off += txm * sC[xi - 1];
          off += txp * sC[xi + 1];
          off += typ * sC[xi + JQ_BX];
          off += tzp * sU[xi];
          const double xc = sC[xi];
          const double dA = (gx == 0 && gy == 0 && jz == 0) ? 2.0 * D : D;
          const double r0 = sC[B::OB + hy * JQ_BX + hx + 1] - (dA * xc - off);
          x1w[id] = in ? xc + omega * div_rn(r0, dA, rcp_fast(dA)) : 0.0;
          if (in && hx >= 1 && hx <= JQ_TX && hy >= 1 && hy <= TY && jz >= k0 && jz < k1)
            vsum += r0 * r0;
        }
      }
      jq_consumer_sync<B::CONS>();  // x1 at plane jz complete
      // ---- residual of x1 at plane rz = jz - 1 on the tile
      const int rz = jz - 1;
      if (rz >= k0) {
        const int tx = lane, ty = warp;
        const int gx = x0 + tx, gy = y0 + ty;
        const double* sR = stage(pj - 1);   // plane rz: b, T
        const double* sRD = stage(pj - 2);  // plane rz-1: Tz below
        const int ti = (ty + 2) * JQ_BX + tx + 2;  // T box
        const double* T = sR + B::OT;
        const double txp = T[ti], txm = T[ti - 1];
        const double typ = T[B::TPL + ti], tym = T[B::TPL + ti - JQ_BX];
        const double tzp = T[2 * B::TPL + ti], tzm = sRD[B::OT + 2 * B::TPL + ti];
        const double D = txp + txm + typ + tym + tzp + tzm;
        const int hi = (ty + 1) * B::HX + tx + 1;  // x1 ring (34-wide)
        const double* xm = x1slot(rz - 1);
        const double* xcr = x1slot(rz);
        const double* xp = x1slot(rz + 1);
        double off = tzm * xm[hi];
        off += tym * xcr[hi - B::HX];
        off += txm * xcr[hi - 1];
        off += txp * xcr[hi + 1];
        off += typ * xcr[hi + B::HX];
        off += tzp * xp[hi];
        const double x1c = xcr[hi];
        const double dA = (gx == 0 && gy == 0 && rz == 0) ? 2.0 * D : D;
        const double r1 = sR[B::OB + (ty + 1) * JQ_BX + tx + 2] - (dA * x1c - off);
        if (gx < nx && gy < ny) {
          const size_t c = (size_t)gx + (size_t)nx * gy + (size_t)nxy * rz;
          xo[c] = x1c;
          rout[c] = r1;
        }
      }
      if (jz >= k0) release(pj - 2);  // plane jz-2: last read by this step's residual
    }
    release(np - 3);
    release(np - 2);
    release(np - 1);
    seq += np;
  }
  if (first) {  // ||b - A x||² over this CTA's tile cells, fixed order
    for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
    if (lane == 0) red[warp] = vsum;
    jq_consumer_sync<B::CONS>();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < TY; ++w) t += red[w];
      partials[blockIdx.x] = t;
    }
  }
}

using JQKern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, double*, double*,
                        Grid3, JQTiles, double, int, double*, const int*);

struct JQSel {
  JQKern kern = nullptr;
  int ty = 4, stages = 6, threads = 160, occ = 1;
  size_t smem = 0;
};

template <int TY, int S>
static void jq_pick(JQSel* o) {
  o->kern = k_jacres_tma<TY, S>;
  o->ty = TY;
  o->stages = S;
  o->threads = 32 * TY + 32;
  o->smem = JQBox<TY>::smem(S);
}

// 4 tile rows, 6 ring stages (the round-1 A/B: TY 4|8 x stages 4|5|6)
static cudaError_t jq_kernel(JQSel* out) {
  static JQSel sel;
  static cudaError_t err = cudaSuccess;
  if (!sel.kern) {
    jq_pick<4, 6>(&sel);
    err = cudaFuncSetAttribute(sel.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel.smem);
    int o = 0;
    if (err == cudaSuccess)
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, sel.kern, sel.threads, sel.smem);
    sel.occ = o < 1 ? 1 : o;
  }
  *out = sel;
  return err;
}

// The fused pass pays off when x, b and T (5 N doubles) do not stay in L2 between two
// separate passes: N * 40 B beyond twice the L2 (B200: 126 MB -> N > ~6.3M cells).
bool jacres_fused_wanted(msb_ctx ctx, msb_op op) {
  static int l2 = -1;
  if (l2 < 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess) v = 0;
    cudaGetLastError();
    l2 = v;
  }
  static const bool ab_off = getenv("MSB_AB_NOFUSE") != nullptr;  // TEMPORARY A/B
  return !ab_off && l2 > 0 && (double)op->N * 40.0 > 2.0 * (double)l2;
}

bool jacres_tma_plan(msb_ctx ctx, msb_op op, const double* x0buf, const double* x1buf,
                     const double* b, JQPlan* out) {
  out->ok = false;
  if (op->nx % 2 || !jacres_fused_wanted(ctx, op)) return false;
  JQSel sel;
  if (jq_kernel(&sel) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int TY = sel.ty, occ = sel.occ;
  const uint64_t d1[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 1};
  const uint64_t d3[4] = {(uint64_t)op->nx, (uint64_t)op->ny, (uint64_t)op->nz, 3};
  const uint64_t st3[3] = {(uint64_t)op->nx, (uint64_t)op->nx * op->ny, (uint64_t)op->N};
  const uint32_t bX[4] = {JQ_BX, (uint32_t)TY + 4, 1, 1}, bB[4] = {JQ_BX, (uint32_t)TY + 2, 1, 1},
                 bT[4] = {JQ_BX, (uint32_t)TY + 3, 1, 3};
  if (!tma_encode_4d(&out->mX[0], x0buf, d1, st3, bX) || !tma_encode_4d(&out->mX[1], x1buf, d1, st3, bX) ||
      !tma_encode_4d(&out->mB, b, d1, st3, bB) || !tma_encode_4d(&out->mT, op->Tx, d3, st3, bT))
    return false;
  const int ntx = (op->nx + JQ_TX - 1) / JQ_TX, nty = (op->ny + TY - 1) / TY;
  const int64_t slots = (int64_t)occ * ctx->sm_count, tiles = (int64_t)ntx * nty;
  int64_t best = INT64_MAX;
  int kz = op->nz, items = (int)tiles;
  for (int nzc = 1; nzc <= op->nz; ++nzc) {  // minimise waves x planes per item (4 halo)
    const int k = (op->nz + nzc - 1) / nzc;
    const int64_t it = tiles * ((op->nz + k - 1) / k);
    const int64_t cost = ((it + slots - 1) / slots) * (k + 4);
    if (cost < best) {
      best = cost;
      kz = k;
      items = (int)it;
    }
  }
  out->ntx = ntx;
  out->nty = nty;
  out->kz = kz;
  out->items = items;
  out->grid = (unsigned)std::min<int64_t>(items, slots);
  out->b = b;
  out->x[0] = x0buf;
  out->x[1] = x1buf;
  out->ok = true;
  return true;
}

msb_status jacres_tma_launch(msb_ctx ctx, msb_op op, const JQPlan& P, int cur, double* xo,
                             double* r, double omega, int first, double* partials,
                             const int* done) {
  JQSel sel;
  MSB_CUDA_TRY(ctx, jq_kernel(&sel));
  JQTiles tl{P.ntx, P.nty, P.kz, P.items};
  sel.kern<<<P.grid, sel.threads, sel.smem, ctx->stream>>>(P.mX[cur], P.mB, P.mT, xo, r,
                                                 make_grid3(op->nx, op->ny, op->nz), tl, omega,
                                                 first, partials, done);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

}  // namespace msb
