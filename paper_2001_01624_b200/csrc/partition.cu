// Row a2 (fault-split partition + flood-fill supports) and the partition half of
// row a10 (Δp-binned dynamic partition).
//
// Connected components use lock-free union-find (hook the larger root under the
// smaller with atomicCAS, path-halving finds, then full compression).  Roots only
// ever move to smaller indices, so the final root of a component is its minimum
// node index — exactly the canonical "ascending minimum cell index" numbering of
// the oracle after an exclusive scan over root flags.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.cuh"

namespace msb {

__device__ __forceinline__ int32_t uf_find(int32_t* __restrict__ par, int32_t x) {
  int32_t p = par[x];
  while (p != x) {
    int32_t g = par[p];
    if (g != p) par[x] = g;  // path halving (benign race: values only decrease)
    x = p;
    p = g;
  }
  return x;
}

__device__ __forceinline__ void uf_union(int32_t* __restrict__ par, int32_t a, int32_t b) {
  while (true) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    if (a == b) return;
    int32_t hi = a > b ? a : b, lo = a > b ? b : a;
    int32_t old = atomicCAS(par + hi, hi, lo);
    if (old == hi) return;
    a = old;  // hi got hooked meanwhile; retry from its new parent
    b = lo;
  }
}

__global__ void k_iota(int32_t* __restrict__ p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

// Compression after all unions: read-only walk to the root (no path-halving writes,
// which could overwrite another thread's already-compressed entry with a non-root
// ancestor), then each thread writes only its own entry.
__global__ void k_compress(int32_t* __restrict__ par, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t x = (int32_t)i;
  int32_t p = *(volatile int32_t*)(par + x);
  while (p != x) {
    x = p;
    p = *(volatile int32_t*)(par + x);
  }
  par[i] = x;
}

// Two-phase labelling (same roots as unioning every face globally: roots are component
// minima either way).  Phase 1: each CTA labels a 16x4x4 tile in shared memory (local
// union-find over the tile's interior faces; local and global index orders agree inside a
// tile, so local minima are global minima) and writes each cell's parent as its tile
// root.  Phase 2 (k_cc_cross) unions only the faces that cross tile boundaries — about a
// fifth of them — through the global forest.
constexpr int CCT_X = 16, CCT_Y = 4, CCT_Z = 4;

__device__ __forceinline__ int lf_find(int* __restrict__ lp, int x) {
  int p = lp[x];
  while (p != x) {
    const int g = lp[p];
    if (g != p) lp[x] = g;
    x = p;
    p = g;
  }
  return x;
}

__device__ __forceinline__ void lf_union(int* __restrict__ lp, int a, int b) {
  while (true) {
    a = lf_find(lp, a);
    b = lf_find(lp, b);
    if (a == b) return;
    const int hi = a > b ? a : b, lo = a > b ? b : a;
    const int old = atomicCAS(lp + hi, hi, lo);
    if (old == hi) return;
    a = old;
    b = lo;
  }
}

__global__ void __launch_bounds__(256) k_cc_tile(const int32_t* __restrict__ klass,
                                                 const uint8_t* __restrict__ open, int nx, int ny,
                                                 int nz, int tiles_x, int tiles_y,
                                                 int32_t* __restrict__ par) {
  __shared__ int lp[256];
  __shared__ int kl[256];
  __shared__ uint8_t om[256];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = (t >> 4) & 3, tz = t >> 6;
  const int b = blockIdx.x;
  const int bx = b % tiles_x, by = (b / tiles_x) % tiles_y, bz = b / (tiles_x * tiles_y);
  const int i = bx * CCT_X + tx, j = by * CCT_Y + ty, k = bz * CCT_Z + tz;
  const bool in = i < nx && j < ny && k < nz;
  const int64_t c = in ? ((int64_t)k * ny + j) * nx + i : 0;
  lp[t] = t;
  kl[t] = in ? klass[c] : INT32_MIN;
  om[t] = in ? (open ? open[c] : 7) : 0;
  __syncthreads();
  if (in) {
    const int kc = kl[t];
    const uint8_t o = om[t];
    if (tx < CCT_X - 1 && i < nx - 1 && (o & 1) && kl[t + 1] == kc) lf_union(lp, t, t + 1);
    if (ty < CCT_Y - 1 && j < ny - 1 && (o & 2) && kl[t + 16] == kc) lf_union(lp, t, t + 16);
    if (tz < CCT_Z - 1 && k < nz - 1 && (o & 4) && kl[t + 64] == kc) lf_union(lp, t, t + 64);
  }
  __syncthreads();
  if (!in) return;
  int r = t, p = lp[r];  // read-only walk to the tile root
  while (p != r) {
    r = p;
    p = lp[r];
  }
  const int rx = bx * CCT_X + (r & 15), ry = by * CCT_Y + ((r >> 4) & 3), rz = bz * CCT_Z + (r >> 6);
  par[c] = (int32_t)(((int64_t)rz * ny + ry) * nx + rx);
}

__global__ void k_cc_cross(const int32_t* __restrict__ klass, const uint8_t* __restrict__ open,
                           int nx, int ny, int nz, int32_t* __restrict__ par) {
  const int64_t N = (int64_t)nx * ny * nz, sxy = (int64_t)nx * ny;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  const bool ex = i < nx - 1 && (i + 1) % CCT_X == 0;
  const bool ey = j < ny - 1 && (j + 1) % CCT_Y == 0;
  const bool ez = k < nz - 1 && (k + 1) % CCT_Z == 0;
  if (!(ex || ey || ez)) return;
  const uint8_t o = open ? open[c] : 7;
  const int32_t kc = klass[c];
  if (ex && (o & 1) && klass[c + 1] == kc) uf_union(par, (int32_t)c, (int32_t)(c + 1));
  if (ey && (o & 2) && klass[c + nx] == kc) uf_union(par, (int32_t)c, (int32_t)(c + nx));
  if (ez && (o & 4) && klass[c + sxy] == kc) uf_union(par, (int32_t)c, (int32_t)(c + sxy));
}

__global__ void k_root_flags(const int32_t* __restrict__ lab, int64_t n, int32_t* __restrict__ f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = lab[i] == (int32_t)i;
}

__global__ void k_gather_ids(const int32_t* __restrict__ lab, const int32_t* __restrict__ ids,
                             int64_t n, int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = ids[lab[i]];
}

// lab[i] must be a cell index that is its own label for the representative cell.
msb_status canonical_number_async(msb_ctx ctx, int64_t N, const int32_t* lab, int32_t* out,
                                  int32_t* scratch, const int32_t** M_dev) {
  int32_t* flags = scratch;
  int32_t* ids = scratch + N;
  k_root_flags<<<grid_for(N, 256), 256, 0, ctx->stream>>>(lab, N, flags);
  MSB_LAUNCH_CHECK(ctx);
  msb_status st = scan_exclusive_async(ctx, flags, ids, N, M_dev);
  if (st != MSB_OK) return st;
  k_gather_ids<<<grid_for(N, 256), 256, 0, ctx->stream>>>(lab, ids, N, out);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

msb_status canonical_number(msb_ctx ctx, int64_t N, const int32_t* lab, int32_t* out,
                            int32_t* scratch, int32_t* M_out, const void* extra_dev,
                            void* extra_host, size_t extra_bytes) {
  int32_t* flags = scratch;
  int32_t* ids = scratch + N;
  k_root_flags<<<grid_for(N, 256), 256, 0, ctx->stream>>>(lab, N, flags);
  MSB_LAUNCH_CHECK(ctx);
  int32_t M = 0;
  msb_status st = scan_exclusive(ctx, flags, ids, N, &M, extra_dev, extra_host, extra_bytes);
  if (st != MSB_OK) return st;
  k_gather_ids<<<grid_for(N, 256), 256, 0, ctx->stream>>>(lab, ids, N, out);
  MSB_LAUNCH_CHECK(ctx);
  *M_out = M;
  return MSB_OK;
}

// bit a of m[c]: the face (c, c + e_a) has base transmissibility T > 0
__global__ void k_tpos_mask(const double* __restrict__ Tb, Grid3 g, uint8_t* __restrict__ m) {
  const int N = g.nxy * g.nz;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i, j, k;
  g3_coords(g, c, i, j, k);
  m[c] = (uint8_t)((i < g.nx - 1 && Tb[c] > 0.0 ? 1 : 0) | (j < g.ny - 1 && Tb[N + c] > 0.0 ? 2 : 0) |
                   (k < g.nz - 1 && Tb[2 * N + c] > 0.0 ? 4 : 0));
}

__global__ void k_count_ne0(const int32_t* __restrict__ lab, int64_t N, int* __restrict__ flag) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < N && lab[c] != 0) atomicOr(flag, 1);
}

msb_status op_connected(msb_ctx ctx, msb_op op, bool* connected) {
  if (op->connected >= 0) {
    *connected = op->connected == 1;
    return MSB_OK;
  }
  const int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  int32_t* klass = dalloc_n<int32_t>(ctx, 2 * N);
  uint8_t* m = dalloc_n<uint8_t>(ctx, N);
  int* flag = dalloc_n<int>(ctx, 1);
  msb_status rc = MSB_OK;
  int h = 0;
  if (!klass || !m || !flag) rc = set_error(ctx, MSB_ENOMEM, "connectivity scratch");
  if (!rc && (cudaMemsetAsync(klass, 0, N * sizeof(int32_t), st) != cudaSuccess ||
              cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess))
    rc = set_error(ctx, MSB_ECUDA, "connectivity memset");
  if (!rc) {
    k_tpos_mask<<<grid_for(N, 256), 256, 0, st>>>(op->Tb, make_grid3(op->nx, op->ny, op->nz), m);
    count_launch();
    rc = cc_label(ctx, op, klass, klass + N, m);
  }
  if (!rc) {
    k_count_ne0<<<grid_for(N, 256), 256, 0, st>>>(klass + N, N, flag);
    count_launch();
    if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      rc = set_error(ctx, MSB_ECUDA, "connectivity readback");
  }
  cudaStreamSynchronize(st);
  dfree(ctx, klass);
  dfree(ctx, m);
  dfree(ctx, flag);
  if (rc) return rc;
  op->connected = h ? 0 : 1;
  *connected = op->connected == 1;
  return MSB_OK;
}

msb_status cc_label(msb_ctx ctx, msb_op op, const int32_t* klass, int32_t* lab,
                    const uint8_t* open) {
  int64_t N = op->N;
  {
    const int tx = (op->nx + CCT_X - 1) / CCT_X, ty = (op->ny + CCT_Y - 1) / CCT_Y,
              tz = (op->nz + CCT_Z - 1) / CCT_Z;
    k_cc_tile<<<(unsigned)((int64_t)tx * ty * tz), 256, 0, ctx->stream>>>(
        klass, open, op->nx, op->ny, op->nz, tx, ty, lab);
    MSB_LAUNCH_CHECK(ctx);
    k_cc_cross<<<grid_for(N, 256), 256, 0, ctx->stream>>>(klass, open, op->nx, op->ny, op->nz,
                                                          lab);
    MSB_LAUNCH_CHECK(ctx);
  }
  k_compress<<<grid_for(N, 256), 256, 0, ctx->stream>>>(lab, N);
  MSB_LAUNCH_CHECK(ctx);
  return MSB_OK;
}

// ---------------------------------------------------------------- flood-fill supports
// Nodes (s, c) of the parent Cartesian level's active slots; node id = s*N + c.
// Joined across open faces when the neighbour holds the same column in slot s.
__global__ void k_cc_slots(const int32_t* __restrict__ tab, const uint8_t* __restrict__ open,
                           int nx, int ny, int nz, int32_t* __restrict__ par) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t sxy = (int64_t)nx * ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  uint8_t o = open[c];
  const int32_t* tx = tab + 2 * i;
  const int32_t* ty = tab + 2 * (nx + j);
  const int32_t* tz = tab + 2 * (nx + ny + k);
  for (int s = 0; s < 8; ++s) {
    int px = s & 1, py = (s >> 1) & 1, pz = s >> 2;
    int jx = tx[px], jy = ty[py], jz = tz[pz];
    if (jx < 0 || jy < 0 || jz < 0) continue;
    int32_t a = (int32_t)(s * N + c);
    if (i < nx - 1 && (o & 1) && tab[2 * (i + 1) + px] == jx) uf_union(par, a, a + 1);
    if (j < ny - 1 && (o & 2) && tab[2 * (nx + j + 1) + py] == jy) uf_union(par, a, (int32_t)(a + nx));
    if (k < nz - 1 && (o & 4) && tab[2 * (nx + ny + k + 1) + pz] == jz)
      uf_union(par, a, (int32_t)(a + sxy));
  }
}

constexpr int KCH = 6;  // max distinct split blocks attached to one box component

// Attach each cell's split block to the component of its own-parent slot node.
__global__ void k_attach(const int32_t* __restrict__ par, const int32_t* __restrict__ ppart,
                         const int32_t* __restrict__ spart, int nbx, int nby, int64_t N,
                         int32_t* __restrict__ lists, int* __restrict__ overflow) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int J = ppart[c];
  int s = (J % nbx & 1) | (((J / nbx) % nby & 1) << 1) | ((J / (nbx * nby) & 1) << 2);
  int32_t root = par[(int64_t)s * N + c];
  int32_t child = spart[c];
  int32_t* L = lists + (int64_t)root * KCH;
  for (int t = 0; t < KCH; ++t) {
    int32_t old = atomicCAS(L + t, -1, child);
    if (old == -1 || old == child) return;
  }
  atomicExch(overflow, 1);
}

__device__ __forceinline__ int gather_cols(const int32_t* __restrict__ tab,
                                           const int32_t* __restrict__ par,
                                           const int32_t* __restrict__ lists, int nx, int ny,
                                           int64_t N, int64_t c, int* cols, int cap) {
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((int64_t)nx * ny));
  const int32_t* tx = tab + 2 * i;
  const int32_t* ty = tab + 2 * (nx + j);
  const int32_t* tz = tab + 2 * (nx + ny + k);
  int n = 0;
  for (int s = 0; s < 8; ++s) {
    if (tx[s & 1] < 0 || ty[(s >> 1) & 1] < 0 || tz[s >> 2] < 0) continue;
    int32_t root = par[(int64_t)s * N + c];
    const int32_t* L = lists + (int64_t)root * KCH;
    for (int t = 0; t < KCH; ++t) {
      int32_t v = L[t];
      if (v < 0) break;
      bool dup = false;
      for (int u = 0; u < n; ++u) dup |= cols[u] == v;
      if (dup) continue;
      if (n < cap) {
        int p = n;
        while (p > 0 && cols[p - 1] > v) {
          cols[p] = cols[p - 1];
          --p;
        }
        cols[p] = v;
      }
      ++n;
    }
  }
  return n;
}

__global__ void k_flood_count(const int32_t* __restrict__ tab, const int32_t* __restrict__ par,
                              const int32_t* __restrict__ lists, int nx, int ny, int64_t N,
                              int* __restrict__ wmax, unsigned long long* __restrict__ nnz) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int cols[64];
  int n = gather_cols(tab, par, lists, nx, ny, N, c, cols, 64);
  atomicMax(wmax, n);
  atomicAdd(nnz, (unsigned long long)n);
}

__global__ void k_flood_fill(const int32_t* __restrict__ tab, const int32_t* __restrict__ par,
                             const int32_t* __restrict__ lists, const int32_t* __restrict__ spart,
                             int nx, int ny, int64_t N, int W, int32_t* __restrict__ col,
                             double* __restrict__ P0, double* __restrict__ P1) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int cols[64];
  int n = gather_cols(tab, par, lists, nx, ny, N, c, cols, 64);
  int own = spart[c];
  for (int s = 0; s < W; ++s) {
    int v = s < n ? cols[s] : -1;
    col[(int64_t)s * N + c] = v;
    double p = (v >= 0 && v == own) ? 1.0 : 0.0;
    P0[(int64_t)s * N + c] = p;
    P1[(int64_t)s * N + c] = 0.0;
  }
}

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_nbs_ell2(const int32_t* __restrict__ col, int W, int nx, int ny, int nz,
                           int8_t* __restrict__ nbs) {
  int64_t N = (int64_t)nx * ny * nz;
  int64_t sxy = (int64_t)nx * ny;
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  int64_t nb[6] = {c - sxy, c - nx, c - 1, c + 1, c + nx, c + sxy};
  bool ex[6] = {k > 0, j > 0, i > 0, i < nx - 1, j < ny - 1, k < nz - 1};
  for (int s = 0; s < W; ++s) {
    int jc = col[(int64_t)s * N + c];
    for (int d = 0; d < 6; ++d) {
      int r = -1;
      if (jc >= 0 && ex[d]) {
        for (int t = 0; t < W; ++t) {
          int v = col[(int64_t)t * N + nb[d]];
          if (v == jc) {
            r = t;
            break;
          }
        }
      }
      nbs[((int64_t)d * W + s) * N + c] = (int8_t)r;
    }
  }
}

}  // namespace msb

using namespace msb;

extern "C" msb_status msb_level_create_split(msb_ctx ctx, msb_op op, msb_level parent,
                                             msb_level* out, int64_t* nnz_out) {
  MSB_NVTX("msb_level_create_split");
  if (!ctx || !op || !parent || !out) return set_error(ctx, MSB_EINVAL, "split level: null");
  if (parent->kind != 0) return set_error(ctx, MSB_EINVAL, "split level needs a Cartesian parent");
  int64_t N = op->N;
  if (8 * N >= (int64_t)INT32_MAX) return set_error(ctx, MSB_EINVAL, "grid too large for split level");
  // 1. split partition: components of each parent block over open faces
  int32_t *lab, *spart, *scratch;
  MSB_ALLOC(ctx, lab, int32_t, N);
  MSB_ALLOC(ctx, spart, int32_t, N);
  MSB_ALLOC(ctx, scratch, int32_t, 2 * N);
  msb_status st = cc_label(ctx, op, parent->part, lab, op->open);
  if (st) return st;
  int32_t Ms = 0;
  st = canonical_number(ctx, N, lab, spart, scratch, &Ms);
  if (st) return st;
  // 2. components of each parent support box (slot nodes) over open faces
  int32_t* par;
  MSB_ALLOC(ctx, par, int32_t, 8 * N);
  k_iota<<<grid_for(8 * N, 256), 256, 0, ctx->stream>>>(par, 8 * N);
  MSB_LAUNCH_CHECK(ctx);
  k_cc_slots<<<grid_for(N, 256), 256, 0, ctx->stream>>>(parent->tab, op->open, op->nx, op->ny,
                                                        op->nz, par);
  MSB_LAUNCH_CHECK(ctx);
  k_compress<<<grid_for(8 * N, 256), 256, 0, ctx->stream>>>(par, 8 * N);
  MSB_LAUNCH_CHECK(ctx);
  // 3. attach split blocks to box components; gather columns per cell
  int32_t* lists;
  MSB_ALLOC(ctx, lists, int32_t, 8 * N * KCH);
  k_fill_i32<<<grid_for(8 * N * KCH, 256), 256, 0, ctx->stream>>>(lists, 8 * N * KCH, -1);
  MSB_LAUNCH_CHECK(ctx);
  int* flags = dalloc_n<int>(ctx, 2);
  unsigned long long* dnnz = dalloc_n<unsigned long long>(ctx, 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(dnnz, 0, 8, ctx->stream));
  k_attach<<<grid_for(N, 256), 256, 0, ctx->stream>>>(par, parent->part, spart, parent->nb[0],
                                                      parent->nb[1], N, lists, flags);
  MSB_LAUNCH_CHECK(ctx);
  k_flood_count<<<grid_for(N, 128), 128, 0, ctx->stream>>>(parent->tab, par, lists, op->nx, op->ny,
                                                           N, flags + 1, dnnz);
  MSB_LAUNCH_CHECK(ctx);
  int hf[2];
  unsigned long long hn = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hn, dnnz, 8, cudaMemcpyDeviceToHost, ctx->stream));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hf[0]) return set_error(ctx, MSB_EINVAL, "split level: more than %d blocks per box component", KCH);
  int W = hf[1];
  if (W > 64 || W > 127) return set_error(ctx, MSB_EINVAL, "split level: %d supports per cell", W);
  msb_level L = new msb_level_s();
  L->ctx = ctx;
  L->kind = 1;
  L->N = N;
  L->M = Ms;
  L->W = W;
  L->nnz = (int64_t)hn;
  L->nx = op->nx; L->ny = op->ny; L->nz = op->nz;
  L->part = spart;
  MSB_ALLOC(ctx, L->col, int32_t, (int64_t)W * N);
  MSB_ALLOC(ctx, L->P[0], double, (int64_t)W * N);
  MSB_ALLOC(ctx, L->P[1], double, (int64_t)W * N);
  MSB_ALLOC(ctx, L->nbs, int8_t, (int64_t)6 * W * N);
  k_flood_fill<<<grid_for(N, 128), 128, 0, ctx->stream>>>(parent->tab, par, lists, spart, op->nx,
                                                          op->ny, N, W, L->col, L->P[0], L->P[1]);
  MSB_LAUNCH_CHECK(ctx);
  k_nbs_ell2<<<grid_for(N, 128), 128, 0, ctx->stream>>>(L->col, W, op->nx, op->ny, op->nz, L->nbs);
  MSB_LAUNCH_CHECK(ctx);
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, lab);
  dfree(ctx, scratch);
  dfree(ctx, par);
  dfree(ctx, lists);
  dfree(ctx, flags);
  dfree(ctx, dnnz);
  if (nnz_out) *nnz_out = L->nnz;
  *out = L;
  return MSB_OK;
}
