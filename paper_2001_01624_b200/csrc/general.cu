// §8 NEXT-3 — static partitions and general MsRSB levels.
//
//   msb_partition_wells       well blocks + background (B9)
//   msb_level_create_general  supports = blocks dilated by `halo` layers of the graph of
//                             A_T (requirement 2 of PAPER.md:220; B8),
//                             explicit ELL pattern, P^0 = constant basis
// (msb_partition_indicator shares the dynamic stage's component/merge kernels, cycle.cu.)
//
// The dilation runs one kernel per layer on sorted per-cell column lists of at most
// GW = 16 entries (the ELL width the sweep supports): each cell merges its own list with
// those of its face neighbours across faces with base transmissibility > 0.  Lists stay
// sorted and unique, so the ELL slots come out with ascending columns (the CSR order of
// msb_level_export) and the result is independent of thread scheduling.
#include <climits>
#include <vector>

#include "internal.cuh"

namespace msb {

constexpr int GW = 16;

__global__ void k_wells_part(int nx, int ny, int nz, const int32_t* __restrict__ perf,
                             const int32_t* __restrict__ wid, int np, int nw, int radius,
                             int32_t* __restrict__ part, int* __restrict__ has_bg) {
  const int64_t N = (int64_t)nx * ny * nz;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((int64_t)nx * ny));
  int best = INT_MAX, owner = -1;
  for (int p = 0; p < np; ++p) {
    const int q = perf[p];
    const int qi = q % nx, qj = (q / nx) % ny, qk = q / (nx * ny);
    const int d = max(max(abs(i - qi), abs(j - qj)), abs(k - qk));
    const int w = wid[p];
    if (d < best || (d == best && w < owner)) {
      best = d;
      owner = w;
    }
  }
  if (best <= radius) {
    part[c] = owner;
  } else {
    part[c] = nw;
    *has_bg = 1;
  }
}

// one dilation layer: out(c) = in(c) ∪ in(neighbours across faces with Tb > 0)
__global__ void k_dilate(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                         const double* __restrict__ Tb, int nx, int ny, int nz,
                         int* __restrict__ overflow) {
  const int64_t N = (int64_t)nx * ny * nz, sxy = (int64_t)nx * ny;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / sxy);
  int32_t buf[GW];
  int n = 0;
  bool over = false;
  auto add = [&](int64_t cc) {
    for (int s = 0; s < GW; ++s) {
      const int32_t v = in[(int64_t)s * N + cc];
      if (v < 0) break;
      int pos = 0;
      while (pos < n && buf[pos] < v) ++pos;
      if (pos < n && buf[pos] == v) continue;
      if (n == GW) {
        over = true;
        continue;
      }
      for (int t = n; t > pos; --t) buf[t] = buf[t - 1];
      buf[pos] = v;
      ++n;
    }
  };
  add(c);
  if (i > 0 && Tb[c - 1] > 0.0) add(c - 1);
  if (i < nx - 1 && Tb[c] > 0.0) add(c + 1);
  if (j > 0 && Tb[N + c - nx] > 0.0) add(c - nx);
  if (j < ny - 1 && Tb[N + c] > 0.0) add(c + nx);
  if (k > 0 && Tb[2 * N + c - sxy] > 0.0) add(c - sxy);
  if (k < nz - 1 && Tb[2 * N + c] > 0.0) add(c + sxy);
  for (int s = 0; s < GW; ++s) out[(int64_t)s * N + c] = s < n ? buf[s] : -1;
  if (over) atomicExch(overflow, 1);
}

__global__ void k_list_init(const int32_t* __restrict__ part, int64_t N, int M,
                            int32_t* __restrict__ lst, int* __restrict__ bad) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int32_t j = part[c];
  if (j < 0 || j >= M) atomicExch(bad, 1);
  lst[c] = j;
  for (int s = 1; s < GW; ++s) lst[(int64_t)s * N + c] = -1;
}

__global__ void k_list_count(const int32_t* __restrict__ lst, int64_t N, int* __restrict__ wmax,
                             unsigned long long* __restrict__ nnz) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int n = 0;
  if (c < N)
    while (n < GW && lst[(int64_t)n * N + c] >= 0) ++n;
  int m = n;
  unsigned long long t = (unsigned long long)n;
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(wmax, m);
    atomicAdd(nnz, t);
  }
}

// ELL planes from the first W list planes; P^0 = [col == part] in both buffers
__global__ void k_general_init(const int32_t* __restrict__ lst, const int32_t* __restrict__ part,
                               int64_t N, int W, int32_t* __restrict__ col, double* __restrict__ P0,
                               double* __restrict__ P1) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int32_t own = part[c];
  for (int s = 0; s < W; ++s) {
    const int32_t v = lst[(int64_t)s * N + c];
    col[(int64_t)s * N + c] = v;
    const double p = v == own ? 1.0 : 0.0;
    P0[(int64_t)s * N + c] = p;
    P1[(int64_t)s * N + c] = p;
  }
}

}  // namespace msb

using namespace msb;

extern "C" {

msb_status msb_partition_wells(msb_ctx ctx, const msb_grid* g, const int32_t* perf_ptr,
                               const int32_t* perf_cells, int32_t n_wells, int32_t radius,
                               int32_t* part, int32_t* M_out) {
  if (!ctx || !g || !perf_ptr || !perf_cells || n_wells < 1 || !M_out)
    return set_error(ctx, MSB_EINVAL, "msb_partition_wells: args");
  if (radius < 0) return set_error(ctx, MSB_EINVAL, "msb_partition_wells: radius < 0");
  const int64_t N = (int64_t)g->nx * g->ny * g->nz;
  if (g->nx < 1 || g->ny < 1 || g->nz < 1) return set_error(ctx, MSB_EDIM, "bad grid");
  std::vector<int32_t> cells, wid;
  for (int w = 0; w < n_wells; ++w) {
    if (perf_ptr[w + 1] <= perf_ptr[w])
      return set_error(ctx, MSB_EINVAL, "msb_partition_wells: well %d has no perforation", w);
    for (int p = perf_ptr[w]; p < perf_ptr[w + 1]; ++p) {
      if (perf_cells[p] < 0 || perf_cells[p] >= N)
        return set_error(ctx, MSB_EINVAL, "msb_partition_wells: cell %d outside the grid",
                         perf_cells[p]);
      cells.push_back(perf_cells[p]);
      wid.push_back(w);
    }
  }
  const int np = (int)cells.size();
  int32_t *dc, *dw, *dpart;
  int* bg;
  MSB_ALLOC(ctx, dc, int32_t, np);
  MSB_ALLOC(ctx, dw, int32_t, np);
  MSB_ALLOC(ctx, dpart, int32_t, N);
  MSB_ALLOC(ctx, bg, int, 1);
  cudaStream_t st = ctx->stream;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(dc, cells.data(), np * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(dw, wid.data(), np * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(bg, 0, sizeof(int), st));
  k_wells_part<<<grid_for(N, 256), 256, 0, st>>>(g->nx, g->ny, g->nz, dc, dw, np, n_wells, radius,
                                                 dpart, bg);
  MSB_LAUNCH_CHECK(ctx);
  int hbg = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hbg, bg, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (part) MSB_CUDA_TRY(ctx, copy_out(ctx, part, dpart, N * sizeof(int32_t)));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  dfree(ctx, dc);
  dfree(ctx, dw);
  dfree(ctx, dpart);
  dfree(ctx, bg);
  *M_out = n_wells + (hbg ? 1 : 0);
  return MSB_OK;
}

msb_status msb_level_create_general(msb_ctx ctx, msb_op op, const int32_t* part, int32_t M,
                                    int32_t halo, msb_level* out, int64_t* nnz_out) {
  if (!ctx || !op || !part || !out || M < 1 || halo < 0)
    return set_error(ctx, MSB_EINVAL, "msb_level_create_general: args");
  const int64_t N = op->N;
  cudaStream_t st = ctx->stream;
  void* o = nullptr;
  const int32_t* dpart = (const int32_t*)stage_in(ctx, part, N * sizeof(int32_t), &o);
  if (!dpart) return set_error(ctx, MSB_ENOMEM, "partition staging");
  int32_t *la, *lb;
  int* flags;  // [0] bad partition, [1] overflow, [2] W
  unsigned long long* nnz_d;
  MSB_ALLOC(ctx, la, int32_t, (size_t)GW * N);
  MSB_ALLOC(ctx, lb, int32_t, (size_t)GW * N);
  MSB_ALLOC(ctx, flags, int, 4);
  MSB_ALLOC(ctx, nnz_d, unsigned long long, 1);
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(flags, 0, 4 * sizeof(int), st));
  MSB_CUDA_TRY(ctx, cudaMemsetAsync(nnz_d, 0, sizeof(unsigned long long), st));
  const unsigned gr = grid_for(N, 256);
  k_list_init<<<gr, 256, 0, st>>>(dpart, N, M, la, flags);
  MSB_LAUNCH_CHECK(ctx);
  for (int l = 0; l < halo; ++l) {
    k_dilate<<<gr, 256, 0, st>>>(la, lb, op->Tb, op->nx, op->ny, op->nz, flags + 1);
    MSB_LAUNCH_CHECK(ctx);
    std::swap(la, lb);
  }
  k_list_count<<<gr, 256, 0, st>>>(la, N, flags + 2, nnz_d);
  MSB_LAUNCH_CHECK(ctx);
  int hf[4];
  unsigned long long hnnz = 0;
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&hnnz, nnz_d, sizeof(hnnz), cudaMemcpyDeviceToHost, st));
  MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
  msb_status rc = MSB_OK;
  if (hf[0]) rc = set_error(ctx, MSB_EINVAL, "partition value out of [0, M)");
  else if (hf[1]) rc = set_error(ctx, MSB_EINVAL, "general level: more than %d supports per cell", GW);
  msb_level L = nullptr;
  if (!rc) {
    const int W = hf[2];
    L = new msb_level_s();
    L->ctx = ctx;
    L->kind = 1;
    L->N = N;
    L->M = M;
    L->W = W;
    L->nnz = (int64_t)hnnz;
    L->nx = op->nx;
    L->ny = op->ny;
    L->nz = op->nz;
    L->P[0] = dalloc_n<double>(ctx, (size_t)W * N);
    L->P[1] = dalloc_n<double>(ctx, (size_t)W * N);
    L->col = dalloc_n<int32_t>(ctx, (size_t)W * N);
    L->part = dalloc_n<int32_t>(ctx, N);
    L->nbs = dalloc_n<int8_t>(ctx, (size_t)6 * W * N);
    if (!L->P[0] || !L->P[1] || !L->col || !L->part || !L->nbs) {
      rc = set_error(ctx, MSB_ENOMEM, "general level allocation");
    } else {
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(L->part, dpart, N * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, st));
      k_general_init<<<gr, 256, 0, st>>>(la, dpart, N, W, L->col, L->P[0], L->P[1]);
      MSB_LAUNCH_CHECK(ctx);
      k_nbs_ell<<<gr, 256, 0, st>>>(L->col, W, op->nx, op->ny, op->nz, L->nbs);
      MSB_LAUNCH_CHECK(ctx);
      MSB_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    }
  }
  dfree(ctx, la);
  dfree(ctx, lb);
  dfree(ctx, flags);
  dfree(ctx, nnz_d);
  if (o) dfree(ctx, o);
  if (rc) {
    level_free(L);
    return rc;
  }
  *out = L;
  if (nnz_out) *nnz_out = L->nnz;
  return MSB_OK;
}

}  // extern "C"
