// TMA streaming-throughput probe: each CTA streams boxes of a 4D fp64 tensor through a
// ring of S smem stages (one elected thread issues, all threads wait), like the sweep.
// usage: tma_bw  -> prints GB/s for several box shapes / CTAs per SM / ring depths
#include <cstdio>
#include <vector>
#include "../../paper_2001_01624_b200/csrc/tma.cuh"
using namespace msb;

__global__ void k_stream(const __grid_constant__ CUtensorMap m, int nx, int ny, int nz, int bx, int by,
                         int planes, int S, int stage_dbl, uint32_t tx_bytes, double* sink) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S * stage_dbl);
  if (threadIdx.x == 0) {
    for (int t = 0; t < S; ++t) mbar_init(&bars[t], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int ntx = nx / bx, nty = ny / by;
  double acc = 0.0;
  uint32_t seq = 0;
  for (int item = blockIdx.x; item < ntx * nty; item += gridDim.x) {
    const int x0 = (item % ntx) * bx, y0 = (item / ntx) * by;
    auto issue = [&](int p) {
      const uint32_t sq = seq + p;
      const int slot = sq % S;
      mbar_expect_tx(&bars[slot], tx_bytes);
      tma_load_4d(sm + slot * stage_dbl, &m, &bars[slot], x0, y0, p, 0);
    };
    if (threadIdx.x == 0)
      for (int p = 0; p < min(S - 1, planes); ++p) issue(p);
    for (int p = 0; p < planes; ++p) {
      if (threadIdx.x == 0 && p + S - 1 < planes) issue(p + S - 1);
      const uint32_t sq = seq + p;
      mbar_wait(&bars[sq % S], (sq / S) & 1u);
      acc += sm[(sq % S) * stage_dbl + threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) fence_proxy_async_smem();
    }
    seq += planes;
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const int nx = 256, ny = 256, nz = 64;  // 8 slot planes x 4M cells = 256 MB
  const size_t N = (size_t)nx * ny * nz;
  double *d, *sink;
  cudaMalloc(&d, 8 * N * 8);
  cudaMemset(d, 0, 8 * N * 8);
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int bx, by, planes8, S, ctas; };
  Cfg cfgs[] = {{36, 6, 1, 4, 3}, {32, 4, 1, 4, 3}, {64, 8, 1, 4, 2}, {32, 4, 1, 8, 3},
                {36, 6, 1, 4, 6}, {128, 8, 1, 3, 2}, {32, 4, 0, 8, 8}, {256, 4, 0, 6, 4}};
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (auto c : cfgs) {
    const int planes_dim = c.planes8 ? 8 : 1;
    CUtensorMap m;
    uint64_t dims[4] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz, (uint64_t)planes_dim};
    uint64_t st[3] = {(uint64_t)nx, (uint64_t)nx * ny, N};
    uint32_t box[4] = {(uint32_t)c.bx, (uint32_t)c.by, 1, (uint32_t)planes_dim};
    if (!tma_encode_4d(&m, d, dims, st, box)) { printf("encode failed %d %d\n", c.bx, c.by); continue; }
    const int stage_dbl = ((c.bx * c.by * planes_dim * 8 + 127) / 128) * 128 / 8;
    const size_t smem = (size_t)c.S * stage_dbl * 8 + 64;
    const int bxe = c.bx > 32 && c.bx < 64 ? 32 : c.bx, bye = c.by > 4 && c.by < 8 ? 4 : c.by;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_stream<<<sms * c.ctas, 128, smem>>>(m, nx, ny, nz, bxe, bye, nz, c.S, stage_dbl,
                                            (uint32_t)(c.bx * c.by * planes_dim * 8), sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)(nx / bxe) * (ny / bye) * nz * c.bx * c.by * planes_dim * 8;
    printf("box %3dx%d x%d planes  S=%d  ctas/SM=%d  smem=%zu  -> %.1f us  %.0f GB/s (%s)\n", c.bx, c.by,
           planes_dim, c.S, c.ctas, smem, ms * 1e3, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
