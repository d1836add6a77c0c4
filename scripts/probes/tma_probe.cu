// Minimal TMA probe: load one fp64 box through the msb helpers and check it.
// usage: tma_probe <variant>   (each variant in its own process: a fault kills the context)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2001_01624_b200/csrc/tma.cuh"
using namespace msb;

__device__ CUtensorMap g_map;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__global__ void k_probe(const __grid_constant__ CUtensorMap m, int rank, int use_global, double* out,
                        int c0, int c1, int c2, int c3, int nbox) {
  extern __shared__ unsigned char raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ uint64_t bar;
  const CUtensorMap* mp = use_global ? &g_map : &m;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, nbox * 8);
    if (rank == 4)
      tma_load_4d(sm, mp, &bar, c0, c1, c2, c3);
    else
      tma_load_2d(sm, mp, &bar, c0, c1);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nbox; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  int v = argc > 1 ? atoi(argv[1]) : 0;
  int nx = 32, ny = 32, nz = 4, N = nx * ny * nz;
  std::vector<double> h(8 * (size_t)N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 64 * 1024);
  CUtensorMap m;
  memset(&m, 0, sizeof(m));
  int rank = 4, c[4] = {0, 0, 1, 0}, nbox = 0, use_global = 0;
  bool ok = false;
  if (v == 0 || v == 1 || v == 4) {  // 4D box {34,6,1,8}; v0 negative coords; v4 global map
    uint64_t dims[4] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz, 8};
    uint64_t st[3] = {(uint64_t)nx, (uint64_t)nx * ny, (uint64_t)N};
    uint32_t box[4] = {34, 6, 1, 8};
    ok = tma_encode_4d(&m, d, dims, st, box);
    nbox = 34 * 6 * 8;
    if (v == 0) { c[0] = -1; c[1] = -1; }
    use_global = v == 4;
  } else if (v == 5 || v == 6 || v == 7) {  // v5: (-2,-1) box 36; v6: (1,0) box 34; v7 (-2,-1,-1)
    uint64_t dims[4] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz, 8};
    uint64_t st[3] = {(uint64_t)nx, (uint64_t)nx * ny, (uint64_t)N};
    uint32_t box[4] = {(uint32_t)(v == 6 ? 34 : 36), 6, 1, 8};
    ok = tma_encode_4d(&m, d, dims, st, box);
    nbox = box[0] * 6 * 8;
    if (v == 5) { c[0] = -2; c[1] = -1; }
    if (v == 6) { c[0] = 1; c[1] = 0; }
    if (v == 7) { c[0] = -2; c[1] = -1; c[2] = -1; }
  } else if (v == 2) {  // 4D box {32,4,1,8}
    uint64_t dims[4] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz, 8};
    uint64_t st[3] = {(uint64_t)nx, (uint64_t)nx * ny, (uint64_t)N};
    uint32_t box[4] = {32, 4, 1, 8};
    ok = tma_encode_4d(&m, d, dims, st, box);
    nbox = 32 * 4 * 8;
  } else if (v == 3) {  // 2D via a 4D map with trailing 1-dims
    uint64_t dims[4] = {(uint64_t)nx, (uint64_t)ny * nz * 8, 1, 1};
    uint64_t st[3] = {(uint64_t)nx, (uint64_t)N * 8, (uint64_t)N * 8};
    uint32_t box[4] = {32, 4, 1, 1};
    ok = tma_encode_4d(&m, d, dims, st, box);
    nbox = 32 * 4;
    rank = 2;
  }
  unsigned char* b = reinterpret_cast<unsigned char*>(&m);
  printf("variant %d encode ok=%d map[0..32]:", v, ok);
  for (int i = 0; i < 32; ++i) printf("%02x", b[i]);
  printf("\n");
  if (use_global) cudaMemcpyToSymbol(g_map, &m, sizeof(m));
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_probe<<<1, 128, 32 * 1024>>>(m, rank, use_global, o, c[0], c[1], c[2], c[3], nbox);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d: %s\n", v, cudaGetErrorString(e));
  if (e == cudaSuccess) {
    std::vector<double> r(nbox);
    cudaMemcpy(r.data(), o, nbox * 8, cudaMemcpyDeviceToHost);
    printf("  first values: %g %g %g %g ... last %g\n", r[0], r[1], r[2], r[3], r[nbox - 1]);
  }
  return 0;
}
