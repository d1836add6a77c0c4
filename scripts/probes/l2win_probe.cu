// Does an access-policy window keep a 64 MB array L2-resident across a 256 MB stream?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2win_probe l2win_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += a[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void rd_plain(const double* a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += a[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  const size_t na = 80ull << 20 >> 3, nb = 256ull << 20 >> 3;
  double *A, *B, *o;
  cudaMalloc(&A, na * 8); cudaMalloc(&B, nb * 8); cudaMalloc(&o, 8);
  cudaMemset(A, 0, na * 8); cudaMemset(B, 0, nb * 8);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int maxp = 0; cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  const size_t sizes[4] = {64ull << 20, 71808000ull, 48ull << 20, 80ull << 20};
  for (int si = 0; si < 4; ++si) {
  const size_t nw = sizes[si] / 8;
  printf("window %zu bytes\n", nw * 8);
  for (int mode = 0; mode < 3; ++mode) {
    // mode 0: none; 1: launch attribute (restrict kernel); 2: stream attribute; 3: launch attr, plain loads
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, mode ? nw * 8 : 0);
    cudaAccessPolicyWindow w{};
    w.base_ptr = A; w.num_bytes = nw * 8; w.hitRatio = 1.0f;
    w.hitProp = cudaAccessPropertyPersisting; w.missProp = cudaAccessPropertyStreaming;
    cudaStreamAttrValue sv{};
    if (mode == 2) sv.accessPolicyWindow = w;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &sv);
    auto launchA = [&]() {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148 * 8); cfg.blockDim = dim3(256); cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeAccessPolicyWindow; at[0].val.accessPolicyWindow = w;
      cfg.attrs = at; cfg.numAttrs = mode == 1 ? 1 : 0;
      cudaLaunchKernelEx(&cfg, rd, (const double*)A, nw, o);
    };
    float tA = 0;
    for (int it = 0; it < 5; ++it) {
      launchA();
      rd<<<148 * 8, 256, 0, st>>>(B, nb, o);
      cudaEventRecord(e0, st);
      launchA();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&tA, e0, e1);
    }
    printf("mode %d (max persist %d): read A after 256 MB stream: %.1f us = %.0f GB/s  (%s)\n", mode, maxp,
           tA * 1e3, nw * 8 / (tA * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaCtxResetPersistingL2Cache();
  }
  }
  return 0;
}
