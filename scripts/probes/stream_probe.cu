// Achievable HBM bandwidth for short multi-stream passes (the shape of the cycle's
// stencil kernels): k arrays of N doubles read, one written, N = 1.122M (config 2).
#include <cstdio>
#include <vector>
template <int K>
__global__ void k_stream(const double* __restrict__ a, double* __restrict__ o, int n, int cpt) {
  int i0 = (blockIdx.x * blockDim.x) * cpt + threadIdx.x;
  for (int u = 0; u < cpt; ++u) {
    int i = i0 + u * blockDim.x;
    if (i >= n) return;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += a[(size_t)k * n + i];
    o[i] = s;
  }
}
int main() {
  std::vector<int> ns = {1122000, 10000000};
  for (int n : ns) {
    double *a, *o;
    cudaMalloc(&a, 6 * (size_t)n * 8);
    cudaMalloc(&o, (size_t)n * 8);
    cudaMemset(a, 0, 6 * (size_t)n * 8);
    double* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int cpt : {1, 4}) {
      auto run = [&](auto kern, int K) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemset(flush, rep, 256 << 20);
          cudaEventRecord(e0);
          kern<<<(n + 256 * cpt - 1) / (256 * cpt), 256>>>(a, o, n, cpt);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
        double bytes = (double)(K + 1) * n * 8;
        printf("n=%d K=%d cpt=%d: %.2f us  %.0f GB/s\n", n, K, cpt, best * 1e3, bytes / best / 1e6);
      };
      run(k_stream<1>, 1);
      run(k_stream<5>, 5);
    }
  }
  return 0;
}
