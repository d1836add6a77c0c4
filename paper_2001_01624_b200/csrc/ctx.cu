// Context, allocation, host|dev staging, error reporting, device scan.
#include "internal.cuh"

namespace msb {

std::atomic<int64_t> g_launches{0};

msb_status set_error(msb_ctx ctx, msb_status code, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
  }
  return code;
}

void* dalloc(msb_ctx ctx, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->alloc) return ctx->alloc(bytes, ctx->user);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dfree(msb_ctx ctx, void* p) {
  if (!p) return;
  if (ctx->free_fn) {
    ctx->free_fn(p, ctx->user);
    return;
  }
  cudaFree(p);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

const void* stage_in(msb_ctx ctx, const void* p, size_t bytes, void** owned) {
  *owned = nullptr;
  if (!p) return nullptr;
  if (is_device_ptr(p)) return p;
  void* d = dalloc(ctx, bytes);
  if (!d) return nullptr;
  if (cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) {
    dfree(ctx, d);
    return nullptr;
  }
  *owned = d;
  return d;
}

void* pinned_scratch(msb_ctx ctx, size_t bytes) {
  if (ctx->pinned_bytes >= bytes) return ctx->pinned;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  ctx->pinned_bytes = 0;
  size_t cap = bytes < 65536 ? 65536 : bytes;
  if (cudaHostAlloc(&ctx->pinned, cap, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    ctx->pinned = nullptr;
    return nullptr;
  }
  ctx->pinned_bytes = cap;
  return ctx->pinned;
}

cudaError_t copy_out(msb_ctx ctx, void* dst, const void* src_dev, size_t bytes) {
  if (!dst || bytes == 0) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDefault, ctx->stream);
  if (e != cudaSuccess) return e;
  if (!is_device_ptr(dst)) return cudaStreamSynchronize(ctx->stream);
  return cudaSuccess;
}

cudaError_t copy_in(msb_ctx ctx, void* dst_dev, const void* src, size_t bytes) {
  if (!src || bytes == 0) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dst_dev, src, bytes, cudaMemcpyDefault, ctx->stream);
  if (e != cudaSuccess) return e;
  // pageable host memory may be reused by the caller right after return
  if (!is_device_ptr(src)) return cudaStreamSynchronize(ctx->stream);
  return cudaSuccess;
}

msb_status sync(msb_ctx ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_error(ctx, MSB_ECUDA, "stream sync: %s", cudaGetErrorString(e));
  return MSB_OK;
}

// ---------------------------------------------------------------- exclusive scan (int32)
static constexpr int SCAN_BLOCK = 1024;

__global__ void k_scan_block(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                             int32_t* __restrict__ sums, int64_t n) {
  __shared__ int32_t warp_tot[32];
  int64_t i = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  int32_t v = i < n ? in[i] : 0;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  int32_t base = w > 0 ? warp_tot[w - 1] : 0;
  if (i < n) out[i] = base + x - v;
  if (threadIdx.x == SCAN_BLOCK - 1) sums[blockIdx.x] = base + x;
}

__global__ void k_scan_add(int32_t* __restrict__ out, const int32_t* __restrict__ offs, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  if (i < n) out[i] += offs[blockIdx.x];
}

// One level: block scans of `in`, their sums scanned recursively into offs, added back.
static msb_status scan_level(msb_ctx ctx, const int32_t* in, int32_t* out, int64_t n, int32_t* scr) {
  const int64_t nb = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
  int32_t* sums = scr;
  int32_t* offs = scr + nb + 1;
  k_scan_block<<<(unsigned)nb, SCAN_BLOCK, 0, ctx->stream>>>(in, out, sums, n);
  MSB_LAUNCH_CHECK(ctx);
  if (nb > 1) {
    msb_status st = scan_level(ctx, sums, offs, nb, scr + 2 * (nb + 1));
    if (st != MSB_OK) return st;
    k_scan_add<<<(unsigned)nb, SCAN_BLOCK, 0, ctx->stream>>>(out, offs, n);
    MSB_LAUNCH_CHECK(ctx);
  }
  return MSB_OK;
}

__global__ void k_scan_total(const int32_t* __restrict__ in, const int32_t* __restrict__ out,
                             int64_t n, int32_t* __restrict__ total) {
  *total = out[n - 1] + in[n - 1];
}

// Exclusive prefix sum of n int32 (device); *total (host, optional) = sum of all, read
// back with one synchronisation.  Scratch is the context's, reused across calls.
msb_status scan_reserve(msb_ctx ctx, int64_t n) {
  int64_t need = 1;  // the total word, then sums|offs of every level scan_level visits
  for (int64_t m = n;;) {
    const int64_t nb = (m + SCAN_BLOCK - 1) / SCAN_BLOCK;
    need += 2 * (nb + 1);
    if (nb <= 1) break;
    m = nb;
  }
  if (ctx->scan_cap < need) {
    dfree(ctx, ctx->scan_scr);
    ctx->scan_scr = nullptr;
    ctx->scan_cap = 0;
    MSB_ALLOC(ctx, ctx->scan_scr, int32_t, need);
    ctx->scan_cap = need;
  }
  return MSB_OK;
}

// scan_exclusive without the readback: the total is left in device memory (*total_dev,
// valid until the next scan); no host synchronisation, so it can be graph-captured.  The
// scratch must have been sized by scan_reserve(n) first.
msb_status scan_exclusive_async(msb_ctx ctx, const int32_t* in, int32_t* out, int64_t n,
                                const int32_t** total_dev) {
  if (n <= 0 || ctx->scan_cap < 1) return set_error(ctx, MSB_EINVAL, "scan_exclusive_async: scratch");
  msb_status st = scan_level(ctx, in, out, n, ctx->scan_scr + 1);
  if (st != MSB_OK) return st;
  k_scan_total<<<1, 1, 0, ctx->stream>>>(in, out, n, ctx->scan_scr);
  MSB_LAUNCH_CHECK(ctx);
  *total_dev = ctx->scan_scr;
  return MSB_OK;
}

msb_status scan_exclusive(msb_ctx ctx, const int32_t* in, int32_t* out, int64_t n,
                          int32_t* total, const void* extra_dev, void* extra_host,
                          size_t extra_bytes) {
  if (n <= 0) {
    if (total) *total = 0;
    return MSB_OK;
  }
  msb_status rs = scan_reserve(ctx, n);
  if (rs != MSB_OK) return rs;
  int32_t* tot = ctx->scan_scr;
  msb_status st = scan_level(ctx, in, out, n, ctx->scan_scr + 1);
  if (st != MSB_OK) return st;
  if (total) {
    k_scan_total<<<1, 1, 0, ctx->stream>>>(in, out, n, tot);
    MSB_LAUNCH_CHECK(ctx);
    int32_t h = 0;
    MSB_CUDA_TRY(ctx, cudaMemcpyAsync(&h, tot, 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (extra_bytes)  // a caller's value read back under the same synchronisation
      MSB_CUDA_TRY(ctx, cudaMemcpyAsync(extra_host, extra_dev, extra_bytes, cudaMemcpyDeviceToHost,
                                        ctx->stream));
    MSB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    *total = h;
  }
  return MSB_OK;
}

}  // namespace msb

// ---------------------------------------------------------------- ABI
extern "C" {

msb_status msb_ctx_create(msb_ctx* out, int device, void* cuda_stream, msb_alloc_fn alloc,
                          msb_free_fn free_fn, void* user) {
  if (!out) return MSB_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return MSB_ECUDA;
  }
  if (device < 0 || device >= n) return MSB_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return MSB_ECUDA;
  msb_ctx c = new msb_ctx_s();
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  c->alloc = alloc;
  c->free_fn = free_fn;
  c->user = user;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  *out = c;
  return MSB_OK;
}

msb_status msb_ctx_destroy(msb_ctx ctx) {
  if (!ctx) return MSB_EINVAL;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  msb::dfree(ctx, ctx->scan_scr);
  msb::dfree(ctx, ctx->gemm_ws);
  delete ctx;
  return MSB_OK;
}

msb_status msb_ctx_set_stream(msb_ctx ctx, void* s) {
  if (!ctx) return MSB_EINVAL;
  ctx->stream = (cudaStream_t)s;
  return MSB_OK;
}

const char* msb_last_error(msb_ctx ctx) { return ctx ? ctx->err : "null context"; }

const char* msb_version(void) { return "libmsb 0.1 sm_100a"; }

int64_t msb_launch_count(void) { return msb::g_launches.load(); }

}  // extern "C"

// ---------------------------------------------------------------- TMA tensor maps (tma.cuh)
#include "tma.cuh"

namespace msb {

static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

bool tma_encode_4d(CUtensorMap* map, const double* base, const uint64_t dims[4],
                   const uint64_t strides_el[3], const uint32_t box[4]) {
  auto fn = tma_encoder();
  if (!fn) return false;
  cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t gs[3] = {strides_el[0] * 8, strides_el[1] * 8, strides_el[2] * 8};
  for (int i = 0; i < 3; ++i)
    if (gs[i] % 16) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16) return false;
  cuuint32_t bd[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), gd, gs, bd, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace msb
