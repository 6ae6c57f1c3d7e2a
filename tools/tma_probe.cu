// Development probe: read-only HBM streaming ceilings on sm_100a for the
// patch-record access pattern (one contiguous chunk per CTA, one TMA bulk copy
// onto an mbarrier), against plain vectorised loads and a persistent ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(
          su32(bar)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma(void* dst, const void* src, unsigned bytes, unsigned long long* bar, int hint) {
  unsigned long long pol;
  if (hint)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}

// one chunk per CTA
__global__ void k_oneshot(const double* src, size_t chunk_d, double* out, int hint) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    bar_init(&bar);
    tma(sm, src + blockIdx.x * chunk_d, unsigned(chunk_d * 8), &bar, hint);
  }
  __syncthreads();
  bar_wait(&bar, 0);
  double s = 0;
  for (size_t i = threadIdx.x; i < chunk_d; i += blockDim.x) s += sm[i];
  if (s == 12345.678) out[blockIdx.x] = s;
}

// persistent: each CTA walks chunks blockIdx.x, +gridDim.x, ... with a `st`-stage ring
__global__ void k_ring(const double* src, size_t chunk_d, int nchunks, int st, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar[8];
  if (threadIdx.x == 0)
    for (int i = 0; i < st; ++i) bar_init(&bar[i]);
  __syncthreads();
  int k = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < st; ++i) {
      const int c = blockIdx.x + i * gridDim.x;
      if (c < nchunks) tma(sm + i * chunk_d, src + c * chunk_d, unsigned(chunk_d * 8), &bar[i], 1);
    }
  double s = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    const int slot = k % st;
    bar_wait(&bar[slot], (k / st) & 1);
    for (size_t i = threadIdx.x; i < chunk_d; i += blockDim.x) s += sm[slot * chunk_d + i];
    __syncthreads();
    const int cn = c + st * gridDim.x;
    if (threadIdx.x == 0 && cn < nchunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma(sm + slot * chunk_d, src + cn * chunk_d, unsigned(chunk_d * 8), &bar[slot], 1);
    }
  }
  if (s == 12345.678) out[blockIdx.x] = s;
}

__global__ void k_ldg(const double2* src, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double2 v = __ldg(src + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[blockIdx.x] = s;
}

int main() {
  const size_t bytes = size_t(1) << 30;  // 1 GiB read per launch
  double* src;
  double* out;
  cudaMalloc(&src, bytes);
  cudaMalloc(&out, 1 << 24);
  cudaMemset(src, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  for (int blocks : {148 * 8, 148 * 32})
    printf("ldg.v2 stream, %d CTAs x 256: %.0f GB/s\n", blocks,
           timeit([&] { k_ldg<<<blocks, 256>>>((const double2*)src, bytes / 16, out); }));
  cudaFuncSetAttribute(k_oneshot, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int kb : {4, 8, 16, 32, 64}) {
    const size_t cd = size_t(kb) * 1024 / 8;
    const int n = int(bytes / (cd * 8));
    for (int hint : {0, 1})
      printf("oneshot TMA %2d KB/CTA (64 thr, hint %d): %.0f GB/s\n", kb, hint,
             timeit([&] { k_oneshot<<<n, 64, cd * 8>>>(src, cd, out, hint); }));
  }
  for (int kb : {8, 16, 32})
    for (int st : {2, 4, 6})
      for (int per_sm : {1, 2, 4}) {
        const size_t cd = size_t(kb) * 1024 / 8;
        if (cd * 8 * st * per_sm > 220 * 1024) continue;
        const int n = int(bytes / (cd * 8));
        printf("ring TMA %2d KB x %d stages, %d CTA/SM: %.0f GB/s\n", kb, st, per_sm,
               timeit([&] { k_ring<<<148 * per_sm, 128, cd * 8 * st>>>(src, cd, n, st, out); }));
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
