// Toolchain/box probe: FP64 stream bandwidth and FMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void triad(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ c, size_t n, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    c[i] = make_double2(x.x + s * y.x, x.y + s * y.y);
  }
}
__global__ void fma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.5, c1 = 0.25, c2 = 0.125, c3 = 0.0625;
  for (int i = 0; i < iters; ++i) {
    c0 = fma(c0, b, a); c1 = fma(c1, b, a); c2 = fma(c2, b, a); c3 = fma(c3, b, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("dev %s sms %d cc %d.%d l2 %d MB smem/blk optin %zu KB\n", p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin >> 10);
  size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB per array
  double2 *a, *b, *c; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&c, n * 16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); triad<<<blocks, 256>>>(a, b, c, n, 1.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("triad blocks=%d: %.1f GB/s\n", blocks, 3.0 * n * 16 / best / 1e6);
  }
  double* o; cudaMalloc(&o, 148 * 64 * 256 * 8);
  int iters = 1 << 16;
  fma_loop<<<148 * 64, 256>>>(o, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); fma_loop<<<148 * 64, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("fp64 fma: %.2f TFLOP/s\n", 2.0 * 4 * iters * 148.0 * 64 * 256 / ms / 1e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
