// Development microbenchmark: grid-stride one-double-per-thread vector kernels
// vs double2 x unroll-4 versions, warm and after an L2 flush (n = config 2's
// 1.57M doubles). nvcc -O3 -gencode arch=compute_100a,code=sm_100a vec_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned counter;
__device__ double partial[4096];

__device__ double block_sum(double v) {
  __shared__ double sh[32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ void fin(double s, double* out) {
  __shared__ bool last;
  s = block_sum(s);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(&counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double a = 0;
    for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x) a += __ldcg(&partial[i]);
    a = block_sum(a);
    if (threadIdx.x == 0) { *out = a; counter = 0; }
  }
}

__global__ void fill1(double* x, long n) {
  for (long t = blockIdx.x * long(blockDim.x) + threadIdx.x; t < n; t += long(gridDim.x) * blockDim.x) x[t] = 0.0;
}
__global__ void fill2(double* x, long n) {
  double2* x2 = reinterpret_cast<double2*>(x);
  const long n2 = n / 2;
  for (long t = blockIdx.x * long(blockDim.x) + threadIdx.x; t < n2; t += long(gridDim.x) * blockDim.x)
    x2[t] = make_double2(0.0, 0.0);
}
__global__ void upd1(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                     const double* __restrict__ q, double a, long n, double* out) {
  double s = 0;
  for (long t = blockIdx.x * long(blockDim.x) + threadIdx.x; t < n; t += long(gridDim.x) * blockDim.x) {
    x[t] += a * p[t];
    const double rt = r[t] - a * q[t];
    r[t] = rt;
    s = fma(rt, rt, s);
  }
  fin(s, out);
}
template <int U>
__global__ void updv(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                     const double* __restrict__ q, double a, long n, double* out) {
  double s = 0;
  const long n2 = n / 2;
  double2 *x2 = (double2*)x, *r2 = (double2*)r;
  const double2 *p2 = (const double2*)p, *q2 = (const double2*)q;
  const long stride = long(gridDim.x) * blockDim.x;
  for (long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x; t0 < n2; t0 += stride * U) {
    double2 xv[U], rv[U], pv[U], qv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n2) { xv[u] = x2[t]; rv[u] = r2[t]; pv[u] = __ldcs(p2 + t); qv[u] = __ldcs(q2 + t); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n2) {
        xv[u].x += a * pv[u].x; xv[u].y += a * pv[u].y;
        rv[u].x -= a * qv[u].x; rv[u].y -= a * qv[u].y;
        x2[t] = xv[u]; r2[t] = rv[u];
        s = fma(rv[u].x, rv[u].x, s); s = fma(rv[u].y, rv[u].y, s);
      }
    }
  }
  fin(s, out);
}
__global__ void dot1(const double* __restrict__ a, const double* __restrict__ b, long n, double* out) {
  double s = 0;
  for (long t = blockIdx.x * long(blockDim.x) + threadIdx.x; t < n; t += long(gridDim.x) * blockDim.x) s = fma(a[t], b[t], s);
  fin(s, out);
}
template <int U>
__global__ void dotv(const double* __restrict__ a, const double* __restrict__ b, long n, double* out) {
  double s0 = 0, s1 = 0;
  const long n2 = n / 2, stride = long(gridDim.x) * blockDim.x;
  const double2 *a2 = (const double2*)a, *b2 = (const double2*)b;
  for (long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x; t0 < n2; t0 += stride * U) {
    double2 av[U], bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n2) { av[u] = a2[t]; bv[u] = b2[t]; } else { av[u] = bv[u] = make_double2(0, 0); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { s0 = fma(av[u].x, bv[u].x, s0); s1 = fma(av[u].y, bv[u].y, s1); }
  }
  fin(s0 + s1, out);
}

int main() {
  const long n = 1572864;  // ~config 2
  double *x, *r, *p, *q, *out, *flush;
  cudaMalloc(&x, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&p, n * 8); cudaMalloc(&q, n * 8); cudaMalloc(&out, 64);
  const size_t fl = size_t(256) << 20;
  cudaMalloc(&flush, fl);
  cudaMemset(x, 0, n * 8); cudaMemset(r, 0, n * 8); cudaMemset(p, 0, n * 8); cudaMemset(q, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double bytes) {
    for (int cold = 0; cold < 2; ++cold) {
      float tot = 0;
      const int reps = 50;
      for (int i = 0; i < reps; ++i) {
        if (cold) cudaMemsetAsync(flush, i, fl);
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
        if (cold) { // measure a cold launch: flush, then time one
          cudaMemsetAsync(flush, i + 1, fl);
          cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1); tot += ms - 0;  // counts both
        }
      }
      const double us = tot * 1e3 / (cold ? 2 * reps : reps);
      printf("%-22s %s %7.2f us  %7.0f GB/s\n", name, cold ? "mixed" : "warm ", us, bytes / us * 1e-3);
    }
  };
  const int R = 1184;
  timeit("fill1", [&] { fill1<<<(n + 255) / 256, 256>>>(x, n); }, 8.0 * n);
  timeit("fill2", [&] { fill2<<<(n / 2 + 255) / 256, 256>>>(x, n); }, 8.0 * n);
  timeit("fill2 g=1184", [&] { fill2<<<R, 256>>>(x, n); }, 8.0 * n);
  timeit("upd1 g=1184", [&] { upd1<<<R, 256>>>(x, r, p, q, 0.5, n, out); }, 48.0 * n);
  timeit("updv<1> g=1184", [&] { updv<1><<<R, 256>>>(x, r, p, q, 0.5, n, out); }, 48.0 * n);
  timeit("updv<2> g=1184", [&] { updv<2><<<R, 256>>>(x, r, p, q, 0.5, n, out); }, 48.0 * n);
  timeit("updv<2> g=592", [&] { updv<2><<<592, 256>>>(x, r, p, q, 0.5, n, out); }, 48.0 * n);
  timeit("dot1 g=1184", [&] { dot1<<<R, 256>>>(x, r, n, out); }, 16.0 * n);
  timeit("dotv<2> g=1184", [&] { dotv<2><<<R, 256>>>(x, r, n, out); }, 16.0 * n);
  timeit("dotv<4> g=592", [&] { dotv<4><<<592, 256>>>(x, r, n, out); }, 16.0 * n);
  timeit("dotv<2> g=296x512", [&] { dotv<2><<<296, 512>>>(x, r, n, out); }, 16.0 * n);
  return 0;
}
