// Development microbenchmark: one modified Gram-Schmidt step (w -= h v_{i-1};
// h_i = w . v_i, last-block reduction) as a chain of 24 graph-launched
// kernels, n = config 5's 1.18M doubles. Variants: grid-stride (as in
// kernels.cu), loads hoisted (unroll 4), grid sizes.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a mgs_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned counter;
__device__ double partial[4096];
__device__ double H[64];

__device__ double block_sum(double v) {
  __shared__ double sh[32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
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
    if (threadIdx.x == 0) { *out = a * 1e-30; counter = 0; }
  }
}

__global__ void mgs0(double* __restrict__ w, const double* V, long ldv, long n, int i) {
  const double hp = H[i - 1];
  const double* vp = V + (i - 1) * ldv;
  const double* vi = V + i * ldv;
  double s = 0;
  for (long t = blockIdx.x * long(blockDim.x) + threadIdx.x; t < n; t += long(gridDim.x) * blockDim.x) {
    const double wt = w[t] - hp * vp[t];
    w[t] = wt;
    s = fma(wt, vi[t], s);
  }
  fin(s, &H[i]);
}
template <int U>
__global__ void mgsU(double* __restrict__ w, const double* __restrict__ V, long ldv, long n, int i) {
  const double hp = H[i - 1];
  const double* vp = V + (i - 1) * ldv;
  const double* vi = V + i * ldv;
  double s = 0;
  const long stride = long(gridDim.x) * blockDim.x;
  for (long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x; t0 < n; t0 += U * stride) {
    double wv[U], pv[U], iv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n) { wv[u] = w[t]; pv[u] = vp[t]; iv[u] = vi[t]; }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n) {
        const double wt = wv[u] - hp * pv[u];
        w[t] = wt;
        s = fma(wt, iv[u], s);
      }
    }
  }
  fin(s, &H[i]);
}

__device__ double part2[2 * 4096];
/// the step's h comes from the previous step's per-block partials, summed by
/// every block in the same order (no atomics, no fence, no last block)
template <int U>
__global__ void mgsP(double* __restrict__ w, const double* __restrict__ V, long ldv, long n, int i) {
  const double* vp = V + (i - 1) * ldv;
  const double* vi = V + i * ldv;
  const long stride = long(gridDim.x) * blockDim.x;
  const long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x;
  double wv[U], pv[U], iv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long t = t0 + u * stride;
    if (t < n) { wv[u] = w[t]; pv[u] = vp[t]; iv[u] = vi[t]; }
  }
  __shared__ double hs;
  const double* prev = part2 + ((i - 1) & 1) * 4096;
  double a = 0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) a += prev[b];
  a = block_sum(a);
  if (threadIdx.x == 0) hs = a * 1e-30;
  __syncthreads();
  const double hp = hs;
  if (blockIdx.x == 0 && threadIdx.x == 0) H[i - 1] = hp;
  double s = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long t = t0 + u * stride;
    if (t < n) {
      const double wt = wv[u] - hp * pv[u];
      w[t] = wt;
      s = fma(wt, iv[u], s);
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part2[(i & 1) * 4096 + blockIdx.x] = s;
}
__device__ double st_i[64];
/// as mgsP, but the step index comes from device memory (dependent address)
template <int U, bool SetCond>
__global__ void mgsD(double* __restrict__ w, const double* __restrict__ V, long ldv, long n, int u,
                     cudaGraphConditionalHandle h) {
  const int i = int(st_i[0]) + u;
  const double* vp = V + (i - 1) * ldv;
  const double* vi = V + i * ldv;
  const long stride = long(gridDim.x) * blockDim.x;
  const long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x;
  double wv[U], pv[U], iv[U];
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const long t = t0 + q * stride;
    if (t < n) { wv[q] = w[t]; pv[q] = vp[t]; iv[q] = vi[t]; }
  }
  __shared__ double hs;
  const double* prev = part2 + ((i - 1) & 1) * 4096;
  double a = 0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) a += prev[b];
  a = block_sum(a);
  if (threadIdx.x == 0) hs = a * 1e-30;
  __syncthreads();
  const double hp = hs;
  if (blockIdx.x == 0 && threadIdx.x == 0) H[i - 1] = hp;
  double s = 0;
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const long t = t0 + q * stride;
    if (t < n) {
      const double wt = wv[q] - hp * pv[q];
      w[t] = wt;
      s = fma(wt, iv[q], s);
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part2[(i & 1) * 4096 + blockIdx.x] = s;
  if (SetCond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 1u);
}
__global__ void bump(int k) { st_i[0] += k; }
__global__ void empty_k() {}
__device__ int cd;
__global__ void countdown(cudaGraphConditionalHandle h) {
  cd -= 1;
  cudaGraphSetConditional(h, cd > 0 ? 1u : 0u);
}
__global__ void set_cd(int v) { cd = v; }
__global__ void fin_only(int i) { fin(double(threadIdx.x), &H[i]); }
template <int U>
__global__ void mgs_nofin(double* __restrict__ w, const double* __restrict__ V, long ldv, long n, int i) {
  const double hp = H[i - 1];
  const double* vp = V + (i - 1) * ldv;
  const double* vi = V + i * ldv;
  double s = 0;
  const long stride = long(gridDim.x) * blockDim.x;
  for (long t0 = blockIdx.x * long(blockDim.x) + threadIdx.x; t0 < n; t0 += U * stride) {
    double wv[U], pv[U], iv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n) { wv[u] = w[t]; pv[u] = vp[t]; iv[u] = vi[t]; }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long t = t0 + u * stride;
      if (t < n) {
        const double wt = wv[u] - hp * pv[u];
        w[t] = wt;
        s = fma(wt, iv[u], s);
      }
    }
  }
  if (s == 12345.0) H[63] = s;
}

int main() {
  const long n = 1179648, ldv = n;
  const int steps = 24;
  double *w, *V, *flush;
  cudaMalloc(&w, n * 8);
  cudaMalloc(&V, (steps + 1) * ldv * 8);
  cudaMalloc(&flush, size_t(512) << 20);
  cudaMemset(w, 0, n * 8);
  cudaMemset(V, 0, (steps + 1) * ldv * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 1; i <= steps; ++i) launch(i);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaMemsetAsync(flush, r, size_t(512) << 20, s);
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-24s %6.2f us per step\n", name, best * 1e3 / steps);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  };
  // the same 24 steps as a while loop of 3 x 8 (conditional body), and 6 x 4
  auto run_while = [&](const char* name, int per, auto launch) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wn;
    cudaGraphAddNode(&wn, g, nullptr, 0, &wp);
    cudaStreamBeginCaptureToGraph(s, wp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    for (int i = 1; i <= per; ++i) launch(i);
    countdown<<<1, 1, 0, s>>>(h);
    cudaGraph_t tmp;
    cudaStreamEndCapture(s, &tmp);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst failed\n"); return; }
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      set_cd<<<1, 1, 0, s>>>(steps / per);
      cudaMemsetAsync(flush, r, size_t(512) << 20, s);
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-24s %6.2f us per step\n", name, best * 1e3 / steps);
  };
  run_while("while 3x8 partials-next", 8, [&](int i) { mgsP<4><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  run_while("while 6x4 partials-next", 4, [&](int i) { mgsP<4><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  {
    cudaGraph_t g0; cudaGraphCreate(&g0, 0);
  }
  run_while("while 3x8 devidx", 8, [&](int i) { if (i == 1) bump<<<1,1,0,s>>>(0); mgsD<4, false><<<1184, 256, 0, s>>>(w, V, ldv, n, i, 0); });
  run_while("while 3x8 empty", 8, [&](int i) { empty_k<<<1184, 256, 0, s>>>(); });
  run("plain partials-next", [&](int i) { mgsP<4><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  for (int grid : {1184, 592, 296, 148}) {
    char nm[64];
    snprintf(nm, 64, "grid-stride g=%d", grid);
    run(nm, [&](int i) { mgs0<<<grid, 256, 0, s>>>(w, V, ldv, n, i); });
    snprintf(nm, 64, "hoisted U=4 g=%d", grid);
    run(nm, [&](int i) { mgsU<4><<<grid, 256, 0, s>>>(w, V, ldv, n, i); });
    snprintf(nm, 64, "hoisted U=8 g=%d", grid);
    run(nm, [&](int i) { mgsU<8><<<grid, 256, 0, s>>>(w, V, ldv, n, i); });
  }
  run("partials-next U=4 g=1184", [&](int i) { mgsP<4><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  run("partials-next U=8 g=592", [&](int i) { mgsP<8><<<592, 256, 0, s>>>(w, V, ldv, n, i); });
  run("partials-next U=16 g=296", [&](int i) { mgsP<16><<<296, 256, 0, s>>>(w, V, ldv, n, i); });
  run("partials-next U=5 g=1184", [&](int i) { mgsP<5><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  run("empty 1 block", [&](int i) { empty_k<<<1, 32, 0, s>>>(); });
  run("empty 1184 blocks", [&](int i) { empty_k<<<1184, 256, 0, s>>>(); });
  run("fin only 1184", [&](int i) { fin_only<<<1184, 256, 0, s>>>(i); });
  run("fin only 296", [&](int i) { fin_only<<<296, 256, 0, s>>>(i); });
  run("no fin U=4 g=592", [&](int i) { mgs_nofin<4><<<592, 256, 0, s>>>(w, V, ldv, n, i); });
  run("no fin U=4 g=1184", [&](int i) { mgs_nofin<4><<<1184, 256, 0, s>>>(w, V, ldv, n, i); });
  run("hoisted U=2 g=1184 512t", [&](int i) { mgsU<2><<<1184/2, 512, 0, s>>>(w, V, ldv, n, i); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
