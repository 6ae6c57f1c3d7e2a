// Small lowest-order levels (bs = 2) in one persistent CTA.
//
// Level 1 of a 16x16 base mesh needs 50 dependent waves per multiplicative
// sweep (the reference's ascending-vertex order, smoother.hpp:53-57), each
// only ~20 patches wide: launch latency, not bandwidth, bounds it. Here a
// single 1024-thread CTA runs a whole pre- (resp. post-) smoothing phase of
// the V-cycle: x, b and every index array of the level (wave lists, patch
// facets, inverse offsets, block columns) are staged in shared memory once,
// so a wave costs one L2 round trip for the A rows and patch inverses plus
// two __syncthreads(). Symmetric operators only.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

namespace {

constexpr int kThreads = 1024;
constexpr int kPerPass = kThreads / 16;  // 16 threads (rows) per patch

struct SmallView {
  double *sx, *sb, *rr;
  int *wave_ptr, *wave, *nf, *fac, *off, *cols;
};

__device__ SmallView stage(const Bsr& A, const Patches& P, const int* __restrict__ wave_ptr, int nwaves, double* sm) {
  const int n = A.nb * 2, npch = P.n;
  SmallView v;
  v.sx = sm;
  v.sb = sm + n;
  v.rr = v.sb + n;
  int* ip = reinterpret_cast<int*>(v.rr + kThreads);
  v.wave_ptr = ip;
  v.wave = v.wave_ptr + (nwaves + 1);
  v.nf = v.wave + npch;
  v.off = v.nf + npch;
  v.cols = v.off + npch;
  v.fac = v.cols + A.nb * kSlots;
  for (int i = threadIdx.x; i <= nwaves; i += blockDim.x) v.wave_ptr[i] = wave_ptr[i];
  for (int i = threadIdx.x; i < npch; i += blockDim.x) {
    v.wave[i] = P.wave[i];
    v.nf[i] = P.nf[i];
    v.off[i] = int(P.off[i]);
  }
  for (int i = threadIdx.x; i < npch * kMaxPatchF; i += blockDim.x) v.fac[i] = P.fac[i];
  for (int i = threadIdx.x; i < A.nb * kSlots; i += blockDim.x) v.cols[i] = A.cols[i];
  return v;
}

__device__ void sweeps(const Bsr& A, const Patches& P, const SmallView& v, int nwaves, int nsweeps, bool reverse) {
  const int pl = threadIdx.x >> 4, row = threadIdx.x & 15;
  for (int s = 0; s < nsweeps; ++s)
    for (int wi = 0; wi < nwaves; ++wi) {
      const int w = reverse ? nwaves - 1 - wi : wi;
      const int w0 = v.wave_ptr[w], w1 = v.wave_ptr[w + 1];
      for (int base = w0; base < w1; base += kPerPass) {
        const int q = base + pl;
        int np = 0, g = 0;
        double inv[2 * kMaxPatchF];
        if (q < w1) {
          const int p = v.wave[q];
          np = 2 * v.nf[p];
          if (row < np) {
            const int f = v.fac[p * kMaxPatchF + (row >> 1)], i = row & 1;
            g = 2 * f + i;
            // row `row` of the packed symmetric inverse (lower triangle by columns)
            const double* iv = P.inv + v.off[p];
            const int ct = row * np - row * (row - 1) / 2 - row;
#pragma unroll
            for (int j = 0; j < 2 * kMaxPatchF; ++j)
              inv[j] = j < np ? __ldg(iv + (j >= row ? ct + j : j * np - j * (j - 1) / 2 + (row - j))) : 0.0;
            double r = v.sb[g];
#pragma unroll
            for (int sl = 0; sl < kSlots; ++sl) {
              const int c = v.cols[f * kSlots + sl];
              if (c < 0) continue;
              const double2 a = __ldg(reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * 2 + i) * 2));
              r = fma(-a.x, v.sx[2 * c], r);
              r = fma(-a.y, v.sx[2 * c + 1], r);
            }
            v.rr[threadIdx.x] = r;
          }
        }
        __syncthreads();
        if (row < np) {
          double d = 0.0;
#pragma unroll
          for (int j = 0; j < 2 * kMaxPatchF; ++j)
            if (j < np) d = fma(inv[j], v.rr[(pl << 4) + j], d);
          v.sx[g] += d;
        }
        __syncthreads();
      }
    }
}

/// x = 0; pre-smooth; r = b - A x; rc = P^T r (reference multigrid.hpp:174-178)
__global__ void __launch_bounds__(kThreads) k_small_pre(Bsr A, Patches P, const int* __restrict__ wave_ptr, int nwaves,
                                                        int nsweeps, BlockCsr PT, const double* __restrict__ b,
                                                        double* __restrict__ x, double* __restrict__ rc) {
  extern __shared__ double sm[];
  const int n = A.nb * 2;
  SmallView v = stage(A, P, wave_ptr, nwaves, sm);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    v.sx[i] = 0.0;
    v.sb[i] = b[i];
  }
  __syncthreads();
  sweeps(A, P, v, nwaves, nsweeps, false);
  // residual in place of b (each row reads only its own b entry and x)
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int f = t >> 1, i = t & 1;
    double s = 0.0;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int c = v.cols[f * kSlots + sl];
      if (c < 0) continue;
      const double2 a = __ldg(reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * 2 + i) * 2));
      s = fma(a.x, v.sx[2 * c], s);
      s = fma(a.y, v.sx[2 * c + 1], s);
    }
    x[t] = v.sx[t];
    v.sb[t] = v.sb[t] - s;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < PT.nrows * 2; t += blockDim.x) {
    const int cb = t >> 1, c = t & 1;
    double s = 0.0;
    for (int q = PT.ptr[cb]; q < PT.ptr[cb + 1]; ++q) {
      const int fb = PT.col[q];
      const double* pv = PT.val + size_t(q) * 4 + c * 2;
      s = fma(pv[0], v.sb[2 * fb], s);
      s = fma(pv[1], v.sb[2 * fb + 1], s);
    }
    rc[t] = s;
  }
}

/// x += P e; post-smooth (reverse sweep) (reference multigrid.hpp:181-182)
__global__ void __launch_bounds__(kThreads) k_small_post(Bsr A, Patches P, const int* __restrict__ wave_ptr,
                                                         int nwaves, int nsweeps, BlockCsr Pm,
                                                         const double* __restrict__ e, const double* __restrict__ b,
                                                         double* __restrict__ x) {
  extern __shared__ double sm[];
  const int n = A.nb * 2;
  SmallView v = stage(A, P, wave_ptr, nwaves, sm);
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int f = t >> 1, c = t & 1;
    double s = 0.0;
    for (int q = Pm.ptr[f]; q < Pm.ptr[f + 1]; ++q) {
      const int cb = Pm.col[q];
      const double* pv = Pm.val + size_t(q) * 4 + c * 2;
      s = fma(pv[0], e[size_t(cb) * 2], s);
      s = fma(pv[1], e[size_t(cb) * 2 + 1], s);
    }
    v.sx[t] = x[t] + s;
    v.sb[t] = b[t];
  }
  __syncthreads();
  sweeps(A, P, v, nwaves, nsweeps, true);
  for (int t = threadIdx.x; t < n; t += blockDim.x) x[t] = v.sx[t];
}

size_t smem_bytes(int nb, int npatch, int nwaves) {
  return sizeof(double) * (size_t(4) * nb + kThreads) +
         sizeof(int) * (size_t(nwaves + 1) + size_t(npatch) * (3 + kMaxPatchF) + size_t(nb) * kSlots);
}

}  // namespace

bool small_level_fits(int nb, int npatch, int nwaves) { return smem_bytes(nb, npatch, nwaves) <= 220 * 1024; }

void small_pre(const Bsr& A, const Patches& P, const int* wave_ptr, int nwaves, int sweeps, const BlockCsr& PT,
               const double* b, double* x, double* rc, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_small_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_small_post, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  k_small_pre<<<1, kThreads, smem_bytes(A.nb, P.n, nwaves), s>>>(A, P, wave_ptr, nwaves, sweeps, PT, b, x, rc);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch: ") + cudaGetErrorString(err));
}

void small_post(const Bsr& A, const Patches& P, const int* wave_ptr, int nwaves, int sweeps, const BlockCsr& Pm,
                const double* e, const double* b, double* x, cudaStream_t s) {
  k_small_post<<<1, kThreads, smem_bytes(A.nb, P.n, nwaves), s>>>(A, P, wave_ptr, nwaves, sweeps, Pm, e, b, x);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch: ") + cudaGetErrorString(err));
}

}  // namespace dev
}  // namespace hpmg
