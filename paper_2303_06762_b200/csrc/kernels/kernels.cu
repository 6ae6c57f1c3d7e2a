// sm_100a FP64 kernels of the hp-MG solve path. Everything here is
// HBM-bandwidth bound (~0.25 flop/byte) except the element condensation,
// which is FP64-FMA bound; see DESIGN.md for the per-kernel roofline.
//
// Determinism: every reduction uses a fixed grid (kRedBlocks) with a fixed
// thread-to-index map, per-block tree sums and a final fixed-order sum by the
// last block to finish (ticket counter), so repeated runs are bit-identical
// (reference tests/test_multigrid.cpp:109-119 asks for that).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

#define HPMG_LAUNCH_CHECK()                                                                        \
  do {                                                                                             \
    cudaError_t err__ = cudaGetLastError();                                                        \
    if (err__ != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (") + __func__ + "): " + cudaGetErrorString(err__)); \
  } while (0)

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

/// Block tree sum (or max); result valid in thread 0. All threads must call.
template <bool kMax>
__device__ double block_reduce(double v) {
  __shared__ double sh[32];
  v = kMax ? warp_max(v) : warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? sh[lane] : (kMax ? -1.0 : 0.0);
    v = kMax ? warp_max(v) : warp_sum(v);
  }
  return v;
}

/// Writes the block partial, the last block sums all partials in fixed order.
template <bool kMax>
__device__ void finalize(double v, Reduce red, double* out) {
  __shared__ bool last;
  v = block_reduce<kMax>(v);
  if (threadIdx.x == 0) {
    red.partial[blockIdx.x] = v;
    __threadfence();
    unsigned t = atomicAdd(red.counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = kMax ? -1.0 : 0.0;
    for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      double p = __ldcg(&red.partial[i]);
      s = kMax ? fmax(s, p) : s + p;
    }
    s = block_reduce<kMax>(s);
    if (threadIdx.x == 0) {
      *out = s;
      *red.counter = 0u;
    }
  }
}

/// finalize() followed by `epi(sum)` on thread 0 of the last block (after the
/// sum is stored): the single-thread bookkeeping of a Krylov loop rides on
/// the reduction kernel instead of a launch of its own.
template <class Epi>
__device__ void finalize_then(double v, Reduce red, double* out, Epi epi) {
  __shared__ bool last;
  v = block_reduce<false>(v);
  if (threadIdx.x == 0) {
    red.partial[blockIdx.x] = v;
    __threadfence();
    unsigned t = atomicAdd(red.counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += __ldcg(&red.partial[i]);
    s = block_reduce<false>(s);
    if (threadIdx.x == 0) {
      *out = s;
      *red.counter = 0u;
      epi(s);
    }
  }
}

/// Grid of a fixed-grid (reduction) kernel: kRedBlocks CTAs of 256 threads,
/// or fewer when the kernel's registers allow fewer than 8 CTAs per SM, so
/// that every CTA is resident at once (no tail wave of leftover CTAs).
/// Fixed per kernel, so reductions stay deterministic.
template <class K>
int resident_grid(K kernel) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 256, 0);
  const int g = sms * (per > 0 ? per : 1);
  return g < kRedBlocks ? g : kRedBlocks;
}

/// Grid of an element-wise (grid-stride) kernel: one CTA per `threads`
/// elements; a grid of one to three waves of resident CTAs (2048 threads per
/// SM) is folded into one wave, since a 1.3-wave grid leaves its second wave
/// latency-bound at low occupancy (config 2 V-cycle 0.721 -> 0.715 ms). Longer
/// streaming grids keep one element per thread (more loads in flight: the
/// 6,128-CTA head operator apply runs 86 us instead of 99 us capped).
inline int grid_for(int64_t n, int threads) {
  static const int64_t sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return int64_t(v > 0 ? v : 148);
  }();
  const int64_t wave = sms * std::max(1, 2048 / threads);
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > wave && g < 3 * wave) g = wave;
  if (g > 148 * 64) g = 148 * 64;
  return int(g);
}

// ---------------------------------------------------------------- condense
// 6 CTAs per SM (the shared-memory limit at k = 3) instead of the 4 that 127
// registers allowed: 80 registers, 48 bytes of stack; head condensation
// 12.2 -> 10.2 ms at config 2 (ncu)
__global__ void __launch_bounds__(128, 6) k_condense(RefT T, const ElemGeo* __restrict__ geo, CondenseParams prm,
                                                     const double* __restrict__ load,
                           int load_stride, double* __restrict__ out, int stride, const double* __restrict__ wind,
                           const double* __restrict__ mfield) {
  extern __shared__ double smem[];
  __shared__ ElemGeo g;
  const int e = blockIdx.x;
  if (threadIdx.x < int(sizeof(ElemGeo) / sizeof(double)))
    reinterpret_cast<double*>(&g)[threadIdx.x] = reinterpret_cast<const double*>(geo + e)[threadIdx.x];
  __syncthreads();
  double* o = out + size_t(e) * stride;
  const double* ld = prm.load_mode ? load + size_t(e) * load_stride : nullptr;
  const double* xw = wind ? wind + size_t(e) * T.nv : nullptr;      // local wind coefficients (Oseen)
  const double* xm = mfield ? mfield + size_t(e) * T.nv : nullptr;  // local mass field (pseudo-time)
  condense_element(threadIdx.x, blockDim.x, T, g, prm, ld, smem, o, o + T.nc * T.nc, nullptr, nullptr, nullptr, xw,
                   xm);
}

/// recover_locals (reference inc/assembly.hpp:513-549) for every element:
/// gathers the element's skeleton coefficients from the full compound vector
/// (reference layout: all flux modes, then all tangential modes).
__global__ void __launch_bounds__(128, 6) k_recover(RefT T, const ElemGeo* __restrict__ geo, CondenseParams prm,
                                                    const double* __restrict__ load,
                          int load_stride, const int* __restrict__ elem_facets, long long nflux,
                          const double* __restrict__ compound, double* __restrict__ interior,
                          double* __restrict__ pres, double* __restrict__ grad, const double* __restrict__ wind,
                          const double* __restrict__ mfield) {
  extern __shared__ double smem[];
  __shared__ ElemGeo g;
  const int e = blockIdx.x;
  const int nfd = T.nfd, nc = T.nc, nz = T.no + T.ns - 1;
  double* xc = smem;
  double* zb = xc + nc;
  double* gb = zb + nz + 1;
  double* scratch = gb + 4 * T.ns;
  if (threadIdx.x < int(sizeof(ElemGeo) / sizeof(double)))
    reinterpret_cast<double*>(&g)[threadIdx.x] = reinterpret_cast<const double*>(geo + e)[threadIdx.x];
  for (int a = threadIdx.x; a < nc; a += blockDim.x) {
    const bool tang = a >= 3 * nfd;
    const int la = tang ? a - 3 * nfd : a;
    const long long f = elem_facets[e * 3 + la / nfd];
    xc[a] = compound[(tang ? nflux : 0) + f * nfd + la % nfd];
  }
  __syncthreads();
  const double* ld = prm.load_mode ? load + size_t(e) * load_stride : nullptr;
  const double* xw = wind ? wind + size_t(e) * T.nv : nullptr;
  const double* xm = mfield ? mfield + size_t(e) * T.nv : nullptr;
  condense_element(threadIdx.x, blockDim.x, T, g, prm, ld, scratch, nullptr, nullptr, xc, zb, gb, xw, xm);
  __syncthreads();
  for (int j = threadIdx.x; j < T.no; j += blockDim.x) interior[size_t(e) * T.no + j] = zb[j];
  for (int m = threadIdx.x; m < T.ns - 1; m += blockDim.x) pres[size_t(e) * (T.ns - 1) + m] = zb[T.no + m];
  for (int r = threadIdx.x; r < 4 * T.ns; r += blockDim.x) grad[size_t(e) * 4 * T.ns + r] = gb[r];
}

__device__ __forceinline__ int local_dof(int lf, int ii, int nfd) {
  // block entry ii = 2 i + t  ->  reference local index (flux: lf*nfd+i, tang: 3nfd + lf*nfd + i)
  const int i = ii >> 1, t = ii & 1;
  return t == 0 ? lf * nfd + i : 3 * nfd + lf * nfd + i;
}

__global__ void k_assemble_bsr(Bsr A, int nfd, const double* __restrict__ acr, int stride, int nc,
                               const int* __restrict__ gath, const ElemGeo* __restrict__ geo, double inv_eps) {
  const int bs = A.bs, bb = bs * bs;
  const int64_t n = int64_t(A.nb) * kSlots * bb;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rs = t / bb;
    const int ii = int(t % bb) / bs, jj = int(t % bb) % bs;
    if (A.cols[rs] < 0) {
      A.val[t] = 0.0;
      continue;
    }
    const int* gp = gath + rs * 6;
    double v = 0.0, d = 0.0;
    bool has_d = false;
    for (int c = 0; c < 2; ++c) {
      const int e = gp[3 * c];
      if (e < 0) continue;
      const int la = gp[3 * c + 1], lb = gp[3 * c + 2];
      v += acr[size_t(e) * stride + local_dof(la, ii, nfd) * nc + local_dof(lb, jj, nfd)];
      if (ii == 0 && jj == 0) {
        const ElemGeo& g = geo[e];
        const double ia = 1.0 / (0.5 * g.detJ);
        const double bi = (g.fac[la] < 0 ? -2.0 : 2.0) * g.ds[la], bj = (g.fac[lb] < 0 ? -2.0 : 2.0) * g.ds[lb];
        d += ia * bi * bj;
        has_d = true;
      }
    }
    A.val[t] = has_d ? v + inv_eps * d : v;
  }
}

__global__ void k_transpose_bsr(Bsr A, const int* __restrict__ tslot, Bsr AT) {
  const int bs = A.bs, bb = bs * bs;
  const int64_t n = int64_t(A.nb) * kSlots * bb;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rs = t / bb;
    const int ii = int(t % bb) / bs, jj = int(t % bb) % bs;
    const int c = A.cols[rs];
    if (c < 0) {
      AT.val[t] = 0.0;
      continue;
    }
    const int s2 = tslot[rs];
    AT.val[t] = A.val[(int64_t(c) * kSlots + s2) * bb + jj * bs + ii];
  }
}

__global__ void k_assemble_rhs(int nb, int bs, int nfd, const int* __restrict__ row_elems,
                               const int* __restrict__ block_facet, const int* __restrict__ elem_facets,
                               const char* __restrict__ dir, const double* __restrict__ g_fac,
                               const double* __restrict__ acr, int stride, int nc, const ElemGeo* __restrict__ geo,
                               double inv_eps, double* __restrict__ rhs) {
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t / bs), ii = int(t % bs);
    double acc = 0.0, dr = 0.0;
    for (int c = 0; c < 2; ++c) {
      const int e = row_elems[f * 4 + 2 * c];
      if (e < 0) continue;
      const int la = row_elems[f * 4 + 2 * c + 1];
      const int a = local_dof(la, ii, nfd);
      const double* Ae = acr + size_t(e) * stride;
      acc += Ae[nc * nc + a];
      for (int b = 0; b < nc; ++b) {
        const int lb = b < 3 * nfd ? b / nfd : (b - 3 * nfd) / nfd;
        const int gf = elem_facets[e * 3 + lb];
        if (!dir[gf]) continue;
        const int mode = b < 3 * nfd ? b % nfd : (b - 3 * nfd) % nfd;
        const int slot = 2 * mode + (b < 3 * nfd ? 0 : 1);
        acc -= Ae[a * nc + b] * g_fac[size_t(gf) * bs + slot];
      }
      if (ii == 0) {
        const ElemGeo& g = geo[e];
        const double ia = 1.0 / (0.5 * g.detJ);
        const double bi = (g.fac[la] < 0 ? -2.0 : 2.0) * g.ds[la];
        for (int j = 0; j < 3; ++j) {
          const int gj = elem_facets[e * 3 + j];
          if (!dir[gj]) continue;
          const double bj = (g.fac[j] < 0 ? -2.0 : 2.0) * g.ds[j];
          dr -= ia * bi * bj * g_fac[size_t(gj) * bs];
        }
      }
    }
    rhs[t] = ii == 0 ? acc + inv_eps * dr : acc;
  }
  (void)block_facet;
}

// --------------------------------------------------------------- operator
template <int BS>
__global__ void k_spmv(Bsr A, const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ y,
                       int minus, int with_dot, Reduce red, double* dot_out) {
  const int64_t n = int64_t(A.nb) * BS;
  double dacc = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t / BS), i = int(t % BS);
    double s = 0.0;
    // branch-free over the slots (empty ones: column 0 read, contribution
    // selected away), so the loads of all slots can be in flight together
    int c[kSlots];
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) c[sl] = __ldg(&A.cols[f * kSlots + sl]);
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const bool on = c[sl] >= 0;
      const double2* blk = reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * BS + i) * BS);
      const double2* xc = reinterpret_cast<const double2*>(x + size_t(on ? c[sl] : 0) * BS);
#pragma unroll
      for (int j = 0; j < BS / 2; ++j) {
        const double2 a = __ldg(blk + j), xv = xc[j];
        s = fma(on ? a.x : 0.0, on ? xv.x : 0.0, s);  // both zeroed: exact even for non-finite values
        s = fma(on ? a.y : 0.0, on ? xv.y : 0.0, s);
      }
    }
    const double v = minus ? b[t] - s : s;
    y[t] = v;
    if (with_dot) dacc = fma(x[t], v, dacc);
  }
  if (with_dot) finalize<false>(dacc, red, dot_out);
}

/// PCG loop operator apply with the direction update folded in (reference
/// krylov.hpp:46-47,69): Ap = A p' and p'.Ap, where p' = z + beta p when
/// `dir` (every column block is formed on the fly from z and the previous p,
/// which stays untouched: k_pcg_loop_update stores p' with the same
/// arithmetic), p' = p otherwise. A no-op once the loop has stopped.
template <int BS>
__global__ void k_spmv_dir(Bsr A, const double* __restrict__ p, const double* __restrict__ z, double* __restrict__ y,
                           int dir, const double* __restrict__ sc, Reduce red, double* dot_out) {
  if (sc[kScStatus] != kLoopRunning) return;  // grid-uniform
  const double beta = dir ? sc[kScBeta] : 0.0;
  const int64_t n = int64_t(A.nb) * BS;
  double dacc = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t / BS), i = int(t % BS);
    double s = 0.0;
    int c[kSlots];
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) c[sl] = __ldg(&A.cols[f * kSlots + sl]);
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const bool on = c[sl] >= 0;
      const double2* blk = reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * BS + i) * BS);
      const size_t co = size_t(on ? c[sl] : 0) * BS;
      const double2* pc = reinterpret_cast<const double2*>(p + co);
      const double2* zc = reinterpret_cast<const double2*>(z + co);
#pragma unroll
      for (int j = 0; j < BS / 2; ++j) {
        const double2 a = __ldg(blk + j), pv = pc[j];
        double2 xv = pv;
        if (dir) {
          const double2 zv = zc[j];
          xv.x = fma(beta, pv.x, zv.x);
          xv.y = fma(beta, pv.y, zv.y);
        }
        s = fma(on ? a.x : 0.0, on ? xv.x : 0.0, s);
        s = fma(on ? a.y : 0.0, on ? xv.y : 0.0, s);
      }
    }
    y[t] = s;
    const double pt = dir ? fma(beta, p[t], z[t]) : p[t];
    dacc = fma(pt, s, dacc);
  }
  finalize<false>(dacc, red, dot_out);
}

/// A0 = the mode-0 rows (block rows 0 and 1) of every block of A, stored
/// [nb][kSlots][2][BS] so that the head residual streams them contiguously
/// (a column-major ELL variant, one 512-byte stream per (slot, column pair),
/// measured slower at BS = 8: 37 -> 49 us per V-cycle at config 2)
template <int BS>
__global__ void k_extract_mode0(Bsr A, Bsr A0) {
  const int64_t n = int64_t(A.nb) * kSlots * 2 * BS;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t blk = t / (2 * BS);
    const int r = int(t % (2 * BS));  // row i = r / BS, column r % BS
    A0.val[t] = A.val[blk * BS * BS + r];
  }
}
/// Mode-0 rows of E^T (b - A x) (reference transfer.hpp:140-158 applied to
/// the residual of multigrid.hpp:124), from A0 (k_extract_mode0): the two rows
/// of a facet's blocks are 2 x 8 x BS contiguous bytes per slot.
template <int BS>
__global__ void k_inject_residual(Bsr A0, const double* __restrict__ x, const double* __restrict__ b,
                                  double* __restrict__ r0, double* __restrict__ x0_zero) {
  const int64_t n = int64_t(A0.nb) * 2;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t >> 1), i = int(t & 1);
    double s = 0.0;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int c = __ldg(&A0.cols[f * kSlots + sl]);
      if (c < 0) continue;
      const double2* blk = reinterpret_cast<const double2*>(A0.val + (size_t(f * kSlots + sl) * 2 + i) * BS);
      const double2* xc = reinterpret_cast<const double2*>(x + size_t(c) * BS);
#pragma unroll
      for (int j = 0; j < BS / 2; ++j) {
        const double2 a = __ldg(blk + j), xv = xc[j];
        s = fma(a.x, xv.x, s);
        s = fma(a.y, xv.y, s);
      }
    }
    r0[t] = b[size_t(f) * BS + i] - s;
    if (x0_zero) x0_zero[t] = 0.0;  // the lowest-order pre-smoothing starts from x = 0
  }
}

__global__ void k_embed_add(int nb, int bs, const double* __restrict__ e, double* __restrict__ x) {
  const int64_t n = int64_t(nb) * 2;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    x[(t >> 1) * bs + (t & 1)] += e[t];
}

// ------------------------------------------------------------ smoothers
/// Patch matrix gather + Gauss-Jordan inversion with partial pivoting,
/// one CTA per patch; the inverse is stored column-major (or packed).
/// Thread t owns column c = t % W of the augmented [A_pp | I] (W = 2 np_max,
/// blockDim = RG W) and the rows r = t / W + RG i: no index division per
/// element, the pivot-row entry a_kc stays in a register for the step.
/// Per step and entry the arithmetic is the textbook one (pivot: largest
/// |a_ik|, lowest row on ties; a_kc <- a_kc / a_kk; a_rc <- a_rc - a_rk a_kc).
template <int BS>
__global__ void k_patch_inverse(Bsr A, Patches P, int rg) {
  extern __shared__ double aug[];
  const bool packed = P.packed != 0;
  __shared__ int fac[kMaxPatchF];
  __shared__ int piv_row;
  const int p = blockIdx.x;
  const int nf = P.nf[p], np = nf * BS, w = 2 * np;
  const int W = blockDim.x / rg;  // 2 np_max >= w
  const int c = threadIdx.x % W, g = threadIdx.x / W;
  const bool col = c < w;
  if (threadIdx.x < kMaxPatchF) fac[threadIdx.x] = P.fac[p * kMaxPatchF + threadIdx.x];
  __syncthreads();
  if (col) {
    const int fcn = c < np ? fac[c / BS] : -1;
    for (int r = g; r < np; r += rg) {
      double v = 0.0;
      if (c < np) {
        const int fr = fac[r / BS];
        for (int sl = 0; sl < kSlots; ++sl)
          if (A.cols[fr * kSlots + sl] == fcn) {
            v = A.val[(size_t(fr * kSlots + sl) * BS + r % BS) * BS + c % BS];
            break;
          }
      } else {
        v = (c - np == r) ? 1.0 : 0.0;
      }
      aug[r * w + c] = v;
    }
  }
  __syncthreads();
  for (int k = 0; k < np; ++k) {
    if (threadIdx.x < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + threadIdx.x; i < np; i += 32) {
        double v = fabs(aug[i * w + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (threadIdx.x == 0) piv_row = bi;
    }
    __syncthreads();
    const int pr = piv_row;
    if (pr != k && g == 0 && col) {
      const double t = aug[k * w + c];
      aug[k * w + c] = aug[pr * w + c];
      aug[pr * w + c] = t;
    }
    __syncthreads();
    const double inv = 1.0 / aug[k * w + k];
    const double akc = col ? aug[k * w + c] * inv : 0.0;
    __syncthreads();  // every thread has read a_kk and its a_kc
    if (col) {
      if (g == 0) aug[k * w + c] = akc;
      if (c != k)
        for (int r = g; r < np; r += rg)
          if (r != k) aug[r * w + c] -= aug[r * w + k] * akc;
    }
    __syncthreads();
    if (c == k)
      for (int r = g; r < np; r += rg)
        if (r != k) aug[r * w + k] = 0.0;
    // (column k is read again only after the next step's pivot barrier)
  }
  __syncthreads();
  double* out = P.inv + P.off[p];
  if (packed) {
    // symmetric operator: symmetrised inverse, lower triangle packed by columns
    // (column c holds rows c..np-1 at c*np - c(c-1)/2)
    for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
      const int cc = e / np, r = e % np;
      if (r < cc) continue;
      out[cc * np - cc * (cc - 1) / 2 + (r - cc)] = 0.5 * (aug[r * w + np + cc] + aug[cc * w + np + r]);
    }
  } else {
    for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
      const int cc = e / np, r = e % np;  // column-major: (r, c) at c*np + r
      out[e] = aug[r * w + np + cc];
    }
  }
}

/// Symmetric multiplicative wave, several patches per CTA (TP threads each).
/// Latency structure: one dependent round for the patch metadata, then every
/// independent load of the patch (its packed inverse, U per thread, and its
/// A rows) is issued back to back; the x gathers are the only second round.
/// The CTA also bulk-prefetches its slice of the NEXT wave's inverses into
/// L2 (they are contiguous because patches are numbered in wave order).
template <int BS, int TP, int U>
__global__ void __launch_bounds__(128) k_gs_wave_sym(Bsr A, Patches P, int p0, int p1, int pk_max,
                                                     const double* __restrict__ b, double* __restrict__ x,
                                                     const char* pf_ptr, unsigned pf_bytes) {
  extern __shared__ double sm[];
  const int ppc = blockDim.x / TP, lp = threadIdx.x / TP, t = threadIdx.x % TP;
  double* sp = sm + size_t(lp) * pk_max;
  double* r = sm + size_t(ppc) * pk_max + lp * TP;
  if (pf_bytes && threadIdx.x == 0) {
    const unsigned chunk = ((pf_bytes / gridDim.x) + 15u) & ~15u;
    const unsigned beg = chunk * blockIdx.x;
    if (beg < pf_bytes) {
      const unsigned len = min(chunk, pf_bytes - beg) & ~15u;
      if (len) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf_ptr + beg), "r"(len) : "memory");
    }
  }
  const int p = p0 + blockIdx.x * ppc + lp;
  int np = 0, f = 0;
  if (p < p1) {
    np = P.nf[p] * BS;
    const int64_t off = P.off[p];
    if (t < np) f = P.fac[p * kMaxPatchF + t / BS];
    const double* src = P.inv + off;
    const int tot = np * (np + 1) / 2;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = t + u * TP;
      v[u] = k < tot ? __ldg(src + k) : 0.0;
    }
    for (int k = t + U * TP; k < tot; k += TP) sp[k] = __ldg(src + k);  // patches above 6 facets
    double s = 0.0;
    if (t < np) {
      const int i = t % BS;
      s = b[size_t(f) * BS + i];
      int cc[kSlots];
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) cc[sl] = __ldg(&A.cols[f * kSlots + sl]);
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        if (cc[sl] < 0) continue;
        const double2* blk = reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * BS + i) * BS);
        const double2* xc = reinterpret_cast<const double2*>(x + size_t(cc[sl]) * BS);
#pragma unroll
        for (int j = 0; j < BS / 2; ++j) {
          const double2 a = __ldg(blk + j), xv = xc[j];
          s = fma(-a.x, xv.x, s);
          s = fma(-a.y, xv.y, s);
        }
      }
      r[t] = s;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = t + u * TP;
      if (k < tot) sp[k] = v[u];
    }
  }
  __syncthreads();
  if (t < np) {
    // S(t, j): j >= t in column t, j < t in column j (packed lower by columns)
    const int ct = t * np - t * (t - 1) / 2 - t;
    double d0 = 0.0, d1 = 0.0;
    int j = 0;
    for (; j + 1 < np; j += 2) {
      const int i0 = j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j);
      const int j1 = j + 1;
      const int i1 = j1 >= t ? ct + j1 : j1 * np - j1 * (j1 - 1) / 2 + (t - j1);
      d0 = fma(sp[i0], r[j], d0);
      d1 = fma(sp[i1], r[j1], d1);
    }
    if (j < np) d0 = fma(sp[j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j)], r[j], d0);
    x[size_t(f) * BS + t % BS] += d0 + d1;
  }
}

/// One multiplicative wave (pull form): every patch of the
/// wave recomputes its residual from A rows and the current x, solves with
/// its explicit inverse and updates its own DOFs; same-wave patches are
/// disjoint and uncoupled, so no atomics are needed.
template <int BS>
__global__ void k_gs_wave(Bsr A, Patches P, int w0, const double* __restrict__ b, double* __restrict__ x,
                          int transposed) {
  __shared__ double r[kMaxPatchF * BS];
  __shared__ int fac[kMaxPatchF];
  const int p = P.wave[w0 + blockIdx.x];
  const int nf = P.nf[p], np = nf * BS;
  if (threadIdx.x < kMaxPatchF) fac[threadIdx.x] = P.fac[p * kMaxPatchF + threadIdx.x];
  __syncthreads();
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    const int f = fac[t / BS], i = t % BS;
    double s = b[size_t(f) * BS + i];
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int c = __ldg(&A.cols[f * kSlots + sl]);
      if (c < 0) continue;
      const double2* blk = reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * BS + i) * BS);
      const double2* xc = reinterpret_cast<const double2*>(x + size_t(c) * BS);
#pragma unroll
      for (int j = 0; j < BS / 2; ++j) {
        const double2 a = __ldg(blk + j), xv = xc[j];
        s = fma(-a.x, xv.x, s);
        s = fma(-a.y, xv.y, s);
      }
    }
    r[t] = s;
  }
  __syncthreads();
  const double* inv = P.inv + P.off[p];
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    double d = 0.0;
    if (!transposed) {
      for (int j = 0; j < np; ++j) d = fma(__ldg(inv + size_t(j) * np + t), r[j], d);
    } else {
      const double* row = inv + size_t(t) * np;
      for (int j = 0; j < np; ++j) d = fma(__ldg(row + j), r[j], d);
    }
    x[size_t(fac[t / BS]) * BS + t % BS] += d;
  }
}

template <int BS>
__global__ void k_jacobi_patch(Patches P, int max_np, const double* __restrict__ rvec, double* __restrict__ dbuf) {
  __shared__ double r[kMaxPatchF * BS];
  __shared__ int fac[kMaxPatchF];
  const int p = blockIdx.x;
  const int nf = P.nf[p], np = nf * BS;
  if (threadIdx.x < kMaxPatchF) fac[threadIdx.x] = P.fac[p * kMaxPatchF + threadIdx.x];
  __syncthreads();
  for (int t = threadIdx.x; t < np; t += blockDim.x) r[t] = rvec[size_t(fac[t / BS]) * BS + t % BS];
  __syncthreads();
  const double* inv = P.inv + P.off[p];
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    double d = 0.0;
    if (P.packed) {
      const int ct = t * np - t * (t - 1) / 2 - t;
      for (int j = 0; j < np; ++j)
        d = fma(__ldg(inv + (j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j))), r[j], d);
    } else {
      for (int j = 0; j < np; ++j) d = fma(__ldg(inv + size_t(j) * np + t), r[j], d);
    }
    dbuf[size_t(p) * max_np + t] = d;
  }
}

__global__ void k_jacobi_combine(int nb, int bs, Patches P, int max_np, const double* __restrict__ dbuf,
                                 double damping, double* __restrict__ x) {
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t / bs), i = int(t % bs);
    double v = x[t];
    for (int q = 0; q < 2; ++q) {
      const int p = P.fpatch[f * 2 + q];
      if (p < 0) continue;
      int pos = 0;
      for (int s = 0; s < kMaxPatchF; ++s)
        if (P.fac[p * kMaxPatchF + s] == f) { pos = s; break; }
      v += damping * dbuf[size_t(p) * max_np + pos * bs + i];
    }
    x[t] = v;
  }
}

// ------------------------------------------------------------- transfers
/// y (+)= M v for a 2x2-block CSR, G lanes per block row (q strided by G,
/// fixed-order butterfly): PT rows hold ~25 blocks, P rows ~6, so one thread
/// per row would serialise that many dependent L2 round trips. The first kU
/// blocks of a lane issue all their loads together (restriction: level-4
/// pre-phase 77 -> 73 us at config 2).
template <int G, bool ACC, int kU>
__global__ void k_bcsr_group(BlockCsr M, const double* __restrict__ v, double* __restrict__ y,
                             double* __restrict__ zero_out = nullptr) {
  // warp-uniform grid stride: every lane of a warp runs the same trip count (shuffles)
  const int64_t total = int64_t(M.nrows) * G, stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); base < total; base += stride) {
  const int64_t gt = base + (threadIdx.x & 31);
  const int row = int(gt / G), lane = int(gt % G);
  const bool live = row < M.nrows;
  double s0 = 0.0, s1 = 0.0;
  if (live) {
    // the first kU blocks of the lane with all loads in flight together
    // (columns first, then values and the gathered v rows), the rest in a loop
    const int q0 = __ldg(&M.ptr[row]) + lane, q1 = __ldg(&M.ptr[row + 1]);
    int c[kU > 0 ? kU : 1];
#pragma unroll
    for (int u = 0; u < kU; ++u) c[u] = q0 + u * G < q1 ? __ldg(&M.col[q0 + u * G]) : -1;
    double2 a0[kU > 0 ? kU : 1], a1[kU > 0 ? kU : 1], w[kU > 0 ? kU : 1];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (c[u] >= 0) {
        const size_t q = size_t(q0 + u * G);
        a0[u] = __ldg(reinterpret_cast<const double2*>(M.val) + q * 2);
        a1[u] = __ldg(reinterpret_cast<const double2*>(M.val) + q * 2 + 1);
        w[u] = __ldg(reinterpret_cast<const double2*>(v) + c[u]);
      }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (c[u] >= 0) {
        s0 = fma(a0[u].x, w[u].x, fma(a0[u].y, w[u].y, s0));
        s1 = fma(a1[u].x, w[u].x, fma(a1[u].y, w[u].y, s1));
      }
    for (int q = q0 + kU * G; q < q1; q += G) {
      const int cq = __ldg(&M.col[q]);
      const double2 b0 = __ldg(reinterpret_cast<const double2*>(M.val) + size_t(q) * 2);
      const double2 b1 = __ldg(reinterpret_cast<const double2*>(M.val) + size_t(q) * 2 + 1);
      const double2 wq = __ldg(reinterpret_cast<const double2*>(v) + cq);
      s0 = fma(b0.x, wq.x, fma(b0.y, wq.y, s0));
      s1 = fma(b1.x, wq.x, fma(b1.y, wq.y, s1));
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o, G);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o, G);
  }
  if (live && lane == 0) {
    // restriction: the coarse level's pre-smoothing starts from x = 0, zeroed
    // here instead of by a separate fill launch
    if (zero_out) reinterpret_cast<double2*>(zero_out)[row] = make_double2(0.0, 0.0);
    double2* yr = reinterpret_cast<double2*>(y) + row;
    if (ACC) {
      const double2 o = *yr;
      *yr = make_double2(o.x + s0, o.y + s1);
    } else {
      *yr = make_double2(s0, s1);
    }
  }
  }
}

/// One thread per coarse element: gather A_TT and W_T = (A I_avg)_T of its
/// medial fine blocks, LU with partial pivoting (the host algorithm,
/// reference transfer.hpp:119-130), subtract the solution into P.
__global__ void k_corrected_prolongation(Bsr A, TransferDev T, double* __restrict__ Pval) {
  constexpr int kM = 2 * kTransferColMax;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < T.nelem; e += gridDim.x * blockDim.x) {
    const int nt = 2 * T.nmed[e];
    if (nt == 0) continue;
    const int nc = T.ncol[e], m = 2 * nc;
    const int* med = T.med + size_t(e) * 3;
    const int* cl = T.col + size_t(e) * kTransferColMax;
    double Att[36], Bm[6 * kM];
    for (int r = 0; r < nt; ++r) {
      const int rb = med[r / 2], rt = r % 2;
      for (int c = 0; c < nt; ++c) {
        const int cb = med[c / 2], ct = c % 2;
        double v = 0.0;
        for (int sl = 0; sl < kSlots; ++sl)
          if (A.cols[rb * kSlots + sl] == cb) v = A.val[((size_t(rb) * kSlots + sl) * 2 + rt) * 2 + ct];
        Att[r * nt + c] = v;
      }
      for (int j = 0; j < m; ++j) Bm[r * m + j] = 0.0;
      for (int sl = 0; sl < kSlots; ++sl) {
        const int jb = A.cols[rb * kSlots + sl];
        if (jb < 0) continue;
        for (int jt = 0; jt < 2; ++jt) {
          const double a = A.val[((size_t(rb) * kSlots + sl) * 2 + rt) * 2 + jt];
          if (a == 0.0) continue;
          for (int q = T.avg_ptr[jb]; q < T.avg_ptr[jb + 1]; ++q) {
            int j = 0;
            while (cl[j] != T.avg_col[q]) ++j;
            Bm[r * m + 2 * j] += a * T.avg_val[size_t(q) * 4 + jt * 2 + 0];
            Bm[r * m + 2 * j + 1] += a * T.avg_val[size_t(q) * 4 + jt * 2 + 1];
          }
        }
      }
    }
    for (int k = 0; k < nt; ++k) {
      int p = k;
      for (int i = k + 1; i < nt; ++i)
        if (fabs(Att[i * nt + k]) > fabs(Att[p * nt + k])) p = i;
      if (p != k) {
        for (int j = 0; j < nt; ++j) {
          const double t = Att[k * nt + j];
          Att[k * nt + j] = Att[p * nt + j];
          Att[p * nt + j] = t;
        }
        for (int j = 0; j < m; ++j) {
          const double t = Bm[k * m + j];
          Bm[k * m + j] = Bm[p * m + j];
          Bm[p * m + j] = t;
        }
      }
      const double d = Att[k * nt + k];
      for (int i = k + 1; i < nt; ++i) {
        const double l = Att[i * nt + k] / d;
        if (l == 0.0) continue;
        for (int j = k + 1; j < nt; ++j) Att[i * nt + j] -= l * Att[k * nt + j];
        for (int j = 0; j < m; ++j) Bm[i * m + j] -= l * Bm[k * m + j];
      }
    }
    for (int j = 0; j < m; ++j)
      for (int i = nt - 1; i >= 0; --i) {
        double sv = Bm[i * m + j];
        for (int l = i + 1; l < nt; ++l) sv -= Att[i * nt + l] * Bm[l * m + j];
        Bm[i * m + j] = sv / Att[i * nt + i];
      }
    for (int r = 0; r < nt; ++r)
      for (int j = 0; j < nc; ++j) {
        const int q = T.pos[(size_t(e) * 3 + r / 2) * kTransferColMax + j];
        Pval[size_t(q) * 4 + (r % 2) * 2 + 0] -= Bm[r * m + 2 * j];
        Pval[size_t(q) * 4 + (r % 2) * 2 + 1] -= Bm[r * m + 2 * j + 1];
      }
  }
}

__global__ void k_block_transpose_perm(int nnz, const int* __restrict__ perm, const double* __restrict__ Pval,
                                       double* __restrict__ PTval) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < nnz; d += gridDim.x * blockDim.x) {
    const double* v = Pval + size_t(perm[d]) * 4;
    PTval[size_t(d) * 4 + 0] = v[0];
    PTval[size_t(d) * 4 + 1] = v[2];
    PTval[size_t(d) * 4 + 2] = v[1];
    PTval[size_t(d) * 4 + 3] = v[3];
  }
}

/// x = Inv b for the dense coarse inverse (column-major) in ONE launch: CTA
/// (rb, chunk) forms the partial sums of rows [128 rb, 128 rb + 128) over the
/// columns of its chunk (all 32 column loads of a thread in flight at once,
/// L2 evict-last so the 17 MB inverse of a 1472-DOF coarse level stays
/// L2-resident across V-cycles), writes them to work[chunk][n], and the last
/// CTA of the row block to arrive (threadfence + counter, as CUDA's
/// threadFenceReduction sample) sums the partials in chunk order: the result
/// is independent of CTA scheduling. The counter resets itself, so captured
/// graphs replay it.
constexpr int kGemvChunk = 32;
__global__ void __launch_bounds__(128) k_gemv(int n, int chunks, const double* __restrict__ inv,
                                              const double* __restrict__ b, double* __restrict__ work,
                                              unsigned* __restrict__ counter, double* __restrict__ x) {
  __shared__ double sb[kGemvChunk];
  __shared__ bool last;
  const int chunk = blockIdx.y;
  const int j0 = chunk * kGemvChunk, nj = min(kGemvChunk, n - j0);
  if (threadIdx.x < nj) sb[threadIdx.x] = b[j0 + threadIdx.x];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const double* col = inv + size_t(j0) * n + i;
    double v[kGemvChunk];
#pragma unroll
    for (int u = 0; u < kGemvChunk; ++u) {
      v[u] = 0.0;
      if (u < nj)
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(v[u])
                     : "l"(col + size_t(u) * n), "l"(pol));
    }
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < kGemvChunk; ++u)
      if (u < nj) s[u & 7] = fma(v[u], sb[u], s[u & 7]);
    work[size_t(chunk) * n + i] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter + blockIdx.x, 1u) == unsigned(chunks - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (i < n) {
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += __ldcg(work + size_t(c) * n + i);
    x[i] = s;
  }
  if (threadIdx.x == 0) counter[blockIdx.x] = 0u;
}

// ---------------------------------------------- dense coarse inverse (setup)
/// Gauss-Jordan step k on aug = [A | I] (n x 2n row-major): pivot search
/// (largest |a_ik|, lowest index on ties), row swap, and copies of the pivot
/// row and column so the elimination kernel never reads what it writes.
__global__ void k_gj_pivot(int n, int k, double* __restrict__ aug, double* __restrict__ rowk,
                           double* __restrict__ colk, int* __restrict__ status) {
  __shared__ double bv[32];
  __shared__ int bi[32];
  const int w = 2 * n;
  double best = -1.0;
  int besti = k;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(aug[size_t(i) * w + k]);
    if (v > best) { best = v; besti = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
    if (ob > best || (ob == best && oi < besti)) { best = ob; besti = oi; }
  }
  if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = besti; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? bv[threadIdx.x] : -1.0;
    besti = threadIdx.x < nw ? bi[threadIdx.x] : n;
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
      if (ob > best || (ob == best && oi < besti)) { best = ob; besti = oi; }
    }
    if (threadIdx.x == 0) { bi[0] = besti; bv[0] = best; }
  }
  __syncthreads();
  const int p = bi[0];
  if (threadIdx.x == 0 && !(bv[0] > 0.0)) *status = 1;  // singular
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    const double a = aug[size_t(k) * w + j], b = aug[size_t(p) * w + j];
    aug[size_t(k) * w + j] = b;
    aug[size_t(p) * w + j] = a;
    rowk[j] = b;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) colk[i] = i == k ? 0.0 : aug[size_t(i) * w + k];
}

__global__ void k_gj_eliminate(int n, int k, double* __restrict__ aug, const double* __restrict__ rowk,
                               const double* __restrict__ colk) {
  const int w = 2 * n;
  const double inv = 1.0 / rowk[k];
  const int64_t tot = int64_t(n) * w;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / w), j = int(e % w);
    const double r = rowk[j] * inv;
    aug[e] = i == k ? r : aug[e] - colk[i] * r;
  }
}

/// Grid barrier of a cooperative launch: ctl[0] counts arrivals within the
/// launch (release atomic, acquire polls), ctl[1] exits; the last CTA out
/// resets both for the next launch.
__device__ __forceinline__ void gj_grid_sync(unsigned* ctl, unsigned i) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctl) : "memory");
    const unsigned target = (i + 1u) * gridDim.x;
    if (old + 1u != target) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctl) : "memory");
      } while (v < target);
    }
  }
  __syncthreads();
}

/// (value, row) candidate of a pivot search; ties go to the lowest row.
struct GjCand {
  double v;
  int i, pad;
};
__device__ __forceinline__ void gj_better(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}
/// block-wide argmax (256 threads); the result is valid in every thread
__device__ __forceinline__ void gj_block_argmax(double& bv, int& bi, double* sv, int* si) {
  for (int o = 16; o > 0; o >>= 1) gj_better(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  bv = sv[0];
  bi = si[0];
  for (int q = 1; q < int(blockDim.x >> 5); ++q) gj_better(bv, bi, sv[q], si[q]);
  __syncthreads();
}

constexpr int kGjMaxRows = 64;  // rows owned per CTA
constexpr int kGjBatch = 12;    // loads in flight per thread and row (2n <= 3072 in one batch)
/// All n Gauss-Jordan steps (partial pivoting) in one cooperative launch with
/// ONE grid barrier per step and no row swaps. CTA b owns the rows b, b + G,
/// ...; pivot rows are tracked, not swapped (inverse row k = right part of
/// pivot row p_k). Step k: every CTA reduces the per-CTA candidates of column
/// k (ties: lowest row) to the pivot p, reads the multipliers a_ik of its own
/// rows, and updates them over columns [k, 2n) as a_ij - a_ik (a_pj / a_pk)
/// (the left columns < k are already eliminated); then it publishes the
/// candidate of column k+1 among its unused rows. Row p is read by every CTA
/// during step k, so its owner normalises it (a_pj / a_pk) only at the start
/// of step k+1, where no other CTA reads it. Operations per entry are those of
/// the swapping formulation (k_gj_pivot + k_gj_eliminate); the only
/// difference is the tie-break order among exactly equal pivot candidates.
__global__ void __launch_bounds__(256) k_gj_implicit(int n, double* __restrict__ aug, GjCand* __restrict__ cand,
                                                     int* __restrict__ piv, int* __restrict__ status, unsigned* ctl) {
  extern __shared__ double srow[];  // [2n] scaled pivot row
  __shared__ double m[kGjMaxRows];
  __shared__ unsigned char used[kGjMaxRows];
  __shared__ double sv[32];
  __shared__ int si[32];
  const int w = 2 * n, G = int(gridDim.x), b = int(blockIdx.x);
  const int nown = (n - b + G - 1) / G;
  for (int r = threadIdx.x; r < kGjMaxRows; r += blockDim.x) used[r] = 0;
  __syncthreads();
  auto publish = [&](int col, int slot) {  // candidate of column col among the unused own rows
    double bv = -1.0;
    int bi = n;
    for (int r = threadIdx.x; r < nown; r += blockDim.x)
      if (!used[r]) {
        const int i = b + r * G;
        gj_better(bv, bi, fabs(__ldcg(aug + size_t(i) * w + col)), i);
      }
    gj_block_argmax(bv, bi, sv, si);
    if (threadIdx.x == 0) {
      __stcg(&cand[size_t(slot) * G + b].v, bv);
      __stcg(&cand[size_t(slot) * G + b].i, bi);
    }
  };
  publish(0, 0);
  unsigned bar = 0;
  gj_grid_sync(ctl, bar++);
  int prev = -1;
  double prev_inv = 0.0;
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int p = n;
    for (int q = threadIdx.x; q < G; q += blockDim.x) {
      const GjCand* c = cand + size_t(k & 1) * G + q;  // L2: written by other CTAs
      gj_better(bv, p, __ldcg(&c->v), __ldcg(&c->i));
    }
    gj_block_argmax(bv, p, sv, si);
    if (b == 0 && threadIdx.x == 0) {
      piv[k] = p < n ? p : 0;  // an all-NaN column leaves p = n: keep k_gj_extract_piv in bounds
      if (!(bv > 0.0)) *status = 1;  // singular
    }
    if (p >= n) p = 0;  // singular (flagged above): keep the addressing in bounds
    // deferred normalisation of the previous pivot row (k_gj_eliminate: rowk[j] * inv)
    if (prev >= 0 && prev % G == b) {
      double* row = aug + size_t(prev) * w;
      for (int j0 = k + threadIdx.x; j0 < w; j0 += kGjBatch * 256) {
        double v[kGjBatch];
#pragma unroll
        for (int u = 0; u < kGjBatch; ++u) v[u] = j0 + u * 256 < w ? __ldcg(row + j0 + u * 256) : 0.0;
#pragma unroll
        for (int u = 0; u < kGjBatch; ++u)
          if (j0 + u * 256 < w) __stcg(row + j0 + u * 256, v[u] * prev_inv);
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < nown; r += blockDim.x) m[r] = __ldcg(aug + size_t(b + r * G) * w + k);
    if (p % G == b && threadIdx.x == 0) used[p / G] = 1;
    __syncthreads();
    const double* R = aug + size_t(p) * w;
    const double inv = 1.0 / __ldcg(R + k);
    // the scaled pivot row a_pj / a_pk once into shared memory, then per own
    // row all of a thread's loads in flight before its stores (loads and
    // stores of aug may alias as far as the compiler knows: without the
    // batching every element would cost its own L2 round trip)
    for (int j0 = k + threadIdx.x; j0 < w; j0 += kGjBatch * 256) {
      double v[kGjBatch];
#pragma unroll
      for (int u = 0; u < kGjBatch; ++u) v[u] = j0 + u * 256 < w ? __ldcg(R + j0 + u * 256) : 0.0;
#pragma unroll
      for (int u = 0; u < kGjBatch; ++u)
        if (j0 + u * 256 < w) srow[j0 + u * 256 - k] = v[u] * inv;
    }
    __syncthreads();
    for (int r = 0; r < nown; ++r) {
      const int i = b + r * G;
      if (i == p) continue;
      const double mi = m[r];
      double* row = aug + size_t(i) * w;
      for (int j0 = k + threadIdx.x; j0 < w; j0 += kGjBatch * 256) {
        double v[kGjBatch];
#pragma unroll
        for (int u = 0; u < kGjBatch; ++u) v[u] = j0 + u * 256 < w ? __ldcg(row + j0 + u * 256) : 0.0;
#pragma unroll
        for (int u = 0; u < kGjBatch; ++u)
          if (j0 + u * 256 < w) __stcg(row + j0 + u * 256, v[u] - mi * srow[j0 + u * 256 - k]);
      }
    }
    __syncthreads();
    if (k + 1 < n) publish(k + 1, (k + 1) & 1);
    prev = p;
    prev_inv = inv;
    gj_grid_sync(ctl, bar++);
  }
  if (prev >= 0 && prev % G == b) {
    double* row = aug + size_t(prev) * w;
    for (int j = n + threadIdx.x; j < w; j += blockDim.x) __stcg(row + j, __ldcg(row + j) * prev_inv);
  }
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctl + 1) : "memory");
    if (old + 1u == gridDim.x) {
      ctl[0] = 0u;
      ctl[1] = 0u;
    }
  }
}

/// inverse row k = right part of pivot row piv[k] (column-major output)
__global__ void k_gj_extract_piv(int n, const double* __restrict__ aug, const int* __restrict__ piv,
                                 double* __restrict__ inv) {
  const int64_t tot = int64_t(n) * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / n), k = int(e % n);
    inv[e] = aug[size_t(piv[k]) * 2 * n + n + j];
  }
}

__global__ void k_gj_extract(int n, const double* __restrict__ aug, double* __restrict__ inv) {
  const int64_t tot = int64_t(n) * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / n), i = int(e % n);  // column-major output
    inv[e] = aug[size_t(i) * 2 * n + n + j];
  }
}

__global__ void k_gj_init(int n, const double* __restrict__ A, double* __restrict__ aug) {
  const int64_t tot = int64_t(n) * 2 * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / (2 * n)), j = int(e % (2 * n));
    aug[e] = j < n ? A[size_t(i) * n + j] : (j - n == i ? 1.0 : 0.0);
  }
}

// --------------------------------------------------------------- vectors
__global__ void k_fill(double* x, double v, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) x[t] = v;
}
__global__ void k_copy(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) y[t] = x[t];
}
__global__ void k_axpy(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    y[t] += a * x[t];
}
__global__ void k_sub(double* __restrict__ y, const double* __restrict__ a, const double* __restrict__ b, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    y[t] = a[t] - b[t];
}
__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, Reduce red, double* out) {
  double s = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    s = fma(a[t], b[t], s);
  finalize<false>(s, red, out);
}
/// Squared L2 norm of an RT velocity field (reference inc/assembly.hpp:487-501):
/// one thread per element, local coefficients from the compound flux part and
/// the interior part, sum over the volume nodes of w detJ |J v_hat c / detJ|^2.
template <int MaxRt>
__global__ void k_rt_norm2(RefT T, const ElemGeo* __restrict__ geo, int ne, const int* __restrict__ elem_facets,
                           const double* __restrict__ compound, const double* __restrict__ interior, Reduce red,
                           double* out) {
  double acc = 0.0;
  const int nfd = T.nfd, nrt = T.nrt;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const ElemGeo& g = geo[e];
    double c[MaxRt];
    for (int r = 0; r < nrt; ++r) {
      if (r < 3 * nfd) {
        const int le = r / nfd, i = r % nfd;
        const double f = ((i & 1) && g.rho[le] < 0) ? -g.fac[le] : g.fac[le];
        c[r] = f * compound[size_t(elem_facets[e * 3 + le]) * nfd + i];
      } else {
        c[r] = interior[size_t(e) * T.no + (r - 3 * nfd)];
      }
    }
    double s = 0.0;
    for (int q = 0; q < T.nq; ++q) {
      const double* vv = T.vval + size_t(q) * 2 * nrt;
      double h0 = 0.0, h1 = 0.0;
      for (int r = 0; r < nrt; ++r) {
        h0 = fma(vv[r], c[r], h0);
        h1 = fma(vv[nrt + r], c[r], h1);
      }
      const double v0 = (g.J[0] * h0 + g.J[1] * h1) / g.detJ, v1 = (g.J[2] * h0 + g.J[3] * h1) / g.detJ;
      s = fma(T.qw[q] * g.detJ, v0 * v0 + v1 * v1, s);
    }
    acc += s;
  }
  finalize<false>(acc, red, out);
}

__global__ void k_pcg_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ Ap, int64_t n, double* sc, int i_num, int i_den, Reduce red,
                             int i_rr) {
  // pAp <= 0: the reference returns before touching x and r (krylov.hpp:49-53);
  // the predicate is grid-uniform, so every block leaves and no reduction runs
  if (!(sc[i_den] > 0.0)) return;
  const double alpha = sc[i_num] / sc[i_den];
  double s = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    x[t] += alpha * p[t];
    const double rv = r[t] - alpha * Ap[t];
    r[t] = rv;
    s = fma(rv, rv, s);
  }
  finalize<false>(s, red, sc + i_rr);
}
// ---- device-resident PCG iteration (one CUDA-graph while loop per solve;
// reference krylov.hpp:30-73). Scalars live in sc[]: the loop slots below,
// the reduction results written by the vector kernels.
/// x += a p, r -= a Ap, r.r, then (last block) the iteration count and the
/// stop test (krylov.hpp:54-62; at the cap the reference still forms z = M r
/// and checks r.z once more), setting the branch and, when stopping, the
/// loop handle.
__global__ void k_pcg_loop_update(double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                                  const double* __restrict__ z, const double* __restrict__ Ap, int64_t n, int dir,
                                  double* sc, Reduce red, cudaGraphConditionalHandle h_loop) {
  if (sc[kScStatus] != kLoopRunning) return;  // stopped by r.z in this iteration
  if (!(sc[kScPAp] > 0.0)) {  // krylov.hpp:49-53: x and r untouched, not applicable
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc[kScStatus] = kLoopNaPAp;
      cudaGraphSetConditional(h_loop, 0u);
    }
    return;
  }
  const double alpha = sc[kScRZ] / sc[kScPAp];
  const double beta = dir ? sc[kScBeta] : 0.0;
  double s = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    double pt = p[t];
    if (dir) {  // p = z + beta p (krylov.hpp:69), as k_spmv_dir formed it
      pt = fma(beta, pt, z[t]);
      p[t] = pt;
    }
    x[t] += alpha * pt;
    const double rv = r[t] - alpha * Ap[t];
    r[t] = rv;
    s = fma(rv, rv, s);
  }
  finalize_then(s, red, sc + kScRR, [&](double rr) {
    sc[kScIt] += 1.0;
    double st = kLoopRunning;
    if (sqrt(rr) <= sc[kScTarget]) st = kLoopConverged;
    else if (sc[kScIt] >= sc[kScMaxIt]) st = kLoopLast;
    sc[kScStatus] = st;
    // the cap still forms z = M r and checks r.z once (k_pcg_loop_rz ends the loop there)
    cudaGraphSetConditional(h_loop, st == kLoopConverged ? 0u : 1u);
  });
}
/// r.z, then (last block) its positivity test (krylov.hpp:63-68) and
/// beta = rz_next / rz, rz = rz_next; the loop handle is cleared when the
/// iteration stops here
__global__ void k_pcg_loop_rz(const double* __restrict__ r, const double* __restrict__ z, int64_t n, double* sc,
                              Reduce red, cudaGraphConditionalHandle h_loop) {
  double s = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    s = fma(r[t], z[t], s);
  finalize_then(s, red, sc + kScRZn, [&](double rzn) {
    if (!(rzn > 0.0)) {
      sc[kScStatus] = kLoopNaRZ;
      cudaGraphSetConditional(h_loop, 0u);
    } else if (sc[kScStatus] == kLoopLast) {
      sc[kScStatus] = kLoopMaxIt;
      cudaGraphSetConditional(h_loop, 0u);
    } else {
      sc[kScBeta] = rzn / sc[kScRZ];
      sc[kScRZ] = rzn;
    }
  });
}

/// p = z + beta p while running (krylov.hpp:69)
__global__ void k_pcg_loop_direction(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                     const double* sc) {
  if (sc[kScStatus] != kLoopRunning) return;
  const double beta = sc[kScBeta];
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    p[t] = z[t] + beta * p[t];
}
/// last node of the loop body: iterate again while running
/// development probe: c -= 1; loop while c > 0
__global__ void k_loop_countdown(double* c, cudaGraphConditionalHandle h_loop) {
  c[0] -= 1.0;
  cudaGraphSetConditional(h_loop, c[0] > 0.0 ? 1u : 0u);
}
__global__ void k_loop_continue(const double* sc, cudaGraphConditionalHandle h_loop) {
  cudaGraphSetConditional(h_loop, sc[kScStatus] == kLoopRunning ? 1u : 0u);
}
__global__ void k_gm_init(double* sc, GmDev G, double target, double max_it, double cap) {
  sc[kScIt] = 0.0;
  sc[kScStatus] = kLoopRunning;
  sc[kScTarget] = target;
  sc[kScMaxIt] = max_it;
  G.st[kGmCap] = cap;
}
__global__ void k_pcg_loop_init(double* sc, double target, double max_it) {
  sc[kScIt] = 0.0;
  sc[kScStatus] = kLoopRunning;
  sc[kScTarget] = target;
  sc[kScMaxIt] = max_it;
}

// ---- device-resident GMRES (reference krylov.hpp:79-144): restart cycles
// and Arnoldi steps as nested graph loops; modified Gram-Schmidt one fused
// pass per basis vector; Givens rotations and the triangular solve in
// single-thread kernels on the device-side Hessenberg columns.
/// top of a cycle, after r = b - A x and r.r: true-residual test, g = (beta)
__global__ void k_gm_start(double* sc, GmDev G, cudaGraphConditionalHandle h_cyc,
                           cudaGraphConditionalHandle h_inner) {
  const double beta = sqrt(sc[kScRR]);
  if (beta <= sc[kScTarget]) {
    sc[kScStatus] = kLoopConverged;
    cudaGraphSetConditional(h_cyc, 0u);
    cudaGraphSetConditional(h_inner, 0u);
    return;
  }
  G.st[kGmBeta] = beta;
  G.st[kGmJ] = 0.0;
  G.st[kGmM] = 0.0;
  G.st[kGmStalled] = 0.0;
  G.g[0] = beta;
  cudaGraphSetConditional(h_cyc, 1u);
  cudaGraphSetConditional(h_inner, sc[kScIt] < sc[kScMaxIt] ? 1u : 0u);
}
/// V[0] = r / beta, also into the preconditioner's input u; arms the
/// Gram-Schmidt loop of column 0
__global__ void k_gm_v0(GmDev G, const double* r, double* u, int64_t n,  // r may alias u
                        cudaGraphConditionalHandle h_mgs) {
  const double beta = G.st[kGmBeta];
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const double v = r[t] / beta;
    G.V[t] = v;
    u[t] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    G.st[kGmI] = 0.0;
    cudaGraphSetConditional(h_mgs, 1u);
  }
}
// development timeline of the GMRES loop kernels (off unless gm_trace arms it):
// (kernel id, step, globaltimer) at the start of CTA 0
__device__ int d_gmt_on = 0;
__device__ unsigned d_gmt_n = 0;
__device__ long long d_gmt[3 * 8192];
__device__ long long d_gmt_end[8192];  // CTA 0's end time of that kernel
__device__ __forceinline__ long long gm_now() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int gm_stamp(int id, int step) {
  if (d_gmt_on && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t = gm_now();
    const unsigned k = atomicAdd(&d_gmt_n, 1u);
    if (k < 8192) {
      d_gmt[3 * k] = id;
      d_gmt[3 * k + 1] = step;
      d_gmt[3 * k + 2] = t;
      return int(k);
    }
  }
  return -1;
}
__device__ __forceinline__ void gm_stamp_end(int k) {
  if (k >= 0) d_gmt_end[k] = gm_now();
}

/// Sum of the previous kernel's per-CTA partials part[0..np), in the same
/// fixed order in every CTA (so every CTA holds the bitwise-same value). This
/// replaces the atomic-ticket last-CTA reduction on a dependent chain: the
/// kernel boundary is the only synchronisation, and the L2 reads overlap the
/// vector loads issued before the call.
__device__ double sum_partials(const double* __restrict__ part, int np) {
  __shared__ double total;
  double a = 0.0;
  for (int b = threadIdx.x; b < np; b += blockDim.x) a += __ldcg(part + b);
  a = block_reduce<false>(a);
  if (threadIdx.x == 0) total = a;
  __syncthreads();
  return total;
}

constexpr int kMgsU = 4;  // vector elements per thread per pass, loads issued together

/// MGS step i of column j (krylov.hpp:100-103), the axpy of step i-1 fused
/// with the dot of step i: w -= h(i-1) v(i-1); partial of w . v(i).
/// h(i-1) is the sum of step i-1's partials (G.part, parity i-1), taken by
/// every CTA; CTA 0 stores it into H. Eight steps per loop body (u = 0..7):
/// steps 0-3 read their base index from st[kGmI], steps 4-7 from st[kGmI2];
/// step 1 writes the second base and step 5 the first one for the next body,
/// so no kernel writes a slot that its own CTAs read.
__global__ void k_mgs(GmDev G, double* __restrict__ w, int64_t n, int u, cudaGraphConditionalHandle h_mgs) {
  const int base = int(G.st[u < 4 ? kGmI : kGmI2]);
  const int i = base + (u & 3), j = int(G.st[kGmJ]);
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int slot = gm_stamp(i > j ? 2 : 1, i);
  if (lead && (u & 3) == 1) G.st[u < 4 ? kGmI2 : kGmI] = double(base + 4);
  if (i > j) {  // past the column's last step: no-op
    if (lead) cudaGraphSetConditional(h_mgs, 0u);
    return;
  }
  const double* vi = G.V + int64_t(i) * G.ldv;
  const double* vp = G.V + int64_t(i > 0 ? i - 1 : 0) * G.ldv;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  double wv[kMgsU], pv[kMgsU], iv[kMgsU];
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int q = 0; q < kMgsU; ++q) {
      const int64_t t = t0 + q * stride;
      if (t < n) {
        wv[q] = w[t];
        iv[q] = vi[t];
        pv[q] = i > 0 ? vp[t] : 0.0;
      }
    }
  };
  int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  load(t0);  // in flight while the previous step's partials are summed
  double hp = 0.0;
  if (i > 0) {
    hp = sum_partials(G.part + ((i - 1) & 1) * kRedBlocks, gridDim.x);
    if (lead) G.H[int64_t(j) * G.ldh + i - 1] = hp;
  }
  double s = 0.0;
  for (;;) {
#pragma unroll
    for (int q = 0; q < kMgsU; ++q) {
      const int64_t t = t0 + q * stride;
      if (t < n) {
        if (i > 0) {
          wv[q] = fma(-hp, pv[q], wv[q]);
          w[t] = wv[q];
        }
        s = fma(wv[q], iv[q], s);
      }
    }
    t0 += kMgsU * stride;
    if (t0 >= n) break;
    load(t0);
  }
  s = block_reduce<false>(s);
  if (threadIdx.x == 0) G.part[(i & 1) * kRedBlocks + blockIdx.x] = s;
  if (lead) cudaGraphSetConditional(h_mgs, i + 1 <= j ? 1u : 0u);
  gm_stamp_end(slot);
}
/// last axpy of column j (h(j) from step j's partials) and the partials of |w|^2
__global__ void k_mgs_tail(GmDev G, double* __restrict__ w, int64_t n) {
  const int j = int(G.st[kGmJ]);
  gm_stamp(3, j);
  const double* vp = G.V + int64_t(j) * G.ldv;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  double wv[kMgsU], pv[kMgsU];
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int q = 0; q < kMgsU; ++q) {
      const int64_t t = t0 + q * stride;
      if (t < n) {
        wv[q] = w[t];
        pv[q] = vp[t];
      }
    }
  };
  int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  load(t0);
  const double hp = sum_partials(G.part + (j & 1) * kRedBlocks, gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) G.H[int64_t(j) * G.ldh + j] = hp;
  double s = 0.0;
  for (;;) {
#pragma unroll
    for (int q = 0; q < kMgsU; ++q) {
      const int64_t t = t0 + q * stride;
      if (t < n) {
        const double wt = fma(-hp, pv[q], wv[q]);
        w[t] = wt;
        s = fma(wt, wt, s);
      }
    }
    t0 += kMgsU * stride;
    if (t0 >= n) break;
    load(t0);
  }
  s = block_reduce<false>(s);
  if (threadIdx.x == 0) G.part[((j + 1) & 1) * kRedBlocks + blockIdx.x] = s;
}
/// Givens rotations of column j and the residual estimate (krylov.hpp:107-118);
/// decides whether the Arnoldi loop continues. One thread.
__device__ void gm_givens_step(double* sc, GmDev G, cudaGraphConditionalHandle h_inner,
                               cudaGraphConditionalHandle h_mgs) {
  const int j = int(G.st[kGmJ]);
  double* h = G.H + int64_t(j) * G.ldh;
  for (int i = 0; i < j; ++i) {
    const double t = G.cs[i] * h[i] + G.sn[i] * h[i + 1];
    h[i + 1] = -G.sn[i] * h[i] + G.cs[i] * h[i + 1];
    h[i] = t;
  }
  const double rho = hypot(h[j], h[j + 1]);
  G.cs[j] = h[j] / rho;
  G.sn[j] = h[j + 1] / rho;
  h[j] = rho;
  h[j + 1] = 0.0;
  G.g[j + 1] = -G.sn[j] * G.g[j];
  G.g[j] *= G.cs[j];
  sc[kScIt] += 1.0;
  G.st[kGmM] = double(j + 1);
  const bool happy = G.st[kGmHappy] != 0.0;
  const double gn = fabs(G.g[j + 1]);
  const bool exit = gn <= sc[kScTarget] || happy;
  if (exit) G.st[kGmStalled] = (happy && gn > sc[kScTarget]) ? 1.0 : 0.0;
  const bool more = !exit && sc[kScIt] < sc[kScMaxIt] && double(j + 1) < G.st[kGmCap];
  if (more) {
    G.st[kGmJ] = double(j + 1);
    G.st[kGmI] = 0.0;  // arm the Gram-Schmidt loop of the next column
    cudaGraphSetConditional(h_mgs, 1u);
  }
  cudaGraphSetConditional(h_inner, more ? 1u : 0u);
}
/// h(j+1) = |w| (the tail's partials, summed in every CTA), the breakdown
/// test, V[j+1] = w / h(j+1), also into the preconditioner's input u (the next
/// column's z = M v); the last CTA then stores h(j+1) and runs the Givens
/// step. After a breakdown the loop ends and u is overwritten by gm_update.
__global__ void k_gm_newv(double* sc, GmDev G, const double* __restrict__ w, double* __restrict__ u, int64_t n,
                          int np, unsigned* counter, cudaGraphConditionalHandle h_inner,
                          cudaGraphConditionalHandle h_mgs) {
  const int j = int(G.st[kGmJ]);
  gm_stamp(4, j);
  const double h = sqrt(sum_partials(G.part + ((j + 1) & 1) * kRedBlocks, np));
  const bool happy = h <= 1e-14 * G.st[kGmBeta];  // krylov.hpp:104-106
  if (!happy) {
    double* v = G.V + int64_t(j + 1) * G.ldv;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
      const double x = w[t] / h;
      v[t] = x;
      u[t] = x;
    }
  }
  __shared__ bool last;
  __syncthreads();  // every thread has read st[J] before the last CTA's Givens step changes it
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    *counter = 0u;
    G.st[kGmHn] = h * h;
    G.H[int64_t(j) * G.ldh + j + 1] = h;
    G.st[kGmHappy] = happy ? 1.0 : 0.0;
    gm_givens_step(sc, G, h_inner, h_mgs);
  }
}
/// back substitution H y = g over the m columns (krylov.hpp:126-131)
__global__ void k_gm_solve(GmDev G) {
  const int m = int(G.st[kGmM]);
  for (int i = m - 1; i >= 0; --i) {
    double s = G.g[i];
    for (int l = i + 1; l < m; ++l) s -= G.H[int64_t(l) * G.ldh + i] * G.y[l];
    G.y[i] = s / G.H[int64_t(i) * G.ldh + i];
  }
}
/// u = sum_i y(i) V[i] (krylov.hpp:132-133), in ascending i per entry
__global__ void k_gm_combine(GmDev G, double* __restrict__ u, int64_t n) {
  const int m = int(G.st[kGmM]);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    double a = 0.0;
    for (int i = 0; i < m; ++i) a += G.y[i] * G.V[int64_t(i) * G.ldv + t];
    u[t] = a;
  }
}
/// after x += M u and r.r: the cycle's exit (krylov.hpp:134-143)
__global__ void k_gm_end(double* sc, GmDev G) {
  if (sqrt(sc[kScRR]) <= sc[kScTarget]) sc[kScStatus] = kLoopConverged;
  else if (G.st[kGmStalled] != 0.0 || sc[kScIt] >= sc[kScMaxIt]) sc[kScStatus] = kLoopMaxIt;
}

__global__ void k_pcg_direction(double* __restrict__ p, const double* __restrict__ z, int64_t n, const double* sc,
                                int i_new, int i_old) {
  const double beta = sc[i_new] / sc[i_old];
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    p[t] = z[t] + beta * p[t];
}
__global__ void k_scal_axpby(double* __restrict__ y, const double* __restrict__ x, int64_t n, const double* sc, int ia,
                             double fa, double fb) {
  const double a = (ia >= 0 ? sc[ia] : 1.0) * fa;
  // fb == 0 overwrites y without reading it (fresh GMRES basis vectors hold garbage, 0 * NaN = NaN)
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
    y[t] = fb == 0.0 ? a * x[t] : a * x[t] + fb * y[t];
}

__global__ void k_to_blocks(int nb, int nfd, const double* __restrict__ ref, double* __restrict__ blk) {
  const int bs = 2 * nfd;
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = t / bs;
    const int ii = int(t % bs), i = ii >> 1, tg = ii & 1;
    blk[t] = ref[(tg ? int64_t(nb) * nfd : 0) + f * nfd + i];
  }
}
/// k_to_blocks that also zeroes `zero` (the cycle's x) in the same pass
__global__ void k_to_blocks_zero(int nb, int nfd, const double* __restrict__ ref, double* __restrict__ blk,
                                 double* __restrict__ zero) {
  // the first pre-smoothing wave (programmatic dependent launch) may start
  // its record copies now; it reads b and x only after this grid completes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int bs = 2 * nfd;
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = t / bs;
    const int ii = int(t % bs), i = ii >> 1, tg = ii & 1;
    blk[t] = ref[(tg ? int64_t(nb) * nfd : 0) + f * nfd + i];
    zero[t] = 0.0;
  }
}
/// (in the drop-in graph launched with programmatic dependent launch after the
/// last post-smoothing wave: its CTAs come up during that wave's tail)
__global__ void k_to_reference(int nb, int nfd, const double* __restrict__ blk, double* __restrict__ ref) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int bs = 2 * nfd;
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = t / bs;
    const int ii = int(t % bs), i = ii >> 1, tg = ii & 1;
    ref[(tg ? int64_t(nb) * nfd : 0) + f * nfd + i] = blk[t];
  }
}

// ------------------------------------------------------------------ uzawa
__global__ void k_uzawa_rhs(int nb, int bs, const double* __restrict__ rhs0, const int* __restrict__ row_elems,
                            const ElemGeo* __restrict__ geo, const double* __restrict__ p, double* __restrict__ rhs) {
  const int64_t n = int64_t(nb) * bs;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t / bs), ii = int(t % bs);
    double add = 0.0;
    if (ii == 0)
      for (int c = 0; c < 2; ++c) {
        const int e = row_elems[f * 4 + 2 * c];
        if (e < 0) continue;
        const int la = row_elems[f * 4 + 2 * c + 1];
        const ElemGeo& g = geo[e];
        add += (g.fac[la] < 0 ? -2.0 : 2.0) * g.ds[la] * p[e];
      }
    rhs[t] = rhs0[t] + add;
  }
}

__global__ void k_uzawa_div(int ne, int bs, const int* __restrict__ elem_facets, const int* __restrict__ facet_block,
                            const double* __restrict__ g_fac, const double* __restrict__ u,
                            const ElemGeo* __restrict__ geo, double* __restrict__ div) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const ElemGeo& g = geo[e];
    int fs[3] = {elem_facets[e * 3], elem_facets[e * 3 + 1], elem_facets[e * 3 + 2]};
    int ord[3] = {0, 1, 2};  // ascending facet id (column order of Bdiv)
    if (fs[ord[0]] > fs[ord[1]]) { int t = ord[0]; ord[0] = ord[1]; ord[1] = t; }
    if (fs[ord[1]] > fs[ord[2]]) { int t = ord[1]; ord[1] = ord[2]; ord[2] = t; }
    if (fs[ord[0]] > fs[ord[1]]) { int t = ord[0]; ord[0] = ord[1]; ord[1] = t; }
    double s = 0.0;
    for (int q = 0; q < 3; ++q) {
      const int le = ord[q], f = fs[le], blk = facet_block[f];
      const double val = blk >= 0 ? u[size_t(blk) * bs] : g_fac[size_t(f) * bs];
      s += (g.fac[le] < 0 ? -2.0 : 2.0) * g.ds[le] * val;
    }
    div[e] = s / (0.5 * g.detJ);
  }
}

__global__ void k_uzawa_p1(int ne, const double* __restrict__ div, const ElemGeo* __restrict__ geo, double inv_eps,
                           double* __restrict__ p, Reduce red, double* out) {
  double s = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const double pv = p[e] - inv_eps * div[e];
    p[e] = pv;
    s = fma(0.5 * geo[e].detJ, pv, s);
  }
  finalize<false>(s, red, out);
}
__global__ void k_area_sum(int ne, const ElemGeo* __restrict__ geo, Reduce red, double* out) {
  double s = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) s += 0.5 * geo[e].detJ;
  finalize<false>(s, red, out);
}
__global__ void k_uzawa_p2(int ne, double* __restrict__ p, const double* sc, int i_s, int i_a) {
  const double m = sc[i_s] / sc[i_a];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) p[e] -= m;
}
__global__ void k_absmax(int ne, const double* __restrict__ v, Reduce red, double* out) {
  double s = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) s = fmax(s, fabs(v[e]));
  finalize<true>(s, red, out);
}

template <typename F>
void by_bs(int bs, F&& f) {
  switch (bs) {
    case 2: f(std::integral_constant<int, 2>()); break;
    case 4: f(std::integral_constant<int, 4>()); break;
    case 6: f(std::integral_constant<int, 6>()); break;
    case 8: f(std::integral_constant<int, 8>()); break;
    case 10: f(std::integral_constant<int, 10>()); break;  // k = 4..6: beyond the reference's k <= 3
    case 12: f(std::integral_constant<int, 12>()); break;
    case 14: f(std::integral_constant<int, 14>()); break;
    default: throw std::runtime_error("unsupported block size");
  }
}

}  // namespace

// ============================================================ launchers
void condense(const RefT& T, const ElemGeo* geo, int ne, CondenseParams prm, const double* load, int load_stride,
              double* out, cudaStream_t s, const double* wind, const double* mass_field) {
  if (ne == 0) return;
  const int nz = T.no + T.ns - 1;
  const size_t smem = sizeof(double) * condense_scratch(T.ns, T.nv, T.nc, nz, T.nrt, T.nq, T.nqe);
  static bool attr = false;
  if (!attr) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_condense);  // opt-in maximum minus the kernel's static shared memory
    cudaFuncSetAttribute(k_condense, cudaFuncAttributeMaxDynamicSharedMemorySize, int(227 * 1024 - fa.sharedSizeBytes));
    attr = true;
  }
  k_condense<<<ne, 128, smem, s>>>(T, geo, prm, load, load_stride, out, T.nc * T.nc + T.nc, wind, mass_field);
  HPMG_LAUNCH_CHECK();
}

void recover(const RefT& T, const ElemGeo* geo, int ne, CondenseParams prm, const double* load, int load_stride,
             const int* elem_facets, long long nflux, const double* compound, double* interior, double* pres,
             double* grad, cudaStream_t s, const double* wind, const double* mass_field) {
  if (ne == 0) return;
  const int nz = T.no + T.ns - 1;
  const size_t smem =
      sizeof(double) * (condense_scratch(T.ns, T.nv, T.nc, nz, T.nrt, T.nq, T.nqe) + T.nc + nz + 1 + 4 * T.ns);
  static bool attr = false;
  if (!attr) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_recover);  // opt-in maximum minus the kernel's static shared memory
    cudaFuncSetAttribute(k_recover, cudaFuncAttributeMaxDynamicSharedMemorySize, int(227 * 1024 - fa.sharedSizeBytes));
    attr = true;
  }
  k_recover<<<ne, 128, smem, s>>>(T, geo, prm, load, load_stride, elem_facets, nflux, compound, interior, pres, grad,
                                  wind, mass_field);
  HPMG_LAUNCH_CHECK();
}

void assemble_bsr(const Bsr& A, int nfd, const double* acr, int stride, int nc, const int* gath, const ElemGeo* geo,
                  double inv_eps, cudaStream_t s) {
  const int64_t n = int64_t(A.nb) * kSlots * A.bs * A.bs;
  k_assemble_bsr<<<grid_for(n, 256), 256, 0, s>>>(A, nfd, acr, stride, nc, gath, geo, inv_eps);
  HPMG_LAUNCH_CHECK();
}

void transpose_bsr(const Bsr& A, const int* tslot, Bsr& AT, cudaStream_t s) {
  const int64_t n = int64_t(A.nb) * kSlots * A.bs * A.bs;
  k_transpose_bsr<<<grid_for(n, 256), 256, 0, s>>>(A, tslot, AT);
  HPMG_LAUNCH_CHECK();
}

void assemble_rhs(int nb, int bs, int nfd, const int* row_elems, const int* block_facet, const int* elem_facets,
                  const char* facet_dirichlet, const double* g_fac, const double* acr, int stride, int nc,
                  const ElemGeo* geo, double inv_eps, double* rhs, cudaStream_t s) {
  k_assemble_rhs<<<grid_for(int64_t(nb) * bs, 256), 256, 0, s>>>(nb, bs, nfd, row_elems, block_facet, elem_facets,
                                                                 facet_dirichlet, g_fac, acr, stride, nc, geo, inv_eps,
                                                                 rhs);
  HPMG_LAUNCH_CHECK();
}

void spmv(const Bsr& A, const double* x, const double* b, double* y, int minus, const Reduce* red, double* dot_out,
          cudaStream_t s) {
  const int64_t n = int64_t(A.nb) * A.bs;
  by_bs(A.bs, [&](auto BS) {
    if (red) {
      static const int grid = resident_grid(k_spmv<BS>);
      k_spmv<BS><<<grid, 256, 0, s>>>(A, x, b, y, minus, 1, *red, dot_out);
    } else {
      k_spmv<BS><<<grid_for(n, 256), 256, 0, s>>>(A, x, b, y, minus, 0, Reduce{}, nullptr);
    }
  });
  HPMG_LAUNCH_CHECK();
}

void extract_mode0(const Bsr& A, Bsr& A0, cudaStream_t s) {
  by_bs(A.bs, [&](auto BS) {
    k_extract_mode0<BS><<<grid_for(int64_t(A.nb) * kSlots * 2 * BS, 256), 256, 0, s>>>(A, A0);
  });
  HPMG_LAUNCH_CHECK();
}
void inject_residual(const Bsr& A, const double* x, const double* b, double* r0, cudaStream_t s, double* x0_zero) {
  by_bs(A.bs, [&](auto BS) {
    k_inject_residual<BS><<<grid_for(int64_t(A.nb) * 2, 256), 256, 0, s>>>(A, x, b, r0, x0_zero);
  });
  HPMG_LAUNCH_CHECK();
}

void embed_add(int nb, int bs, const double* e, double* x, cudaStream_t s) {
  k_embed_add<<<grid_for(int64_t(nb) * 2, 256), 256, 0, s>>>(nb, bs, e, x);
  HPMG_LAUNCH_CHECK();
}

void patch_inverse(const Bsr& A, const Patches& P, int max_nf, cudaStream_t s) {
  if (P.n == 0) return;
  by_bs(A.bs, [&](auto BS) {
    const int np = max_nf * BS;
    const size_t smem = sizeof(double) * size_t(np) * 2 * np;
    cudaFuncSetAttribute(k_patch_inverse<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // one thread per augmented column, row groups up to ~256 threads
    const int W = 2 * np, rg = std::max(1, std::min(np, 256 / W));
    k_patch_inverse<BS><<<P.n, rg * W, smem, s>>>(A, P, rg);
  });
  HPMG_LAUNCH_CHECK();
}

void gs_wave(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int transposed_inv,
             int max_nf, cudaStream_t s, const void* prefetch, size_t prefetch_len) {
  if (w1 <= w0) return;
  const char* prefetch_ptr = static_cast<const char*>(prefetch);
  unsigned prefetch_bytes = unsigned(std::min<size_t>(prefetch_len, 0xFFFFFFF0u)) & ~15u;
  if (P.packed) {
    if (transposed_inv) throw std::runtime_error("packed (symmetric) inverses have no transposed sweep");
    by_bs(A.bs, [&](auto BS) {
      constexpr int TP = BS == 2 ? 16 : (BS == 4 ? 32 : 64);
      constexpr int NP6 = 6 * BS;                               // interior vertex: 6 facets
      constexpr int U = (NP6 * (NP6 + 1) / 2 + TP - 1) / TP;   // staged loads per thread
      const int npmax = max_nf * BS;
      if (npmax > TP) throw std::runtime_error("vertex patch too large for the sweep kernel");
      const int ppc = 128 / TP, pk = npmax * (npmax + 1) / 2;
      const size_t smem = sizeof(double) * (size_t(ppc) * pk + 128);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_gs_wave_sym<BS, TP, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
      const int nblk = (w1 - w0 + ppc - 1) / ppc;
      k_gs_wave_sym<BS, TP, U><<<nblk, 128, smem, s>>>(A, P, w0, w1, pk, b, x, prefetch_ptr, prefetch_bytes);
    });
  } else {
    by_bs(A.bs, [&](auto BS) {
      const int np = max_nf * BS;
      const int threads = ((np + 31) / 32) * 32;
      k_gs_wave<BS><<<w1 - w0, threads, 0, s>>>(A, P, w0, b, x, transposed_inv);
    });
  }
  HPMG_LAUNCH_CHECK();
}

void jacobi_patch(const Bsr& A, const Patches& P, const double* r, double* d, int max_nf, cudaStream_t s) {
  by_bs(A.bs, [&](auto BS) {
    const int np = max_nf * BS;
    k_jacobi_patch<BS><<<P.n, ((np + 31) / 32) * 32, 0, s>>>(P, np, r, d);
  });
  HPMG_LAUNCH_CHECK();
}

void jacobi_combine(int nb, int bs, const Patches& P, const double* d, int max_nf, double damping, double* x,
                    cudaStream_t s) {
  k_jacobi_combine<<<grid_for(int64_t(nb) * bs, 256), 256, 0, s>>>(nb, bs, P, max_nf * bs, d, damping, x);
  HPMG_LAUNCH_CHECK();
}

namespace {
/// base[q] = the averaging block of P's block q (zero where only the
/// correction has a block): a sorted merge of the two column lists per row
__global__ void k_prolong_base(int nrows, const int* __restrict__ pptr, const int* __restrict__ pcol,
                               const int* __restrict__ aptr, const int* __restrict__ acol,
                               const double* __restrict__ aval, double* __restrict__ base) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    int j = aptr[r];
    const int je = aptr[r + 1];
    for (int q = pptr[r]; q < pptr[r + 1]; ++q) {
      const int c = pcol[q];
      while (j < je && acol[j] < c) ++j;
      const bool hit = j < je && acol[j] == c;
#pragma unroll
      for (int t = 0; t < 4; ++t) base[size_t(q) * 4 + t] = hit ? aval[size_t(j) * 4 + t] : 0.0;
    }
  }
}
}  // namespace

void prolong_base(const BlockCsr& P, const TransferDev& T, cudaStream_t s) {
  if (P.nrows > 0)
    k_prolong_base<<<grid_for(P.nrows, 256), 256, 0, s>>>(P.nrows, P.ptr, P.col, T.avg_ptr, T.avg_col, T.avg_val,
                                                             T.base);
  HPMG_LAUNCH_CHECK();
}

void corrected_prolongation(const Bsr& A, const TransferDev& T, BlockCsr& P, BlockCsr& PT, cudaStream_t s) {
  cudaError_t err = cudaMemcpyAsync(P.val, T.base, sizeof(double) * 4 * size_t(T.nnz), cudaMemcpyDeviceToDevice, s);
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA copy: ") + cudaGetErrorString(err));
  if (T.nelem > 0) k_corrected_prolongation<<<grid_for(T.nelem, 128), 128, 0, s>>>(A, T, P.val);
  HPMG_LAUNCH_CHECK();
  if (T.nnz > 0) k_block_transpose_perm<<<grid_for(T.nnz, 256), 256, 0, s>>>(T.nnz, T.tperm, P.val, PT.val);
  HPMG_LAUNCH_CHECK();
}

void prolong_add(const BlockCsr& P, const double* e, double* x, cudaStream_t s) {
  constexpr int G = 4;
  // P rows hold ~6 blocks (1-2 per lane): the plain loop; unrolling it measured slower
  k_bcsr_group<G, true, 0><<<grid_for(int64_t(P.nrows) * G, 256), 256, 0, s>>>(P, e, x);
  HPMG_LAUNCH_CHECK();
}

void restrict_(const BlockCsr& PT, const double* r, double* rc, cudaStream_t s, double* xc_zero) {
  constexpr int G = 8;
  // PT rows hold ~25 blocks (3-4 per lane): four in flight at once
  k_bcsr_group<G, false, 4><<<grid_for(int64_t(PT.nrows) * G, 256), 256, 0, s>>>(PT, r, rc, xc_zero);
  HPMG_LAUNCH_CHECK();
}

// partials [chunks][n] then the per-row-block arrival counters (zero-initialised by the caller)
size_t dense_gemv_work(int n) { return size_t(n) * ((n + kGemvChunk - 1) / kGemvChunk) + (n + 127) / 128 + 1; }

void dense_gemv(int n, const double* inv, const double* b, double* x, double* work, cudaStream_t s) {
  const int chunks = (n + kGemvChunk - 1) / kGemvChunk;
  unsigned* counter = reinterpret_cast<unsigned*>(work + size_t(n) * chunks);
  k_gemv<<<dim3((n + 127) / 128, chunks), 128, 0, s>>>(n, chunks, inv, b, work, counter, x);
  HPMG_LAUNCH_CHECK();
}

namespace {
__global__ void k_bsr_to_dense(Bsr A, double* __restrict__ D) {
  const int n = A.nb * 2;
  const int64_t tot = int64_t(A.nb) * kSlots * 4;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = e >> 2;  // block (row, slot)
    const int r = int(q / kSlots), ij = int(e & 3), i = ij >> 1, j = ij & 1;
    const int c = A.cols[q];
    if (c >= 0) D[int64_t(2 * r + i) * n + 2 * c + j] = A.val[e];
  }
}
}  // namespace

void bsr_to_dense(const Bsr& A, double* D, cudaStream_t s) {
  if (A.bs != 2) throw std::runtime_error("bsr_to_dense: lowest-order (bs = 2) operators only");
  const int n = A.nb * 2;
  cudaMemsetAsync(D, 0, sizeof(double) * size_t(n) * n, s);
  k_bsr_to_dense<<<grid_for(int64_t(A.nb) * kSlots * 4, 256), 256, 0, s>>>(A, D);
  HPMG_LAUNCH_CHECK();
}

void dense_invert_alloc(int n, DenseInvertWork& W) {
  if (W.n == n) return;
  dense_invert_free(W);
  W.n = n;
  auto need = [](cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error("CUDA allocation failed (dense_invert)");
  };
  need(cudaMalloc(&W.aug, sizeof(double) * size_t(n) * 2 * n));
  need(cudaMalloc(&W.rowk, sizeof(double) * 2 * n));
  need(cudaMalloc(&W.colk, sizeof(double) * n));
  need(cudaMalloc(&W.status, sizeof(int)));
  // one cooperative launch for all steps when the grid can be co-resident
  int per_sm = 0, dev = 0, sms = 0;
  cudaFuncSetAttribute(k_gj_implicit, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gj_implicit, 256, sizeof(double) * 2 * size_t(n));
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // two CTAs per SM: enough for the row updates, few candidates to reduce per step
  W.grid = int(std::min<int64_t>(std::min(per_sm, 2) * int64_t(sms), n));
  W.coop = per_sm > 0 && int64_t(W.grid) * kGjMaxRows >= n && 2 * size_t(n) * sizeof(double) <= 200 * 1024 &&
           cudaMalloc(&W.ctl, 2 * sizeof(unsigned)) == cudaSuccess &&
           cudaMalloc(&W.cand, sizeof(GjCand) * 2 * size_t(W.grid)) == cudaSuccess &&
           cudaMalloc(&W.piv, sizeof(int) * size_t(n)) == cudaSuccess;
  cudaGetLastError();
}

void dense_invert_free(DenseInvertWork& W) {
  for (void* p : {(void*)W.aug, (void*)W.rowk, (void*)W.colk, (void*)W.status, (void*)W.ctl, W.cand, (void*)W.piv})
    if (p) cudaFree(p);
  W = DenseInvertWork{};
}

void dense_invert_async(int n, const double* A_rowmajor, double* inv_colmajor, DenseInvertWork& W, cudaStream_t s) {
  if (W.n != n) throw std::runtime_error("dense_invert: workspace not allocated for this size");
  cudaMemsetAsync(W.status, 0, sizeof(int), s);
  const int64_t tot = int64_t(n) * 2 * n;
  k_gj_init<<<grid_for(tot, 256), 256, 0, s>>>(n, A_rowmajor, W.aug);
  bool coop = W.coop;
  if (coop) {
    cudaMemsetAsync(W.ctl, 0, 2 * sizeof(unsigned), s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(W.grid));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = sizeof(double) * 2 * size_t(n);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, k_gj_implicit, n, W.aug, static_cast<GjCand*>(W.cand), W.piv,
                                             W.status, W.ctl);
    coop = le == cudaSuccess;
    if (!coop) cudaGetLastError();
    if (std::getenv("HPMG_SETUP_TRACE"))
      std::fprintf(stderr, "[setup] coarse GJ: n %d, cooperative %d (%s), grid %u\n", n, int(coop),
                   cudaGetErrorString(le), cfg.gridDim.x);
  }
  if (coop) {
    k_gj_extract_piv<<<grid_for(int64_t(n) * n, 256), 256, 0, s>>>(n, W.aug, W.piv, inv_colmajor);
  } else {
    for (int k = 0; k < n; ++k) {
      k_gj_pivot<<<1, 1024, 0, s>>>(n, k, W.aug, W.rowk, W.colk, W.status);
      k_gj_eliminate<<<grid_for(tot, 256), 256, 0, s>>>(n, k, W.aug, W.rowk, W.colk);
    }
    k_gj_extract<<<grid_for(int64_t(n) * n, 256), 256, 0, s>>>(n, W.aug, inv_colmajor);
  }
  HPMG_LAUNCH_CHECK();
}

void dense_invert_check(const DenseInvertWork& W, cudaStream_t s) {
  int hs = 0;
  cudaMemcpyAsync(&hs, W.status, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (hs) throw std::runtime_error("singular coarse operator");
}

void dense_invert(int n, const double* A_rowmajor, double* inv_colmajor, cudaStream_t s) {
  DenseInvertWork W;
  struct Free {
    DenseInvertWork& w;
    ~Free() { dense_invert_free(w); }
  } release{W};
  dense_invert_alloc(n, W);
  dense_invert_async(n, A_rowmajor, inv_colmajor, W, s);
  dense_invert_check(W, s);
}

void fill(double* x, double v, int64_t n, cudaStream_t s) {
  k_fill<<<grid_for(n, 256), 256, 0, s>>>(x, v, n);
  HPMG_LAUNCH_CHECK();
}
void copy(double* y, const double* x, int64_t n, cudaStream_t s) {
  k_copy<<<grid_for(n, 256), 256, 0, s>>>(y, x, n);
  HPMG_LAUNCH_CHECK();
}
void axpy(double* y, double a, const double* x, int64_t n, cudaStream_t s) {
  k_axpy<<<grid_for(n, 256), 256, 0, s>>>(y, a, x, n);
  HPMG_LAUNCH_CHECK();
}
void sub(double* y, const double* a, const double* b, int64_t n, cudaStream_t s) {
  k_sub<<<grid_for(n, 256), 256, 0, s>>>(y, a, b, n);
  HPMG_LAUNCH_CHECK();
}
void rt_norm2(const RefT& T, const ElemGeo* geo, int ne, const int* elem_facets, const double* compound,
              const double* interior, const Reduce& red, double* out, cudaStream_t s) {
  if (T.nrt > kMaxRt) throw std::runtime_error("RT space too large for rt_norm2");
  if (T.nrt <= 24)
    k_rt_norm2<24><<<kRedBlocks, 256, 0, s>>>(T, geo, ne, elem_facets, compound, interior, red, out);
  else
    k_rt_norm2<kMaxRt><<<kRedBlocks, 256, 0, s>>>(T, geo, ne, elem_facets, compound, interior, red, out);
  HPMG_LAUNCH_CHECK();
}
void dot(const double* a, const double* b, int64_t n, const Reduce& red, double* out, cudaStream_t s) {
  k_dot<<<kRedBlocks, 256, 0, s>>>(a, b, n, red, out);
  HPMG_LAUNCH_CHECK();
}
void pcg_update(double* x, double* r, const double* p, const double* Ap, int64_t n, double* sc, int i_num, int i_den,
                const Reduce& red, int i_rr, cudaStream_t s) {
  k_pcg_update<<<kRedBlocks, 256, 0, s>>>(x, r, p, Ap, n, sc, i_num, i_den, red, i_rr);
  HPMG_LAUNCH_CHECK();
}
void gm_init(double* sc, const GmDev& G, double target, double max_it, int cap, cudaStream_t s) {
  k_gm_init<<<1, 1, 0, s>>>(sc, G, target, max_it, double(cap));
  HPMG_LAUNCH_CHECK();
}
void gm_start(double* sc, const GmDev& G, cudaGraphConditionalHandle h_cyc, cudaGraphConditionalHandle h_inner,
              cudaStream_t s) {
  k_gm_start<<<1, 1, 0, s>>>(sc, G, h_cyc, h_inner);
  HPMG_LAUNCH_CHECK();
}
void gm_v0(const GmDev& G, const double* r, double* u, int64_t n, cudaGraphConditionalHandle h_mgs, cudaStream_t s) {
  k_gm_v0<<<grid_for(n, 256), 256, 0, s>>>(G, r, u, n, h_mgs);
  HPMG_LAUNCH_CHECK();
}
void gm_trace(int arm, long long* out) {
  const unsigned zero = 0;
  if (arm) cudaMemcpyToSymbol(d_gmt_n, &zero, sizeof(unsigned));
  cudaMemcpyToSymbol(d_gmt_on, &arm, sizeof(int));
  if (out) {
    unsigned k = 0;
    cudaMemcpyFromSymbol(&k, d_gmt_n, sizeof(unsigned));
    k = k < 8192 ? k : 8192;
    out[0] = k;
    cudaMemcpyFromSymbol(out + 1, d_gmt, sizeof(long long) * 3 * k);
    cudaMemcpyFromSymbol(out + 1 + 3 * 8192, d_gmt_end, sizeof(long long) * k);
  }
}
constexpr int kMgsGrid = kRedBlocks;  // the MGS kernels' grid = their partial count
void mgs_step(const GmDev& G, double* w, int64_t n, int u, cudaGraphConditionalHandle h_mgs, cudaStream_t s) {
  k_mgs<<<kMgsGrid, 256, 0, s>>>(G, w, n, u, h_mgs);
  HPMG_LAUNCH_CHECK();
}
void mgs_tail(const GmDev& G, double* w, int64_t n, cudaStream_t s) {
  k_mgs_tail<<<kMgsGrid, 256, 0, s>>>(G, w, n);
  HPMG_LAUNCH_CHECK();
}
void gm_arnoldi_close(double* sc, const GmDev& G, const double* w, double* u, int64_t n, const Reduce& red,
                      cudaGraphConditionalHandle h_inner, cudaGraphConditionalHandle h_mgs, cudaStream_t s) {
  static const int grid = resident_grid(k_gm_newv);
  k_gm_newv<<<grid, 256, 0, s>>>(sc, G, w, u, n, kMgsGrid, red.counter, h_inner, h_mgs);
  HPMG_LAUNCH_CHECK();
}
void gm_update(const GmDev& G, double* u, int64_t n, cudaStream_t s) {
  k_gm_solve<<<1, 1, 0, s>>>(G);
  HPMG_LAUNCH_CHECK();
  k_gm_combine<<<grid_for(n, 256), 256, 0, s>>>(G, u, n);
  HPMG_LAUNCH_CHECK();
}
void gm_end(double* sc, const GmDev& G, cudaStream_t s) {
  k_gm_end<<<1, 1, 0, s>>>(sc, G);
  HPMG_LAUNCH_CHECK();
}
void pcg_loop_update(double* x, double* r, double* p, const double* z, const double* Ap, int64_t n, int dir,
                     double* sc, const Reduce& red, cudaGraphConditionalHandle h_loop, cudaStream_t s) {
  k_pcg_loop_update<<<kRedBlocks, 256, 0, s>>>(x, r, p, z, Ap, n, dir, sc, red, h_loop);
  HPMG_LAUNCH_CHECK();
}
void pcg_spmv_dir(const Bsr& A, const double* p, const double* z, double* Ap, int dir, double* sc, const Reduce& red,
                  cudaStream_t s) {
  by_bs(A.bs, [&](auto BS) {
    static const int grid = resident_grid(k_spmv_dir<BS>);
    k_spmv_dir<BS><<<grid, 256, 0, s>>>(A, p, z, Ap, dir, sc, red, sc + kScPAp);
  });
  HPMG_LAUNCH_CHECK();
}
void pcg_loop_rz(const double* r, const double* z, int64_t n, double* sc, const Reduce& red,
                 cudaGraphConditionalHandle h_loop, cudaStream_t s) {
  k_pcg_loop_rz<<<kRedBlocks, 256, 0, s>>>(r, z, n, sc, red, h_loop);
  HPMG_LAUNCH_CHECK();
}
void pcg_loop_direction(double* p, const double* z, int64_t n, const double* sc, cudaStream_t s) {
  k_pcg_loop_direction<<<grid_for(n, 256), 256, 0, s>>>(p, z, n, sc);
  HPMG_LAUNCH_CHECK();
}
void loop_countdown(double* c, cudaGraphConditionalHandle h_loop, cudaStream_t s) {
  k_loop_countdown<<<1, 1, 0, s>>>(c, h_loop);
  HPMG_LAUNCH_CHECK();
}
void loop_continue(const double* sc, cudaGraphConditionalHandle h_loop, cudaStream_t s) {
  k_loop_continue<<<1, 1, 0, s>>>(sc, h_loop);
  HPMG_LAUNCH_CHECK();
}
void pcg_loop_init(double* sc, double target, double max_it, cudaStream_t s) {
  k_pcg_loop_init<<<1, 1, 0, s>>>(sc, target, max_it);
  HPMG_LAUNCH_CHECK();
}
void pcg_direction(double* p, const double* z, int64_t n, double* sc, int i_new, int i_old, cudaStream_t s) {
  k_pcg_direction<<<grid_for(n, 256), 256, 0, s>>>(p, z, n, sc, i_new, i_old);
  HPMG_LAUNCH_CHECK();
}
void scal_axpby(double* y, const double* x, int64_t n, const double* sc, int ia, double fa, double fb, cudaStream_t s) {
  k_scal_axpby<<<grid_for(n, 256), 256, 0, s>>>(y, x, n, sc, ia, fa, fb);
  HPMG_LAUNCH_CHECK();
}
void to_blocks(int nb, int nfd, const double* ref, double* blk, cudaStream_t s) {
  k_to_blocks<<<grid_for(int64_t(nb) * 2 * nfd, 256), 256, 0, s>>>(nb, nfd, ref, blk);
  HPMG_LAUNCH_CHECK();
}
void to_blocks_zero(int nb, int nfd, const double* ref, double* blk, double* zero, cudaStream_t s) {
  k_to_blocks_zero<<<grid_for(int64_t(nb) * 2 * nfd, 256), 256, 0, s>>>(nb, nfd, ref, blk, zero);
  HPMG_LAUNCH_CHECK();
}
void set_io_nodes(cudaGraphExec_t ge, cudaGraphNode_t in_node, cudaGraphNode_t out_node, int nb, int nfd,
                  const double* ref_in, double* blk_in, double* zero, const double* blk_out, double* ref_out) {
  const int grid = grid_for(int64_t(nb) * 2 * nfd, 256);
  {
    void* args[] = {&nb, &nfd, &ref_in, &blk_in, &zero};
    cudaKernelNodeParams p = {};
    p.func = reinterpret_cast<void*>(k_to_blocks_zero);
    p.gridDim = dim3(grid);
    p.blockDim = dim3(256);
    p.kernelParams = args;
    const cudaError_t e = cudaGraphExecKernelNodeSetParams(ge, in_node, &p);
    if (e != cudaSuccess) throw std::runtime_error(std::string("io graph input node: ") + cudaGetErrorString(e));
  }
  {
    void* args[] = {&nb, &nfd, &blk_out, &ref_out};
    cudaKernelNodeParams p = {};
    p.func = reinterpret_cast<void*>(k_to_reference);
    p.gridDim = dim3(grid);
    p.blockDim = dim3(256);
    p.kernelParams = args;
    const cudaError_t e = cudaGraphExecKernelNodeSetParams(ge, out_node, &p);
    if (e != cudaSuccess) throw std::runtime_error(std::string("io graph output node: ") + cudaGetErrorString(e));
  }
}
void to_reference(int nb, int nfd, const double* blk, double* ref, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid_for(int64_t(nb) * 2 * nfd, 256)));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_to_reference, nb, nfd, blk, ref);
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (to_reference): ") + cudaGetErrorString(e));
  HPMG_LAUNCH_CHECK();
}
void uzawa_rhs(int nb, int bs, const double* rhs0, const int* row_elems, const ElemGeo* geo, const double* p,
               double* rhs, cudaStream_t s) {
  k_uzawa_rhs<<<grid_for(int64_t(nb) * bs, 256), 256, 0, s>>>(nb, bs, rhs0, row_elems, geo, p, rhs);
  HPMG_LAUNCH_CHECK();
}
void uzawa_div(int ne, int bs, const int* elem_facets, const int* facet_block, const double* g_fac, const double* u,
               const ElemGeo* geo, double* div, cudaStream_t s) {
  k_uzawa_div<<<grid_for(ne, 256), 256, 0, s>>>(ne, bs, elem_facets, facet_block, g_fac, u, geo, div);
  HPMG_LAUNCH_CHECK();
}
void uzawa_pressure(int ne, const double* div, const ElemGeo* geo, double inv_eps, double* p, int enclosed,
                    const Reduce& red, double* sc, int i_s, int i_a, int i_max, cudaStream_t s) {
  k_uzawa_p1<<<kRedBlocks, 256, 0, s>>>(ne, div, geo, inv_eps, p, red, sc + i_s);
  if (enclosed) {
    k_area_sum<<<kRedBlocks, 256, 0, s>>>(ne, geo, red, sc + i_a);
    k_uzawa_p2<<<grid_for(ne, 256), 256, 0, s>>>(ne, p, sc, i_s, i_a);
  }
  k_absmax<<<kRedBlocks, 256, 0, s>>>(ne, div, red, sc + i_max);
  HPMG_LAUNCH_CHECK();
}

}  // namespace dev
}  // namespace hpmg
