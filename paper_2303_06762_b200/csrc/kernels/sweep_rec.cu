// Patch-record multiplicative sweep (symmetric operators): the dominant
// kernel of the hp-MG V-cycle (reference
// inc/smoother.hpp:53-67, 83-94).
//
// Every vertex patch owns one fixed-stride record in HBM, built once at setup:
//   [ patch inverse S_p (packed lower triangle by columns, or full)
//   | A_pe: per patch facet the <= 2 blocks coupling it to facets outside the
//     patch (facet (v,w) of the star of v couples to (v,a), (v,b) inside and
//     to the far edges (w,a), (w,b) outside)
//   | int32 meta: nf, facet ids, the external block columns ]
// and the sweep sets x_p = S_p (b_p - A_pe x_e): with S_p A_pp = I this is the
// reference update x_p += S_p (b - A x)_p without ever reading A_pp, which
// cuts the A bytes per sweep from 10 to 4 blocks per facet (each facet sits in
// two patches). A CTA needs no dependent index loads: one elected thread
// issues a single TMA bulk copy (cp.async.bulk, L2 evict-first so the
// streamed records do not evict x and b) of the records of its patch group,
// addressed by the patch id alone, onto an mbarrier. The threads then gather
// the external x blocks (the only dependent round, L2-resident), form the
// right-hand side from shared memory and apply the inverse.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

namespace {

__device__ __forceinline__ unsigned su32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(su32(bar))
      : "memory");
}
/// one TMA bulk copy global -> shared with an L2 evict-first policy
__device__ __forceinline__ void tma_stream(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}

/// Records of G consecutive patches per CTA, TP threads per patch.
template <int BS, int TP, int G>
__global__ void __launch_bounds__(G* TP) k_sweep_rec(PatchRecords R, int p0, int p1, const double* __restrict__ b,
                                                     double* __restrict__ x) {
  constexpr int kRow = kExt * BS * BS;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* srec = reinterpret_cast<double*>(smraw);  // G * stride
  double* sx = srec + size_t(G) * R.stride;          // G * max_nf * kExt * BS
  double* r = sx + G * R.max_nf * kExt * BS;         // G * TP
  __shared__ unsigned long long bar;
  const int lp = threadIdx.x / TP, t = threadIdx.x % TP;
  const int q0 = p0 + blockIdx.x * G;
  const int ng = min(G, p1 - q0);
  if (threadIdx.x == 0) {
    bar_init(&bar);
    tma_stream(srec, R.rec + size_t(q0) * R.stride, unsigned(ng) * unsigned(R.stride) * 8u, &bar);
  }
  // Programmatic dependent launch: the records do not depend on the previous
  // wave, so the copy above may overlap its tail; x and b may not be touched
  // before the previous grid has completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  bar_wait(&bar);
  const double* rec = srec + size_t(lp) * R.stride;
  const int* meta = reinterpret_cast<const int*>(rec + R.meta_off);
  const int nf = lp < ng ? meta[0] : 0, np = nf * BS;
  const int* fac = meta + 1;
  const int* ecol = meta + 1 + R.max_nf;
  double* xs = sx + lp * R.max_nf * kExt * BS;
  for (int e = t; e < nf * kExt * BS; e += TP) {
    const int c = ecol[e / BS];
    xs[e] = c >= 0 ? x[size_t(c) * BS + e % BS] : 0.0;
  }
  double bv = 0.0;
  if (t < np) bv = b[size_t(fac[t / BS]) * BS + t % BS];
  __syncthreads();
  if (t < np) {
    const int lf = t / BS, i = t % BS;
    const double* arow = rec + R.a_off + lf * kRow + i * BS;
    const double* xr = xs + lf * kExt * BS;
    double a0 = bv, a1 = 0.0;
#pragma unroll
    for (int sl = 0; sl < kExt; ++sl)
#pragma unroll
      for (int jj = 0; jj < BS; jj += 2) {
        const int j0 = (jj + i) % BS, j1 = (jj + 1 + i) % BS;  // rotated: rows of a block hit distinct banks
        a0 = fma(-arow[sl * BS * BS + j0], xr[sl * BS + j0], a0);
        a1 = fma(-arow[sl * BS * BS + j1], xr[sl * BS + j1], a1);
      }
    r[threadIdx.x] = a0 + a1;
  }
  __syncthreads();
  if (t < np) {
    const double* S = rec;  // packed lower triangle by columns
    const double* rr = r + lp * TP;
    const int ct = t * np - t * (t - 1) / 2 - t;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int j = 0;
    for (; j + 3 < np; j += 4) {
      double s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ju = j + u;
        s4[u] = S[ju >= t ? ct + ju : ju * np - ju * (ju - 1) / 2 + (t - ju)];
      }
      d0 = fma(s4[0], rr[j], d0);
      d1 = fma(s4[1], rr[j + 1], d1);
      d2 = fma(s4[2], rr[j + 2], d2);
      d3 = fma(s4[3], rr[j + 3], d3);
    }
    for (; j < np; ++j) d0 = fma(S[j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j)], rr[j], d0);
    x[size_t(fac[t / BS]) * BS + t % BS] = (d0 + d1) + (d2 + d3);
  }
}

/// Builds the records from the packed inverses and the ELL operator.
__global__ void k_build_records(Bsr A, Patches P, PatchRecords R, int bs) {
  const int p = blockIdx.x;
  double* rec = R.rec + size_t(p) * R.stride;
  const int nf = P.nf[p], np = nf * bs;
  const int pk = np * (np + 1) / 2;
  const double* inv = P.inv + P.off[p];
  if (R.full) {  // unpack the symmetric triangle: (r, c) at c*np + r
    for (int k = threadIdx.x; k < R.a_off; k += blockDim.x) {
      double v = 0.0;
      if (k < np * np) {
        const int c = k / np, r = k % np, lo = r > c ? c : r, hi = r > c ? r : c;
        v = inv[lo * np - lo * (lo - 1) / 2 + (hi - lo)];
      }
      rec[k] = v;
    }
  } else {
    for (int k = threadIdx.x; k < R.a_off; k += blockDim.x) rec[k] = k < pk ? inv[k] : 0.0;
  }
  // external blocks: slots whose column is a facet outside the patch, in slot order
  const int* pf = P.fac + p * kMaxPatchF;
  const int blk = bs * bs;
  int* meta = reinterpret_cast<int*>(rec + R.meta_off);
  for (int k = threadIdx.x; k < R.max_nf * kExt * blk; k += blockDim.x) rec[R.a_off + k] = 0.0;
  if (threadIdx.x == 0) meta[0] = nf;
  for (int k = threadIdx.x; k < R.max_nf; k += blockDim.x) meta[1 + k] = k < nf ? pf[k] : -1;
  for (int k = threadIdx.x; k < R.max_nf * kExt; k += blockDim.x) meta[1 + R.max_nf + k] = -1;
  __syncthreads();
  for (int lf = threadIdx.x; lf < nf; lf += blockDim.x) {
    const int f = pf[lf];
    int ne = 0;
    for (int sl = 0; sl < kSlots; ++sl) {
      const int c = A.cols[f * kSlots + sl];
      if (c < 0) continue;
      bool inside = false;
      for (int q = 0; q < nf; ++q) inside |= pf[q] == c;
      if (inside) continue;
      if (ne == kExt) {  // cannot happen on a triangle mesh: flag the record
        meta[0] = -1;
        break;
      }
      meta[1 + R.max_nf + lf * kExt + ne] = c;
      for (int e = 0; e < blk; ++e)
        rec[R.a_off + (lf * kExt + ne) * blk + e] = A.val[(size_t(f) * kSlots + sl) * blk + e];
      ++ne;
    }
  }
}

template <int BS>
struct RecCfg;
template <>
struct RecCfg<2> {
  static constexpr int TP = 16, G = 8;
};
template <>
struct RecCfg<4> {
  static constexpr int TP = 32, G = 2;
};
template <>
struct RecCfg<6> {
  static constexpr int TP = 64, G = 1;
};
template <>
struct RecCfg<8> {
  static constexpr int TP = 64, G = 1;
};

template <int BS>
void launch_rec(const PatchRecords& R, int w0, int w1, const double* b, double* x, cudaStream_t s) {
  constexpr int TP = RecCfg<BS>::TP, G = RecCfg<BS>::G;
  if (R.max_nf * BS > TP) throw std::runtime_error("vertex patch too large for the record sweep");
  const size_t smem = sizeof(double) * (size_t(G) * R.stride + size_t(G) * R.max_nf * kExt * BS + G * TP);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_rec<BS, TP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((w1 - w0 + G - 1) / G);
  cfg.blockDim = dim3(G * TP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  cudaError_t err = cudaLaunchKernelEx(&cfg, k_sweep_rec<BS, TP, G>, R, w0, w1, b, x);
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (sweep_rec): ") + cudaGetErrorString(err));
}

}  // namespace

PatchRecords record_layout(int bs, int max_nf, bool full) {
  PatchRecords R;
  R.bs = bs;
  R.max_nf = max_nf;
  R.full = full ? 1 : 0;
  const int npmax = max_nf * bs;
  R.a_off = full ? ((npmax * npmax + 1) & ~1) : (((npmax * (npmax + 1) / 2) + 1) & ~1);
  R.meta_off = R.a_off + max_nf * kExt * bs * bs;
  const int meta_ints = 1 + max_nf + max_nf * kExt;
  R.stride = (R.meta_off + (meta_ints + 1) / 2 + 1) & ~1;  // even => 16-byte aligned records
  return R;
}

void build_records(const Bsr& A, const Patches& P, PatchRecords& R, cudaStream_t s) {
  if (P.n == 0) return;
  k_build_records<<<P.n, 128, 0, s>>>(A, P, R, R.bs);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (build_records): ") + cudaGetErrorString(err));
}

void gs_wave_rec(const PatchRecords& R, int w0, int w1, const double* b, double* x, cudaStream_t s) {
  if (w1 <= w0) return;
  switch (R.bs) {
    case 2: launch_rec<2>(R, w0, w1, b, x, s); break;
    case 4: launch_rec<4>(R, w0, w1, b, x, s); break;
    case 6: launch_rec<6>(R, w0, w1, b, x, s); break;
    case 8: launch_rec<8>(R, w0, w1, b, x, s); break;
    default: throw std::runtime_error("unsupported block size");
  }
}

}  // namespace dev
}  // namespace hpmg
