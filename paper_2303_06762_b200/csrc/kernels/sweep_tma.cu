// TMA-fed multiplicative wave sweep (symmetric operators), the dominant
// kernel of the V-cycle (reference
// inc/smoother.hpp:53-67, 83-94).
//
// Per patch the sweep streams its packed symmetric inverse (np(np+1)/2
// doubles) and the A rows of its facets (nf x 5 blocks x bs^2 doubles); both
// are contiguous in HBM, so one elected thread moves them into shared memory
// with cp.async.bulk (TMA bulk copies) that complete on an mbarrier. Each CTA
// is persistent over its share of the wave and keeps kStages groups of
// patches in flight: while the threads compute group k (residual from the
// staged A rows and the current x, then d = S r from the staged triangle),
// the copies for groups k+1 .. k+kStages-1 are already landing. Same-wave
// patches share no DOF and no coupling (plan.hpp), so the CTAs never
// synchronise with each other inside a wave.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

namespace {

constexpr int kStages = 3;

__device__ __forceinline__ unsigned su32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
}

struct Meta {
  int nf;
  int fac[kMaxPatchF];
  long long off;
};

/// G patches per group, TP threads per patch; stage = [inverses | A rows].
template <int BS, int TP, int G>
__global__ void __launch_bounds__(G* TP) k_sweep_tma(Bsr A, Patches P, int p0, int p1, int ngroups, int gpc,
                                                     int inv_stage, int max_nf, const double* __restrict__ b,
                                                     double* __restrict__ x) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int kRow = kSlots * BS * BS;  // doubles of one facet's A row block
  const int arow_stage = G * max_nf * kRow;
  const int stage_d = inv_stage + arow_stage;
  double* stage_base = reinterpret_cast<double*>(smraw);
  double* r = stage_base + size_t(kStages) * stage_d;                    // G*TP
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(r + G * TP);  // kStages
  Meta* meta = reinterpret_cast<Meta*>(bar + kStages);                   // gpc*G

  const int lp = threadIdx.x / TP, t = threadIdx.x % TP;
  // groups of this CTA: g = blockIdx.x + k * gridDim.x, k < my_groups
  const int my_groups = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int e = threadIdx.x; e < my_groups * G; e += blockDim.x) {
    const int k = e / G, q = e % G;
    const int p = p0 + (blockIdx.x + k * gridDim.x) * G + q;
    Meta m;
    m.nf = 0;
    m.off = 0;
    if (p < p1) {
      m.nf = P.nf[p];
      m.off = P.off[p];
#pragma unroll
      for (int i = 0; i < kMaxPatchF; ++i) m.fac[i] = P.fac[p * kMaxPatchF + i];
    }
    meta[e] = m;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int k) {  // thread 0 only: copies of group k into stage k % kStages
    const int s = k % kStages;
    double* inv_dst = stage_base + size_t(s) * stage_d;
    double* a_dst = inv_dst + inv_stage;
    const Meta* mg = meta + k * G;
    int last = 0;
    for (int q = 0; q < G; ++q)
      if (mg[q].nf) last = q;
    const long long o0 = mg[0].off;
    const int npl = mg[last].nf * BS;
    const long long o1 = mg[last].off + ((npl * (npl + 1) / 2 + 1) & ~1);
    unsigned bytes = unsigned(o1 - o0) * 8u;
    for (int q = 0; q < G; ++q) bytes += unsigned(mg[q].nf) * kRow * 8u;
    mbar_expect_tx(&bar[s], bytes);
    tma_bulk_g2s(inv_dst, P.inv + o0, unsigned(o1 - o0) * 8u, &bar[s]);
    for (int q = 0; q < G; ++q)
      for (int i = 0; i < mg[q].nf; ++i)
        tma_bulk_g2s(a_dst + (q * max_nf + i) * kRow, A.val + size_t(mg[q].fac[i]) * kRow, kRow * 8u, &bar[s]);
  };

  if (threadIdx.x == 0)
    for (int k = 0; k < kStages - 1 && k < my_groups; ++k) issue(k);

  for (int k = 0; k < my_groups; ++k) {
    if (threadIdx.x == 0 && k + kStages - 1 < my_groups) {
      // the stage being refilled was released by the __syncthreads() closing k-1
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + kStages - 1);
    }
    const int s = k % kStages;
    mbar_wait(&bar[s], unsigned((k / kStages) & 1));
    const Meta& m = meta[k * G + lp];
    const int np = m.nf * BS;
    const double* sinv = stage_base + size_t(s) * stage_d + (m.off - meta[k * G].off);
    const double* sa = stage_base + size_t(s) * stage_d + inv_stage + lp * max_nf * kRow;
    int g = 0;
    if (t < np) {
      const int lf = t / BS, i = t % BS, f = m.fac[lf];
      g = f * BS + i;
      double acc = b[g];
      const double* arow = sa + lf * kRow + i * BS;  // slot sl block row i at sl*BS*BS
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int c = __ldg(&A.cols[f * kSlots + sl]);
        if (c < 0) continue;
        const double2* xc = reinterpret_cast<const double2*>(x + size_t(c) * BS);
        const double2* av = reinterpret_cast<const double2*>(arow + sl * BS * BS);
#pragma unroll
        for (int j = 0; j < BS / 2; ++j) {
          const double2 a = av[j], xv = xc[j];
          acc = fma(-a.x, xv.x, acc);
          acc = fma(-a.y, xv.y, acc);
        }
      }
      r[threadIdx.x] = acc;
    }
    __syncthreads();
    if (t < np) {
      const int ct = t * np - t * (t - 1) / 2 - t;
      const double* rr = r + lp * TP;
      double d0 = 0.0, d1 = 0.0;
      int j = 0;
      for (; j + 1 < np; j += 2) {
        const int j1 = j + 1;
        const int i0 = j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j);
        const int i1 = j1 >= t ? ct + j1 : j1 * np - j1 * (j1 - 1) / 2 + (t - j1);
        d0 = fma(sinv[i0], rr[j], d0);
        d1 = fma(sinv[i1], rr[j1], d1);
      }
      if (j < np) d0 = fma(sinv[j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j)], rr[j], d0);
      x[g] += d0 + d1;
    }
    __syncthreads();
  }
}

/// Non-persistent variant: one CTA per group of G patches. Thread 0 starts a
/// single TMA bulk copy of the group's contiguous packed inverses into shared
/// memory; meanwhile every thread pulls its residual row from the A rows
/// (vector loads straight into registers) and the current x; the GEMV waits
/// on the mbarrier. No register staging => high occupancy.
template <int BS, int TP, int G>
__global__ void __launch_bounds__(G* TP) k_sweep_tma1(Bsr A, Patches P, int p0, int p1, int pk,
                                                      const double* __restrict__ b, double* __restrict__ x) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* sinv = reinterpret_cast<double*>(smraw);  // G * pk
  double* r = sinv + G * pk;                          // G * TP
  __shared__ unsigned long long bar;
  const int lp = threadIdx.x / TP, t = threadIdx.x % TP;
  const int q0 = p0 + blockIdx.x * G;
  const int p = q0 + lp;
  const long long base_off = P.off[q0];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int ql = min(q0 + G, p1) - 1;
    const int npl = P.nf[ql] * BS;
    const long long o1 = P.off[ql] + ((npl * (npl + 1) / 2 + 1) & ~1);
    const unsigned bytes = unsigned(o1 - base_off) * 8u;
    mbar_expect_tx(&bar, bytes);
    tma_bulk_g2s(sinv, P.inv + base_off, bytes, &bar);
  }
  int np = 0, g = 0;
  long long loff = 0;
  if (p < p1) {
    np = P.nf[p] * BS;
    loff = P.off[p] - base_off;
    if (t < np) {
      const int f = P.fac[p * kMaxPatchF + t / BS], i = t % BS;
      g = f * BS + i;
      double acc = b[g];
      int cc[kSlots];
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) cc[sl] = __ldg(&A.cols[f * kSlots + sl]);
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        if (cc[sl] < 0) continue;
        const double2* av = reinterpret_cast<const double2*>(A.val + (size_t(f * kSlots + sl) * BS + i) * BS);
        const double2* xc = reinterpret_cast<const double2*>(x + size_t(cc[sl]) * BS);
#pragma unroll
        for (int j = 0; j < BS / 2; ++j) {
          const double2 a = __ldg(av + j), xv = xc[j];
          acc = fma(-a.x, xv.x, acc);
          acc = fma(-a.y, xv.y, acc);
        }
      }
      r[threadIdx.x] = acc;
    }
  }
  __syncthreads();  // r complete; also orders the mbarrier init before the waits
  mbar_wait(&bar, 0u);
  if (t < np) {
    const double* S = sinv + loff;
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
    x[g] += (d0 + d1) + (d2 + d3);
  }
}

/// Fully staged variant for the order-k head (bs >= 4), one patch per CTA:
/// thread 0 issues TMA bulk copies of the packed inverse and of the nf A row
/// blocks (row stride padded by 2 doubles to spread shared-memory banks);
/// the threads gather the x blocks of every (facet, slot) column of the patch
/// into shared memory; the residual then runs entirely from shared memory
/// with a rotated column index (row i starts at column i), which keeps the
/// 8 rows of a block on distinct banks.
template <int BS, int TP>
__global__ void __launch_bounds__(TP) k_sweep_tma2(Bsr A, Patches P, int p0, int pk, int max_nf,
                                                   const double* __restrict__ b, double* __restrict__ x) {
  constexpr int kRow = kSlots * BS * BS, kRowPad = kRow + 2;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* sinv = reinterpret_cast<double*>(smraw);            // pk
  double* sa = sinv + pk;                                       // max_nf * kRowPad
  double* sx = sa + max_nf * kRowPad;                           // max_nf * kSlots * BS
  double* r = sx + max_nf * kSlots * BS;                        // TP
  __shared__ unsigned long long bar;
  __shared__ int scols[kMaxPatchF * kSlots];
  __shared__ int sfac[kMaxPatchF];
  const int t = threadIdx.x;
  const int p = p0 + blockIdx.x;
  const int nf = P.nf[p], np = nf * BS;
  if (t < kMaxPatchF) sfac[t] = P.fac[p * kMaxPatchF + t];
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long off = P.off[p];
    const unsigned ib = unsigned((np * (np + 1) / 2 + 1) & ~1) * 8u;
    mbar_expect_tx(&bar, ib + unsigned(nf) * kRow * 8u);
    tma_bulk_g2s(sinv, P.inv + off, ib, &bar);
    for (int i = 0; i < nf; ++i)
      tma_bulk_g2s(sa + i * kRowPad, A.val + size_t(P.fac[p * kMaxPatchF + i]) * kRow, kRow * 8u, &bar);
  }
  __syncthreads();
  for (int e = t; e < nf * kSlots; e += TP) scols[e] = __ldg(&A.cols[sfac[e / kSlots] * kSlots + e % kSlots]);
  double bv = 0.0;
  if (t < np) bv = b[size_t(sfac[t / BS]) * BS + t % BS];
  __syncthreads();
  for (int e = t; e < nf * kSlots * BS; e += TP) {
    const int c = scols[e / BS];
    sx[e] = c >= 0 ? x[size_t(c) * BS + e % BS] : 0.0;
  }
  __syncthreads();
  mbar_wait(&bar, 0u);
  if (t < np) {
    const int lf = t / BS, i = t % BS;
    const double* arow = sa + lf * kRowPad + i * BS;
    const double* xr = sx + lf * kSlots * BS;
    double a0 = bv, a1 = 0.0;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
      for (int jj = 0; jj < BS; jj += 2) {
        const int j0 = (jj + i) % BS, j1 = (jj + 1 + i) % BS;
        a0 = fma(-arow[sl * BS * BS + j0], xr[sl * BS + j0], a0);
        a1 = fma(-arow[sl * BS * BS + j1], xr[sl * BS + j1], a1);
      }
    r[t] = a0 + a1;
  }
  __syncthreads();
  if (t < np) {
    const int ct = t * np - t * (t - 1) / 2 - t;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int j = 0;
    for (; j + 3 < np; j += 4) {
      double s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ju = j + u;
        s4[u] = sinv[ju >= t ? ct + ju : ju * np - ju * (ju - 1) / 2 + (t - ju)];
      }
      d0 = fma(s4[0], r[j], d0);
      d1 = fma(s4[1], r[j + 1], d1);
      d2 = fma(s4[2], r[j + 2], d2);
      d3 = fma(s4[3], r[j + 3], d3);
    }
    for (; j < np; ++j) d0 = fma(sinv[j >= t ? ct + j : j * np - j * (j - 1) / 2 + (t - j)], r[j], d0);
    x[size_t(sfac[t / BS]) * BS + t % BS] += (d0 + d1) + (d2 + d3);
  }
}

template <int BS>
void launch2(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int max_nf,
             cudaStream_t s) {
  constexpr int TP = BS == 4 ? 32 : 64;
  const int npmax = max_nf * BS;
  if (npmax > TP) throw std::runtime_error("vertex patch too large for the TMA sweep");
  const int pk = ((npmax * (npmax + 1) / 2) + 1) & ~1;
  const size_t smem = sizeof(double) * (size_t(pk) + size_t(max_nf) * (kSlots * BS * BS + 2) +
                                        size_t(max_nf) * kSlots * BS + TP);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_tma2<BS, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_sweep_tma2<BS, TP><<<w1 - w0, TP, smem, s>>>(A, P, w0, pk, max_nf, b, x);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (sweep_tma2): ") + cudaGetErrorString(err));
}

template <int BS>
struct Cfg;
template <>
struct Cfg<2> {
  static constexpr int TP = 16, G = 8;
};
template <>
struct Cfg<4> {
  static constexpr int TP = 32, G = 4;
};
template <>
struct Cfg<6> {
  static constexpr int TP = 64, G = 2;
};
template <>
struct Cfg<8> {
  static constexpr int TP = 64, G = 1;
};

template <int BS>
void launch1(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int max_nf, cudaStream_t s) {
  constexpr int TP = Cfg<BS>::TP, G = Cfg<BS>::G;
  const int npmax = max_nf * BS;
  if (npmax > TP) throw std::runtime_error("vertex patch too large for the TMA sweep");
  const int pk = ((npmax * (npmax + 1) / 2) + 1) & ~1;
  const size_t smem = sizeof(double) * (size_t(G) * pk + G * TP);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_tma1<BS, TP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int nblk = (w1 - w0 + G - 1) / G;
  k_sweep_tma1<BS, TP, G><<<nblk, G * TP, smem, s>>>(A, P, w0, w1, pk, b, x);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (sweep_tma1): ") + cudaGetErrorString(err));
}

template <int BS>
void launch(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int max_nf, cudaStream_t s) {
  constexpr int TP = Cfg<BS>::TP, G = Cfg<BS>::G;
  const int npmax = max_nf * BS;
  if (npmax > TP) throw std::runtime_error("vertex patch too large for the TMA sweep");
  const int pk = ((npmax * (npmax + 1) / 2) + 1) & ~1;
  const int inv_stage = G * pk;
  const int stage_d = inv_stage + G * max_nf * kSlots * BS * BS;
  const int ngroups = (w1 - w0 + G - 1) / G;
  static int occ = 0;
  static int attr_done = 0;
  const size_t base_smem = sizeof(double) * (size_t(kStages) * stage_d + G * TP) + 8 * kStages;
  if (!attr_done) {
    cudaFuncSetAttribute(k_sweep_tma<BS, TP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_tma<BS, TP, G>, G * TP,
                                                  base_smem + sizeof(Meta) * G * 8);
    if (occ < 1) occ = 1;
    attr_done = 1;
  }
  int grid = std::min(ngroups, 148 * occ);
  const int gpc = (ngroups + grid - 1) / grid;
  const size_t smem = base_smem + sizeof(Meta) * size_t(gpc) * G;
  if (smem > 227 * 1024) throw std::runtime_error("TMA sweep: shared memory budget exceeded");
  k_sweep_tma<BS, TP, G><<<grid, G * TP, smem, s>>>(A, P, w0, w1, ngroups, gpc, inv_stage, max_nf, b, x);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (sweep_tma): ") + cudaGetErrorString(err));
}

}  // namespace

void gs_wave_tma(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int max_nf,
                 cudaStream_t s) {
  if (w1 <= w0) return;
  static const bool kPersistent = [] {
    const char* e = std::getenv("HPMG_SWEEP");
    return e && std::string(e) == "persistent";
  }();
  switch (A.bs) {
    // HPMG_SWEEP=persistent selects the multi-stage persistent pipeline
    case 2: kPersistent ? launch<2>(A, P, w0, w1, b, x, max_nf, s) : launch1<2>(A, P, w0, w1, b, x, max_nf, s); break;
    case 4: kPersistent ? launch<4>(A, P, w0, w1, b, x, max_nf, s) : launch2<4>(A, P, w0, w1, b, x, max_nf, s); break;
    case 6: kPersistent ? launch<6>(A, P, w0, w1, b, x, max_nf, s) : launch2<6>(A, P, w0, w1, b, x, max_nf, s); break;
    case 8: kPersistent ? launch<8>(A, P, w0, w1, b, x, max_nf, s) : launch2<8>(A, P, w0, w1, b, x, max_nf, s); break;
    default: throw std::runtime_error("unsupported block size");
  }
}

}  // namespace dev
}  // namespace hpmg
