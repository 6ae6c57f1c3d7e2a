// Patch-record multiplicative sweep (symmetric operators): the dominant
// kernel of the hp-MG V-cycle (reference
// inc/smoother.hpp:53-67, 83-94).
//
// Every vertex patch owns one fixed-stride record in HBM, built once at setup:
//   [ patch inverse S_p (packed lower triangle by columns, or full)
//   | A_pe: per patch facet the <= 2 blocks coupling it to facets outside the
//     patch (facet (v,w) of the star of v couples to (v,a), (v,b) inside and
//     to the far edges (w,a), (w,b) outside), each block column-major
//   | int32 meta: nf, facet ids, the external block columns ]
// and the sweep sets x_p = S_p (b_p - A_pe x_e): with S_p A_pp = I this is the
// reference update x_p += S_p (b - A x)_p without ever reading A_pp, which
// cuts the A bytes per sweep from 10 to 4 blocks per facet (each facet sits in
// two patches). A CTA needs no dependent index loads: one elected thread
// issues TMA bulk copies (cp.async.bulk, L2 evict-first so the streamed
// records do not evict x and b) of the records of its patch group, addressed
// by the patch id alone, onto mbarriers. The threads then gather the external
// x blocks (the only dependent round, L2-resident), form the right-hand side
// from shared memory and apply the inverse.
//
// Ordering. The reference sweep is sequential in ascending vertex order; two
// patches conflict iff their vertices are mesh neighbours.
// One launch per wave of mutually independent patches (gs_wave_rec),
// chained by programmatic dependent launch, reproduces it exactly. (Round 1
// also kept a one-launch-per-sweep dataflow schedule and a cooperative
// persistent one; both were slower on B200 and were removed.)
#include <cuda_runtime.h>

#include <algorithm>
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
__device__ __forceinline__ void bar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
/// bulk copy completing on `bar` (whose expected bytes were announced by bar_expect)
__device__ __forceinline__ void tma_part(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}

// development timeline (R.dbg & 4): per CTA of the last launches, globaltimer
// at start / A-part landed / gather done / S landed / end
__device__ long long d_sweep_trace[5 * 32768];
__device__ __forceinline__ void sweep_stamp(const PatchRecords& R, int k) {
  if ((R.dbg & 4) && threadIdx.x == 0 && blockIdx.x < 32768) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    d_sweep_trace[5 * blockIdx.x + k] = t;
  }
}

/// One patch update x_p = S_p (b_p - A_pe x_e) from its record in shared
/// memory (meta words landed): the x_e gather with b_p, the residual rows
/// (waiting for A_pe through wait_a), the packed / full GEMV (waiting for
/// S_p through wait_s), the store of x_p.
template <int BS, int TP, bool kOneCopy, class WaitA, class WaitS>
__device__ __forceinline__ void patch_update(const PatchRecords& R, const double* rec, int lp, int ng, int t,
                                             double* sx, double* r, const double* __restrict__ b,
                                             double* __restrict__ x, int xz, WaitA wait_a, WaitS wait_s) {
  constexpr int kRow = kExt * BS * BS;
  const int* meta = reinterpret_cast<const int*>(rec + R.meta_off);
  const int nf = lp < ng ? meta[0] : 0, np = nf * BS;
  const int* fac = meta + 1;
  const int* ecol = meta + 1 + R.max_nf;
  double* xs = sx + lp * R.max_nf * kExt * BS;
  // TR threads per patch row: with TR = 2 each takes one external block of
  // the residual and half of the GEMV columns, combined by a lane shuffle
  constexpr int TR = TP >= 2 * kMaxPatchF * BS ? 2 : 1;
  const int row = t / TR, part = t % TR;
  // b_p is issued together with the x_e gather (both L2 round trips)
  double bv = 0.0;
  if (row < np && part == 0) bv = __ldg(b + size_t(fac[row / BS]) * BS + row % BS);
  if (!xz) {
    // all loads of this thread in flight at once, then the shared stores
    constexpr int kPer = (kMaxPatchF * kExt * BS + TP - 1) / TP;
    const int ne = nf * kExt * BS;
    double v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = t + u * TP;
      const int c = e < ne ? ecol[e / BS] : -1;
      v[u] = c < 0 ? 0.0 : x[size_t(c) * BS + e % BS];
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u)
      if (t + u * TP < ne) xs[t + u * TP] = v[u];
  }
  if (!kOneCopy && !xz) wait_a();
  __syncthreads();
  sweep_stamp(R, 2);
  double rsum = 0.0;
  if (row < np && xz) {
    rsum = bv;  // x_e = 0: the residual rows are b_p
  } else if (row < np) {
    const int lf = row / BS, i = row % BS;
    // external blocks are stored column-major: A(i, j) at j*BS + i, so the
    // rows of a block are consecutive words; the column order is rotated by
    // the facet so the facets of a warp hit distinct banks, while all rows of
    // one facet read the same x_e word (broadcast)
    const double* acol = rec + R.a_off + lf * kRow + i;
    const double* xr = xs + lf * kExt * BS;
    double a0 = bv, a1 = 0.0;
#pragma unroll
    for (int sq = 0; sq < kExt / TR; ++sq) {
      const int sl = sq * TR + part;
#pragma unroll
      for (int jj = 0; jj < BS; jj += 2) {
        const int j0 = (jj + lf) % BS, j1 = (jj + 1 + lf) % BS;
        a0 = fma(-acol[sl * BS * BS + j0 * BS], xr[sl * BS + j0], a0);
        a1 = fma(-acol[sl * BS * BS + j1 * BS], xr[sl * BS + j1], a1);
      }
    }
    rsum = a0 + a1;
  }
  if (TR == 2) rsum += __shfl_xor_sync(0xffffffffu, rsum, 1);
  if (r == sx) __syncthreads();  // r aliases the x_e staging (one patch per CTA)
  if (row < np && part == 0) r[lp * TP + row] = rsum;
  __syncthreads();
  if (!kOneCopy) wait_s();
  sweep_stamp(R, 3);
  double dsum = 0.0;
  if (row < np && R.full) {
    // full inverse (nonsymmetric operators), column-major with the level's
    // largest patch as column stride: S(t, j) at j*npm + t
    const int npm = R.max_nf * BS;
    const double* S = rec + row;
    const double* rr = r + lp * TP;
    const int jb = TR == 2 ? part * (np / 2) : 0, je = TR == 2 ? (part + 1) * (np / 2) : np;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int j = jb;
    for (; j + 3 < je; j += 4) {
      d0 = fma(S[j * npm], rr[j], d0);
      d1 = fma(S[(j + 1) * npm], rr[j + 1], d1);
      d2 = fma(S[(j + 2) * npm], rr[j + 2], d2);
      d3 = fma(S[(j + 3) * npm], rr[j + 3], d3);
    }
    for (; j < je; ++j) d0 = fma(S[j * npm], rr[j], d0);
    dsum = (d0 + d1) + (d2 + d3);
  } else if (row < np) {
    // S(t, j): j < t in column j at cs(j) + t - j, j >= t in column t at ct + j,
    // cs(j) = j np - j (j - 1) / 2 the uniform column start (packed lower, by columns);
    // with TR = 2 the two lanes of a row take the columns [0, np/2) and [np/2, np)
    const int t = row;
    const double* S = rec;
    const double* rr = r + lp * TP;
    const int ct = t * np - t * (t - 1) / 2 - t;
    const int jb = TR == 2 ? part * (np / 2) : 0, je = TR == 2 ? (part + 1) * (np / 2) : np;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int cs = jb * np - jb * (jb - 1) / 2, j = jb;
    for (; j + 3 < je; j += 4) {
      const int o0 = j < t ? cs + t - j : ct + j;
      cs += np - j;
      const int o1 = j + 1 < t ? cs + t - j - 1 : ct + j + 1;
      cs += np - j - 1;
      const int o2 = j + 2 < t ? cs + t - j - 2 : ct + j + 2;
      cs += np - j - 2;
      const int o3 = j + 3 < t ? cs + t - j - 3 : ct + j + 3;
      cs += np - j - 3;
      const double2 r01 = *reinterpret_cast<const double2*>(rr + j);  // broadcast, 16-byte words
      const double2 r23 = *reinterpret_cast<const double2*>(rr + j + 2);
      d0 = fma(S[o0], r01.x, d0);
      d1 = fma(S[o1], r01.y, d1);
      d2 = fma(S[o2], r23.x, d2);
      d3 = fma(S[o3], r23.y, d3);
    }
    for (; j < je; ++j) {
      d0 = fma(S[j < t ? cs + t - j : ct + j], rr[j], d0);
      cs += np - j;
    }
    dsum = (d0 + d1) + (d2 + d3);
  }
  if (TR == 2) dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
  if (row < np && part == 0) x[size_t(fac[row / BS]) * BS + row % BS] = dsum;
}

/// Records of G consecutive patches per CTA, TP threads per patch: one wave [p0, p1).
/// xz: the wave's x_e is known to be zero (first wave of a sweep started from
/// x = 0): r_p = b_p exactly, so A_pe is neither copied nor applied and x_e is
/// not gathered (bitwise the same result).
template <int BS, int TP, int G>
__global__ void __launch_bounds__(G* TP) k_sweep(PatchRecords R, int p0, int p1, const double* __restrict__ b,
                                                 double* __restrict__ x, int xz) {
  constexpr bool kOneCopy = G > 1;  // grouped small records: one copy per CTA
  extern __shared__ __align__(128) unsigned char smraw[];
  double* srec = reinterpret_cast<double*>(smraw);  // G * stride
  double* sx = srec + size_t(G) * R.stride;          // G * max_nf * kExt * BS
  // one patch per CTA: the residual rows live in the x_e staging area, dead
  // once the residual is formed (patch_update orders the two with a barrier)
  double* r = G == 1 ? sx : sx + G * R.max_nf * kExt * BS;  // G * TP
  __shared__ unsigned long long bar, bar_s, bar_m;
  const int lp = threadIdx.x / TP, t = threadIdx.x % TP;
  const int q0 = p0 + blockIdx.x * G, ng = min(G, p1 - q0);
  sweep_stamp(R, 0);
  if (threadIdx.x == 0) {
    // three copies per patch: the meta words first (the x_e gather needs only
    // them), then A_pe (residual), then the inverse S_p, which lands while
    // x_e is being gathered
    bar_init(&bar);
    bar_init(&bar_s);
    bar_init(&bar_m);
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (kOneCopy) {
      // small records of consecutive patches: one bulk copy for the group
      const unsigned all = unsigned(ng) * unsigned(R.stride) * 8u;
      bar_expect(&bar_m, all);
      tma_part(srec, R.rec + size_t(q0) * R.stride, all, &bar_m, pol);
    } else {
      const unsigned mbytes = unsigned(R.stride - R.meta_off) * 8u, abytes = unsigned(R.meta_off - R.a_off) * 8u,
                     head = unsigned(R.a_off) * 8u;
      bar_expect(&bar_m, unsigned(ng) * mbytes);
      if (!xz) bar_expect(&bar, unsigned(ng) * abytes);
      bar_expect(&bar_s, unsigned(ng) * head);
      for (int q = 0; q < ng; ++q)
        tma_part(srec + size_t(q) * R.stride + R.meta_off, R.rec + size_t(q0 + q) * R.stride + R.meta_off, mbytes,
                 &bar_m, pol);
      if (!xz)
        for (int q = 0; q < ng; ++q)
          tma_part(srec + size_t(q) * R.stride + R.a_off, R.rec + size_t(q0 + q) * R.stride + R.a_off, abytes, &bar,
                   pol);
      for (int q = 0; q < ng; ++q)
        tma_part(srec + size_t(q) * R.stride, R.rec + size_t(q0 + q) * R.stride, head, &bar_s, pol);
    }
  }
  // Programmatic dependent launch: the records do not depend on the previous
  // kernel, so the copies above may overlap its tail; x and b may not be
  // touched before it has completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  bar_wait(&bar_m);
  sweep_stamp(R, 1);
  patch_update<BS, TP, kOneCopy>(R, srec + size_t(lp) * R.stride, lp, ng, t, sx, r, b, x, xz,
                                 [&] { bar_wait(&bar); }, [&] { bar_wait(&bar_s); });
  if (R.dbg & 4) {
    __syncthreads();
    sweep_stamp(R, 4);
  }
}

/// Builds the records from the packed inverses and the ELL operator.
__global__ void k_build_records(Bsr A, Patches P, PatchRecords R, int bs, int transpose) {
  const int p = blockIdx.x;
  double* rec = R.rec + size_t(p) * R.stride;
  const int nf = P.nf[p], np = nf * bs;
  const int pk = np * (np + 1) / 2;
  const double* inv = P.inv + P.off[p];
  if (R.full) {
    // unpack the symmetric triangle: (r, c) at c*npmax + r, zero-padded to the
    // level's largest patch, so readers address S without the patch's own size
    const int npmax = R.max_nf * bs;
    for (int k = threadIdx.x; k < R.a_off; k += blockDim.x) {
      double v = 0.0;
      const int c = k / npmax, r = k % npmax;
      if (c < np && r < np) {
        if (P.packed) {
          const int lo = r > c ? c : r, hi = r > c ? r : c;
          v = inv[lo * np - lo * (lo - 1) / 2 + (hi - lo)];
        } else {  // full column-major inverse (nonsymmetric); S^T for the transposed sweep
          v = transpose ? inv[r * np + c] : inv[c * np + r];
        }
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
      if (ne == kExt) break;  // excluded by the host check (triangle meshes)
      meta[1 + R.max_nf + lf * kExt + ne] = c;
      for (int e = 0; e < blk; ++e) {  // A.val block row-major: (r, c) = e
        const int r = e / bs, c = e % bs;
        // column-major block: (r, c) at c*bs + r; rowext: a patch row's
        // 2 x kExt values contiguous (one 32-byte read per row, bs = 2)
        const int at = R.rowext ? ((lf * bs + r) * kExt + ne) * bs + c : (lf * kExt + ne) * blk + c * bs + r;
        rec[R.a_off + at] = A.val[(size_t(f) * kSlots + sl) * blk + e];
      }
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
  static constexpr int TP = 128, G = 1;  // two threads per patch row
};
template <>
struct RecCfg<10> {  // k = 4..6 (beyond the reference): one thread per row, np <= 8 * 14
  static constexpr int TP = 128, G = 1;
};
template <>
struct RecCfg<12> {
  static constexpr int TP = 128, G = 1;
};
template <>
struct RecCfg<14> {
  static constexpr int TP = 128, G = 1;
};

/// dataflow launches carry a fixed per-CTA cost (dependency polls, release
/// fence), so they group more patches per CTA
template <int BS>
struct Grp {
  static constexpr int G = RecCfg<BS>::G;
};

template <int BS>
void launch(const PatchRecords& R, int p0, int p1, int nblocks, const double* b, double* x, int xz, cudaStream_t s) {
  constexpr int TP = RecCfg<BS>::TP, G = Grp<BS>::G;
  if (R.max_nf * BS * (TP >= 2 * kMaxPatchF * BS ? 2 : 1) > TP)
    throw std::runtime_error("vertex patch too large for the record sweep");
  const size_t smem = sizeof(double) * (size_t(G) * R.stride + size_t(G) * R.max_nf * kExt * BS + (G == 1 ? 0 : G * TP));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep<BS, TP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(G * TP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  cudaError_t err = cudaLaunchKernelEx(&cfg, k_sweep<BS, TP, G>, R, p0, p1, b, x, xz);
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (sweep): ") + cudaGetErrorString(err));
}

void launch_bs(const PatchRecords& R, int p0, int p1, int nblocks, const double* b, double* x, int xz,
               cudaStream_t s) {
  switch (R.bs) {
    case 2: launch<2>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 4: launch<4>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 6: launch<6>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 8: launch<8>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 10: launch<10>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 12: launch<12>(R, p0, p1, nblocks, b, x, xz, s); break;
    case 14: launch<14>(R, p0, p1, nblocks, b, x, xz, s); break;
    default: throw std::runtime_error("unsupported block size");
  }
}

int group_of(int bs) {
  switch (bs) {
    case 2: return Grp<2>::G;
    case 4: return Grp<4>::G;
    case 6: return Grp<6>::G;
    case 8: return Grp<8>::G;
    case 10: return Grp<10>::G;
    case 12: return Grp<12>::G;
    case 14: return Grp<14>::G;
    default: throw std::runtime_error("unsupported block size");
  }
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

void build_records(const Bsr& A, const Patches& P, PatchRecords& R, cudaStream_t s, bool transpose) {
  if (P.n == 0) return;
  if (!P.packed && !R.full) throw std::runtime_error("nonsymmetric patch inverses need full records");
  k_build_records<<<P.n, 128, 0, s>>>(A, P, R, R.bs, transpose ? 1 : 0);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (build_records): ") + cudaGetErrorString(err));
}

void sweep_trace(long long* out) { cudaMemcpyFromSymbol(out, d_sweep_trace, sizeof(long long) * 5 * 32768); }

void gs_wave_rec(const PatchRecords& R, int w0, int w1, const double* b, double* x, cudaStream_t s, bool x_zero) {
  if (w1 <= w0) return;
  const int G = group_of(R.bs);
  launch_bs(R, w0, w1, (w1 - w0 + G - 1) / G, b, x, x_zero ? 1 : 0, s);
}

}  // namespace dev
}  // namespace hpmg
