// Small lowest-order levels (bs = 2) in one persistent CTA.
//
// Level 1 of a 16x16 base mesh needs 50 dependent waves per multiplicative
// sweep (the reference's ascending-vertex order, smoother.hpp:53-57), each
// only ~16 patches wide: latency, not bandwidth, bounds it. One CTA runs a
// whole pre- (resp. post-) smoothing phase of the V-cycle with x and b
// resident in shared memory. The sweep is cut into passes (<= kPass patches
// of one wave, host-built list). Warp-specialised: a producer warp streams the
// patch records of pass k+2 by a TMA bulk copy (L2 evict-last, so they stay
// L2-resident across V-cycles) into a 3-slot mbarrier ring while the kPass x 16
// consumer threads compute pass k: r = b_p - A_pe x_e from the staged external
// blocks (sweep_rec.cu), then x_p = S r with the FULL patch inverse
// (column-major in the record, so the GEMV reads are bank-conflict free). A pass costs one __syncthreads().
// Symmetric operators only.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

namespace {

constexpr int kTP = 16;                      // threads (rows) per patch
constexpr int kPass = 24;                    // patches per pass (level-1 waves are 16-17 wide)
constexpr int kConsumers = kPass * kTP;      // 384
constexpr int kThreads = kConsumers + 32;    // + one producer warp
constexpr int kStages = 3;

__device__ __forceinline__ unsigned su32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

// development timeline of the one-CTA sweep (off unless hpmg_debug_small_trace arms it)
__device__ int d_trace_on = 0;
__device__ long long d_trace[4096];
__device__ __forceinline__ void stamp(int slot) {
  if (threadIdx.x == 0 && d_trace_on) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    d_trace[slot] = t;
  }
}

/// TMA bulk copy with an L2 evict-last hint.
__device__ __forceinline__ void ring_issue(unsigned long long* bar, double* dst, const double* src, unsigned bytes) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void ring_wait(unsigned long long* bar, unsigned phase) {
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

struct Smem {
  double *sx, *sb, *ring, *r;
  unsigned long long* bar;
  int2* pass;
};

__device__ Smem carve(int n, int stride, double* sm) {
  Smem v;
  v.sx = sm;
  v.sb = sm + n;
  v.ring = v.sb + n;
  v.r = v.ring + size_t(kStages) * kPass * stride;
  v.bar = reinterpret_cast<unsigned long long*>(v.r + kConsumers);
  v.pass = reinterpret_cast<int2*>(v.bar + kStages);
  return v;
}

/// All passes of `nsweeps` sweeps, forward or reversed, over the patch
/// records; NPM = 2 max_nf rows per patch (the level's largest patch), so
/// every load is unpredicated (S_p and the meta words are padded: rows past
/// the patch have facet -1 and zero S_p rows/columns). A patch's 16 threads
/// sit in one half-warp: the residual rows are exchanged under __syncwarp,
/// and one CTA barrier per pass publishes x_p to the next pass.
template <int NPM>
__device__ void sweeps(const PatchRecords& R, const int2* __restrict__ passes, int npass, int nsweeps, bool reverse,
                       const Smem& v) {
  static_assert(NPM <= kTP && NPM % 2 == 0, "patch rows per half-warp");
  const int lp = threadIdx.x / kTP, t = threadIdx.x % kTP;
  const bool producer = threadIdx.x >= kConsumers;
  const int total = npass * nsweeps;
  const bool trace = threadIdx.x == 0 && d_trace_on;  // read once: a global load per pass costs ~1 us
  for (int i = threadIdx.x; i < npass; i += blockDim.x) v.pass[i] = passes[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&v.bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto pass_of = [&](int k) {
    const int q = k % npass;
    return v.pass[reverse ? npass - 1 - q : q];
  };
  auto issue = [&](int k) {
    const int2 ps = pass_of(k);
    ring_issue(&v.bar[k % kStages], v.ring + size_t(k % kStages) * kPass * R.stride, R.rec + size_t(ps.x) * R.stride,
               unsigned(ps.y) * unsigned(R.stride) * 8u);
  };
  if (producer && threadIdx.x == kConsumers)
    for (int k = 0; k < kStages - 1 && k < total; ++k) issue(k);
  const int lf = t >> 1, i = t & 1;
  const bool rowthread = t < NPM;
  double* rr = v.r + lp * kTP;
  if (producer) {
    for (int k = 0; k < total; ++k) {
      // slot (k+2) % 3 held pass k-1, whose records the consumers moved to
      // registers before the barrier that closed pass k-2
      if (threadIdx.x == kConsumers && k + kStages - 1 < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + kStages - 1);
      }
      __syncthreads();
    }
    return;
  }
  // Software pipeline: everything of pass k that does not depend on x (the
  // S_p row, the external blocks, the meta words, b_p) is loaded into
  // registers during pass k-1, before the barrier that publishes pass k-1's
  // x; after the barrier a pass is only x_e -> residual -> GEMV -> x_p.
  double srow[NPM], w0[kExt], w1[kExt], bv = 0.0;
  int f = -1, c[kExt];
  bool active = false;
  auto fetch = [&](int k, int q) {
    const int2 ps = v.pass[reverse ? npass - 1 - q : q];
    active = lp < ps.y && rowthread;
    ring_wait(&v.bar[k % kStages], unsigned((k / kStages) & 1));
    if (!active) return;
    const double* rec = v.ring + (size_t(k % kStages) * kPass + lp) * R.stride;
    // row t of the full column-major S_p: S(t, j) at j*NPM + t
#pragma unroll
    for (int j = 0; j < NPM; ++j) srow[j] = rec[j * NPM + t];
    const int* meta = reinterpret_cast<const int*>(rec + R.meta_off);
    f = meta[1 + lf];  // -1: row past the patch
    const int* cols = meta + 1 + (NPM / 2) + lf * kExt;
    // the row's external-block entries [slot][col], contiguous (rowext
    // records; zero for empty slots): two 16-byte loads, no bank conflicts
    const double2* arow = reinterpret_cast<const double2*>(rec + R.a_off + t * kExt * 2);
#pragma unroll
    for (int sl = 0; sl < kExt; ++sl) {
      c[sl] = cols[sl];
      const double2 w = arow[sl];
      w0[sl] = w.x;
      w1[sl] = w.y;
    }
    bv = v.sb[2 * (f >= 0 ? f : 0) + i];
  };
  if (total > 0) fetch(0, 0);
  int q = 0;  // k % npass, kept incrementally (no division on the critical path)
  for (int k = 0; k < total; ++k) {
    if (trace && k < 1000) d_trace[4 * k] = d_trace[4 * k + 1] = clock64();
    if (active) {
      const int g = 2 * (f >= 0 ? f : 0) + i;
      double a0 = bv, a1 = 0.0;
#pragma unroll
      for (int sl = 0; sl < kExt; ++sl) {
        const double2 xe = *reinterpret_cast<const double2*>(v.sx + 2 * (c[sl] >= 0 ? c[sl] : 0));
        a0 = fma(-w0[sl], xe.x, a0);
        a1 = fma(-w1[sl], xe.y, a1);
      }
      rr[t] = f >= 0 ? a0 + a1 : 0.0;
      __syncwarp(((1u << NPM) - 1u) << (threadIdx.x & 16));  // the patch's row threads
      if (trace && k < 1000) d_trace[4 * k + 2] = clock64();
      // x_p = S_p (b_p - A_pe x_e) (sweep_rec.cu); padded columns are zero
      double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < NPM; j += 2) {
        const double2 r2 = *reinterpret_cast<const double2*>(rr + j);
        d[j & 3] = fma(srow[j], r2.x, d[j & 3]);
        d[(j + 1) & 3] = fma(srow[j + 1], r2.y, d[(j + 1) & 3]);
      }
      if (f >= 0) v.sx[g] = (d[0] + d[1]) + (d[2] + d[3]);
    }
    q = q + 1 == npass ? 0 : q + 1;
    if (k + 1 < total) fetch(k + 1, q);
    __syncthreads();
    if (trace && k < 1000) d_trace[4 * k + 3] = clock64();
  }
}

/// x = 0; pre-smooth (reference multigrid.hpp:174-175). The residual and the
/// restriction run grid-wide after it (small_pre): their latency-bound CSR
/// loops cost ~90 us in one CTA.
template <int NPM>
__global__ void __launch_bounds__(kThreads) k_small_pre(int n, PatchRecords R, const int2* __restrict__ passes,
                                                        int npass, int nsweeps, const double* __restrict__ b,
                                                        double* __restrict__ x, int64_t ld, int unit0) {
  extern __shared__ __align__(128) double sm[];
  Smem v = carve(n, R.stride, sm);
  stamp(4088);
  // batched (setup of the dense level-1 cycle, dense_level.cu): CTA j sweeps
  // column j of x (leading dimension ld) with b = e_{unit0 + j}
  x += blockIdx.x * ld;
  const int unit = unit0 >= 0 ? unit0 + int(blockIdx.x) : -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    v.sx[i] = 0.0;
    v.sb[i] = unit >= 0 ? (i == unit ? 1.0 : 0.0) : b[i];
  }
  __syncthreads();
  stamp(4089);
  sweeps<NPM>(R, passes, npass, nsweeps, false, v);
  stamp(4090);
  for (int t = threadIdx.x; t < n; t += blockDim.x) x[t] = v.sx[t];
  stamp(4091);
}

/// post-smooth (reverse sweep) of x, after the grid-wide x += P e (multigrid.hpp:181-182)
template <int NPM>
__global__ void __launch_bounds__(kThreads) k_small_post(int n, PatchRecords R, const int2* __restrict__ passes,
                                                         int npass, int nsweeps, const double* __restrict__ b,
                                                         double* __restrict__ x, int64_t ld, int unit0) {
  extern __shared__ __align__(128) double sm[];
  Smem v = carve(n, R.stride, sm);
  stamp(4092);
  x += blockIdx.x * ld;
  const int unit = unit0 >= 0 ? unit0 + int(blockIdx.x) : -1;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    v.sx[t] = x[t];
    v.sb[t] = unit >= 0 ? (t == unit ? 1.0 : 0.0) : b[t];
  }
  __syncthreads();
  stamp(4093);
  sweeps<NPM>(R, passes, npass, nsweeps, true, v);
  stamp(4094);
  for (int t = threadIdx.x; t < n; t += blockDim.x) x[t] = v.sx[t];
  stamp(4095);
}

/// launches k_small_pre / k_small_post for the level's patch row count
template <bool kPost>
void launch_small(const PatchRecords& R, int n, const int2* passes, int npass, int nsweeps, const double* b,
                  double* x, size_t smem, cudaStream_t s, int ncols = 1, int64_t ld = 0, int unit0 = -1) {
  auto go = [&](auto kernel) {
    // once per kernel instantiation (all of them share this lambda's type)
    static const void* done[16] = {};
    bool set = false;
    for (const void* d : done) set = set || d == reinterpret_cast<const void*>(kernel);
    if (!set) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      for (auto& d : done)
        if (!d) {
          d = reinterpret_cast<const void*>(kernel);
          break;
        }
    }
    kernel<<<ncols, kThreads, smem, s>>>(n, R, passes, npass, nsweeps, b, x, ld, unit0);
  };
  switch (R.max_nf) {
    case 4: go(kPost ? k_small_post<8> : k_small_pre<8>); break;
    case 5: go(kPost ? k_small_post<10> : k_small_pre<10>); break;
    case 6: go(kPost ? k_small_post<12> : k_small_pre<12>); break;
    case 7: go(kPost ? k_small_post<14> : k_small_pre<14>); break;
    case 8: go(kPost ? k_small_post<16> : k_small_pre<16>); break;
    default: throw std::runtime_error("small-level sweep: unsupported patch size");
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA launch: ") + cudaGetErrorString(err));
}

size_t smem_bytes(int nb, int stride, int npass) {
  return sizeof(double) * (size_t(4) * nb + size_t(kStages) * kPass * stride + kConsumers) + 8 * kStages +
         sizeof(int2) * size_t(npass);
}

}  // namespace

int small_pass_patches() { return kPass; }

void small_trace(int arm, long long* out) {
  cudaMemcpyToSymbol(d_trace_on, &arm, sizeof(int));
  if (out) cudaMemcpyFromSymbol(out, d_trace, sizeof(long long) * 4096);
}

bool small_level_fits(int nb, int record_stride, int npass) {
  return smem_bytes(nb, record_stride, npass) <= 225 * 1024;
}

void small_pre(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& PT,
               const double* b, double* x, double* r, double* rc, cudaStream_t s) {
  if (!R.full || !R.rowext || R.bs != 2) throw std::runtime_error("small-level sweeps need full-inverse row-ordered records");
  launch_small<false>(R, A.nb * 2, passes, npass, sweeps, b, x, smem_bytes(A.nb, R.stride, npass), s);
  spmv(A, x, b, r, 1, nullptr, nullptr, s);
  restrict_(PT, r, rc, s);
}

void small_post(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& Pm,
                const double* e, const double* b, double* x, cudaStream_t s) {
  prolong_add(Pm, e, x, s);
  launch_small<true>(R, A.nb * 2, passes, npass, sweeps, b, x, smem_bytes(A.nb, R.stride, npass), s);
}

void small_pre_batch(const PatchRecords& R, int nb, const int2* passes, int npass, int sweeps, int ncols, int unit0,
                     double* X, int64_t ld, cudaStream_t s) {
  launch_small<false>(R, nb * 2, passes, npass, sweeps, nullptr, X, smem_bytes(nb, R.stride, npass), s, ncols, ld, unit0);
}

void small_post_batch(const PatchRecords& R, int nb, const int2* passes, int npass, int sweeps, int ncols, int unit0,
                      double* X, int64_t ld, cudaStream_t s) {
  launch_small<true>(R, nb * 2, passes, npass, sweeps, nullptr, X, smem_bytes(nb, R.stride, npass), s, ncols, ld, unit0);
}

}  // namespace dev
}  // namespace hpmg
