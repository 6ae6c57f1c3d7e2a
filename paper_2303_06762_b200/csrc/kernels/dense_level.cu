// Level 1 + the coarse solve as one dense operator.
//
// On a V(1,1) cycle with the multiplicative smoother the level-1 sub-cycle of
// the reference (multigrid.hpp:166-185 at l = 1: forward patch sweep from
// x = 0, r = b - A x, x += P C^-1 P^T r, backward sweep) is a fixed linear map
// b -> x of the level-1 residual: x = M1 b. Its one-CTA sweeps are bound by
// 2 x 50 dependent passes (~33 us each), not by data. At setup M1 is formed
// column by column by running exactly those steps on the unit vectors
// (the batched one-CTA sweeps of small_levels.cu, one CTA per column, and
// batched residual / transfer / coarse kernels below), transposed to
// row-major, and every V-cycle then applies it with one HBM-bound GEMV
// (k_dense_rowgemv). Same map, different rounding: each column is the
// reference algorithm applied to e_j, and M1 b sums them in a fixed order.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

namespace {

#define DL_CHECK()                                                                               \
  do {                                                                                           \
    cudaError_t e_ = cudaGetLastError();                                                         \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA launch: ") + cudaGetErrorString(e_)); \
  } while (0)

/// R[:, j] = e_{unit0 + j} - A X[:, j] (bs = 2), one column per blockIdx.y
__global__ void k_batch_residual(Bsr A, const double* __restrict__ X, double* __restrict__ R, int64_t ld, int unit0) {
  const int j = blockIdx.y;
  const int64_t n = int64_t(A.nb) * 2;
  const double* x = X + j * ld;
  double* r = R + j * ld;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int f = int(t >> 1), i = int(t & 1);
    double s = 0.0;
    for (int sl = 0; sl < kSlots; ++sl) {
      const int c = __ldg(&A.cols[f * kSlots + sl]);
      if (c < 0) continue;
      const double* blk = A.val + (size_t(f * kSlots + sl) * 2 + i) * 2;
      s = fma(__ldg(blk), x[2 * c], s);
      s = fma(__ldg(blk + 1), x[2 * c + 1], s);
    }
    r[t] = (t == unit0 + j ? 1.0 : 0.0) - s;
  }
}

/// Y[:, j] (+)= M V[:, j] for a 2x2 block CSR matrix, one column per blockIdx.y
__global__ void k_batch_bcsr(BlockCsr M, const double* __restrict__ V, int64_t ldv, double* __restrict__ Y, int64_t ldy,
                             int acc) {
  const int j = blockIdx.y;
  const double* v = V + j * ldv;
  double* y = Y + j * ldy;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < M.nrows; row += gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    for (int q = __ldg(&M.ptr[row]); q < __ldg(&M.ptr[row + 1]); ++q) {
      const int c = __ldg(&M.col[q]);
      const double* a = M.val + size_t(q) * 4;
      s0 = fma(__ldg(a), v[2 * c], fma(__ldg(a + 1), v[2 * c + 1], s0));
      s1 = fma(__ldg(a + 2), v[2 * c], fma(__ldg(a + 3), v[2 * c + 1], s1));
    }
    if (acc) {
      y[2 * row] += s0;
      y[2 * row + 1] += s1;
    } else {
      y[2 * row] = s0;
      y[2 * row + 1] = s1;
    }
  }
}

/// C = A B, column-major: A n x n (lda n), B n x m (ldb n), C n x m (ldc n).
/// Setup only (the coarse inverse applied to every restricted column):
/// 64 x 64 tiles, 16-deep k slabs, 4 x 4 outputs per thread.
constexpr int kT = 64, kK = 16;
__global__ void __launch_bounds__(256) k_dgemm_nn(int n, int m, const double* __restrict__ A, const double* __restrict__ B,
                                                  double* __restrict__ C) {
  __shared__ double sa[kK][kT + 1], sb[kK][kT + 1];
  const int i0 = blockIdx.x * kT, j0 = blockIdx.y * kT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += kK) {
    for (int e = threadIdx.x; e < kK * kT; e += 256) {
      const int kk = e / kT, ii = e % kT;  // A(i0 + ii, k0 + kk): consecutive threads down a column
      sa[kk][ii] = (i0 + ii < n && k0 + kk < n) ? A[size_t(k0 + kk) * n + i0 + ii] : 0.0;
      const int kb = e % kK, jj = e / kK;  // B(k0 + kb, j0 + jj)
      sb[kb][jj] = (k0 + kb < n && j0 + jj < m) ? B[size_t(j0 + jj) * n + k0 + kb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = sa[kk][tx + 16 * u];
        b[u] = sb[kk][ty + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = fma(a[u], b[w], acc[u][w]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int i = i0 + tx + 16 * u, j = j0 + ty + 16 * w;
      if (i < n && j < m) C[size_t(j) * n + i] = acc[u][w];
    }
}

/// M[i][j] = X[j][i] (n x n, M with row stride ld), 32 x 32 tiles through shared memory
__global__ void k_transpose_sq(int n, int ld, const double* __restrict__ X, double* __restrict__ M) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = by + r, i = bx + threadIdx.x;
    if (i < n && j < n) t[r][threadIdx.x] = X[size_t(j) * n + i];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + r, j = by + threadIdx.x;
    if (i < n && j < n) M[size_t(i) * ld + j] = t[threadIdx.x][r];
  }
}

/// y = M b, M row-major n x ld with ld a multiple of 2,048 (zero columns
/// past n; b readable and zero up to ld). Two rows per 256-thread CTA, four
/// warps per row; warp w takes the row's 256-double2 batches w, w + 4, ...,
/// eight loads per lane in flight at constant offsets (no tail: a clamped or
/// predicated remainder made ptxas serialise each load with its FMAs). M
/// streams evict-first, b stays cache-resident; the partial sums are combined
/// in a fixed order (shuffle tree, then the four warps in order). 3,008 CTAs
/// at n = 6,016 spread evenly over the SMs (one warp per row left a 1.27-wave
/// tail).
constexpr int kRowPad = 2048;
__global__ void __launch_bounds__(256) k_dense_rowgemv(int n, int ld, const double* __restrict__ M,
                                                      const double* __restrict__ b, double* __restrict__ y) {
  __shared__ double part[8];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = blockIdx.x * 2 + w / 4, wq = w % 4;
  double v = 0.0;
  if (row < n) {
    const double2* m = reinterpret_cast<const double2*>(M + size_t(row) * ld) + lane;
    const double2* bb = reinterpret_cast<const double2*>(b) + lane;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = wq * 256; q < ld / 2; q += 4 * 256) {
      double2 a[8], x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldcs(m + q + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(bb + q + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s[u & 3] = fma(a[u].x, x[u].x, s[u & 3]);
        s[u & 3] = fma(a[u].y, x[u].y, s[u & 3]);
      }
    }
    v = (s[0] + s[1]) + (s[2] + s[3]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) part[w] = v;
  __syncthreads();
  if (threadIdx.x < 2) {
    const int r = blockIdx.x * 2 + threadIdx.x;
    const double* p = part + 4 * threadIdx.x;
    if (r < n) y[r] = (p[0] + p[1]) + (p[2] + p[3]);
  }
}

/// Symmetric storage (the default: M1 is symmetric in exact arithmetic for
/// the symmetric operators the one-CTA level serves; stored as S = (M1 +
/// M1^T) / 2): the lower-triangle 64 x 64 tiles (I >= J) row-major, tile
/// t(I, J) = I (I + 1) / 2 + J, half the bytes of the full map. One warp per
/// tile, two per 64-thread CTA (102 registers: small CTAs keep the SMs evenly
/// loaded): lane l holds columns 2l, 2l + 1 of each row; the column part
/// T^T b_I accumulates lane-locally, the row part T b_J per row is reduced
/// across the warp 32 rows at a time by a transposing butterfly (31
/// shuffles per 32 rows, lane r ends with row r). Both parts go to per-tile
/// partials, summed per output row in a fixed order by k_sym_combine.
constexpr int kTile = 64;
__host__ __device__ __forceinline__ size_t tri(int i) { return size_t(i) * (i + 1) / 2; }

__global__ void k_sym_pack(int n, int nb, const double* __restrict__ X, double* __restrict__ T) {
  // one CTA per tile; X column-major: M1(i, j) = X[j n + i]
  const int t = blockIdx.x;
  int I = int((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
  while (tri(I + 1) <= size_t(t)) ++I;
  while (tri(I) > size_t(t)) --I;
  const int J = t - int(tri(I));
  double* out = T + size_t(t) * kTile * kTile;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile, i = I * kTile + r, j = J * kTile + c;
    out[e] = (i < n && j < n) ? 0.5 * (X[size_t(j) * n + i] + X[size_t(i) * n + j]) : 0.0;
  }
}

__global__ void __launch_bounds__(64) k_sym_tiles(int ntiles, const double* __restrict__ T, const double* __restrict__ b,
                                                  double* __restrict__ prow, double* __restrict__ pcol) {
  const int t = blockIdx.x * 2 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= ntiles) return;
  int I = int((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
  while (tri(I + 1) <= size_t(t)) ++I;
  while (tri(I) > size_t(t)) --I;
  const int J = t - int(tri(I));
  const double2* tile = reinterpret_cast<const double2*>(T + size_t(t) * kTile * kTile) + lane;
  const double2 bj = __ldg(reinterpret_cast<const double2*>(b + J * kTile) + lane);
  const double* bi = b + I * kTile;
  double cx = 0.0, cy = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double p[32];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      double2 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldcs(tile + (h * 32 + g * 8 + u) * (kTile / 2));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = h * 32 + g * 8 + u;
        const double br = __ldg(bi + r);
        p[g * 8 + u] = fma(a[u].x, bj.x, a[u].y * bj.y);
        cx = fma(a[u].x, br, cx);
        cy = fma(a[u].y, br, cy);
      }
    }
    // transposing butterfly: after the stage with offset o each lane keeps o
    // values; lane l ends with the warp sum of row (h * 32 + l)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const bool up = lane & o;
#pragma unroll
      for (int i = 0; i < o; ++i) {
        const double send = up ? p[i] : p[i + o];
        const double keep = up ? p[i + o] : p[i];
        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    prow[size_t(t) * kTile + h * 32 + lane] = p[0];
  }
  if (I != J) reinterpret_cast<double2*>(pcol + size_t(t) * kTile)[lane] = make_double2(cx, cy);
}

/// y_i, i = 64 K + r: the row parts of tiles (K, 0..K), then the column parts
/// of tiles (K+1..nb-1, K), four lanes per output (terms q = g, g + 4, ...),
/// combined in a fixed order
__global__ void __launch_bounds__(256) k_sym_combine(int n, int nb, const double* __restrict__ prow,
                                                    const double* __restrict__ pcol, double* __restrict__ y) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = gt / 4, g = gt % 4;
  const int K = min(i / kTile, nb - 1), r = i % kTile;
  double s = 0.0;
  if (i < n) {
    for (int q = g; q < nb; q += 4) {
      const double v = q <= K ? prow[(tri(K) + q) * kTile + r] : pcol[(tri(q) + K) * kTile + r];
      s += v;
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (i < n && g == 0) y[i] = s;
}

}  // namespace

void dense_level1(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& PT,
                  const BlockCsr& Pm, int n0, const double* coarse_inv, double* M1, double* work, bool sym,
                  cudaStream_t s) {
  const int n = A.nb * 2;
  if (n % 2 || n0 % 2) throw std::runtime_error("dense level 1: odd size");
  auto chk = [](cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA dense level 1: ") + cudaGetErrorString(e));
  };
  const size_t nn = size_t(n) * n, nc = size_t(n0) * n;
  double *X = work, *Rr = X + nn, *Rc = Rr + nn, *E = Rc + nc;
  // X[:, j] = forward sweep(s) of e_j from x = 0
  small_pre_batch(R, A.nb, passes, npass, sweeps, n, 0, X, n, s);
  const int gx = (n + 255) / 256;
  k_batch_residual<<<dim3(std::min(gx, 32), n), 256, 0, s>>>(A, X, Rr, n, 0);  // R = I - A X
  DL_CHECK();
  k_batch_bcsr<<<dim3((PT.nrows + 255) / 256, n), 256, 0, s>>>(PT, Rr, n, Rc, n0, 0);  // Rc = P^T R
  DL_CHECK();
  k_dgemm_nn<<<dim3((n0 + kT - 1) / kT, (n + kT - 1) / kT), 256, 0, s>>>(n0, n, coarse_inv, Rc, E);  // E = C^-1 Rc
  DL_CHECK();
  k_batch_bcsr<<<dim3((Pm.nrows + 255) / 256, n), 256, 0, s>>>(Pm, E, n0, X, n, 1);  // X += P E
  DL_CHECK();
  // X[:, j] = backward sweep(s) of X[:, j] with b = e_j: column j of M1
  small_post_batch(R, A.nb, passes, npass, sweeps, n, 0, X, n, s);
  if (sym) {
    const int nb = (n + kTile - 1) / kTile;
    k_sym_pack<<<int(tri(nb)), 256, 0, s>>>(n, nb, X, M1);
    DL_CHECK();
    return;
  }
  const int ld = dense_level1_ld(n);
  chk(cudaMemsetAsync(M1, 0, sizeof(double) * size_t(n) * ld, s));  // zero columns past n
  k_transpose_sq<<<dim3((n + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, s>>>(n, ld, X, M1);
  DL_CHECK();
}

size_t dense_level1_size(int n, bool sym) {
  if (!sym) return size_t(n) * dense_level1_ld(n);
  const int nb = (n + kTile - 1) / kTile;
  return tri(nb) * (kTile * kTile + 2 * kTile);  // tiles, then the row and column partials
}

void dense_apply(int n, bool sym, const double* M, const double* b, double* y, cudaStream_t s) {
  if (!sym) {
    dense_rowgemv(n, M, b, y, s);
    return;
  }
  const int nb = (n + kTile - 1) / kTile;
  const int nt = int(tri(nb));
  double* prow = const_cast<double*>(M) + size_t(nt) * kTile * kTile;
  double* pcol = prow + size_t(nt) * kTile;
  k_sym_tiles<<<(nt + 1) / 2, 64, 0, s>>>(nt, M, b, prow, pcol);
  DL_CHECK();
  k_sym_combine<<<(4 * n + 255) / 256, 256, 0, s>>>(n, nb, prow, pcol, y);
  DL_CHECK();
}

size_t dense_level1_work(int n, int n0) { return 2 * (size_t(n) * n + size_t(n0) * n); }

int dense_level1_ld(int n) { return (n + kRowPad - 1) / kRowPad * kRowPad; }

void dense_rowgemv(int n, const double* M, const double* b, double* y, cudaStream_t s) {
  k_dense_rowgemv<<<(n + 1) / 2, 256, 0, s>>>(n, dense_level1_ld(n), M, b, y);
  DL_CHECK();
}

}  // namespace dev
}  // namespace hpmg
