// Launch wrappers of the sm_100a FP64 kernels (definitions in kernels.cu).
// All vectors are in the device block layout: block f (free facet) holds
// bs = 2(k+1) doubles [flux_0, tang_0, ..., flux_k, tang_k].
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "condense.cuh"

namespace hpmg {
namespace dev {

constexpr int kSlots = 5;
constexpr int kMaxPatchF = 8;
constexpr int kRedBlocks = 1184;  // 8 x 148 SMs (full occupancy at 256 threads): fixed partial count => deterministic sums

/// Block-sparse operator of one level: nb rows x kSlots fixed-width slots.
struct Bsr {
  int nb = 0, bs = 2;
  double* val = nullptr;  // [nb][kSlots][bs][bs]
  int* cols = nullptr;    // [nb][kSlots], -1 empty
};

/// Vertex patches with explicit inverses (column-major, (nf*bs)^2 each).
struct Patches {
  int n = 0;
  int* nf = nullptr;        // [n]
  int* fac = nullptr;       // [n][kMaxPatchF]
  int64_t* off = nullptr;   // [n]
  double* inv = nullptr;
  int* wave = nullptr;      // patch ids grouped by wave
  int* fpatch = nullptr;    // [nb][2] patches holding block f (ascending)
  int packed = 1;           // 1: symmetric, lower triangle packed by columns
};

/// 2x2-block CSR (prolongation P: fine rows; PT: coarse rows).
struct BlockCsr {
  int nrows = 0, nnz = 0;
  int* ptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;  // [nnzb][2][2] row-major
};

struct Reduce {
  double* partial = nullptr;      // [kRedBlocks]
  unsigned* counter = nullptr;    // zero-initialised ticket
};

/// wind: per-element local wind coefficients [ne][nv] (Oseen / Newton) or
/// nullptr (Stokes); mass_field: same layout, pseudo-time load (prm.mass_coef)
void condense(const RefT& T, const ElemGeo* geo, int ne, CondenseParams prm, const double* load, int load_stride,
              double* out, cudaStream_t s, const double* wind = nullptr, const double* mass_field = nullptr);
/// recover_locals on every element from the full compound skeleton vector
/// (same linearisation state as the condensation).
void recover(const RefT& T, const ElemGeo* geo, int ne, CondenseParams prm, const double* load, int load_stride,
             const int* elem_facets, long long nflux, const double* compound, double* interior, double* pres,
             double* grad, cudaStream_t s, const double* wind = nullptr, const double* mass_field = nullptr);
void assemble_bsr(const Bsr& A, int nfd, const double* acr, int acr_stride, int nc, const int* gath,
                  const ElemGeo* geo, double inv_eps, cudaStream_t s);
void transpose_bsr(const Bsr& A, const int* tslot, Bsr& AT, cudaStream_t s);
void assemble_rhs(int nb, int bs, int nfd, const int* row_elems, const int* block_facet, const int* elem_facets,
                  const char* facet_dirichlet, const double* g_fac, const double* acr, int acr_stride, int nc,
                  const ElemGeo* geo, double inv_eps, double* rhs, cudaStream_t s);

/// y = A x (minus = 0) or y = b - A x (minus = 1); if red != null also
/// reduces dot(x, y) into *dot_out.
void spmv(const Bsr& A, const double* x, const double* b, double* y, int minus, const Reduce* red, double* dot_out,
          cudaStream_t s);
/// A0.val[nb][kSlots][2][bs] = rows 0 and 1 (mode 0) of every block of A
void extract_mode0(const Bsr& A, Bsr& A0, cudaStream_t s);
/// Residual restricted to mode-0 rows, written in lowest-order layout
/// (fused E^T (b - A x), reference multigrid.hpp:123-124); A0 from extract_mode0.
void inject_residual(const Bsr& A0, const double* x, const double* b, double* r0, cudaStream_t s,
                     double* x0_zero = nullptr);  // optionally zeroes x0 (same length as r0)
/// x[f][0..1] += e[f][0..1] (the embedding E, transfer.hpp:140-158).
void embed_add(int nb, int bs, const double* e, double* x, cudaStream_t s);

void patch_inverse(const Bsr& A, const Patches& P, int max_nf, cudaStream_t s);
/// One wave of the multiplicative sweep: x_p += Inv_p (b - A x)_p for the
/// patches wave[w0..w1). transposed_inv selects (Inv_p)^T (nonsymmetric backward).
void gs_wave(const Bsr& A, const Patches& P, int w0, int w1, const double* b, double* x, int transposed_inv,
             int max_nf, cudaStream_t s, const void* prefetch = nullptr, size_t prefetch_len = 0);
/// Fixed-stride per-patch records (sweep_rec.cu): the patch inverse (packed
/// triangle or full), the <= 2 A blocks per patch facet that couple it to
/// facets OUTSIDE the patch, and int32 meta (nf, facets, external columns).
/// The sweep applies x_p = Inv_p (b_p - A_pe x_e), algebraically identical to
/// x_p += Inv_p (b - A x)_p since Inv_p A_pp = I: A_pp is never read.
constexpr int kExt = 2;  // external blocks per patch facet (the two far edges of its triangles)
struct PatchRecords {
  double* rec = nullptr;
  int bs = 2, max_nf = 0;
  int stride = 0, a_off = 0, meta_off = 0;  // in doubles
  int full = 0;  // 1: full np x np column-major inverse instead of the packed triangle
  int rowext = 0;  // 1 (bs = 2, one-CTA levels): external blocks by patch row, [lf][i][slot][col]
  int n = 0;         // patches
  int dbg = 0;       // development: 4 = per-CTA globaltimer trace (sweep_trace)
};
PatchRecords record_layout(int bs, int max_nf, bool full = false);
/// transpose: records of the transposed sweep (A = A^T rows, S_p^T; full layout only)
void build_records(const Bsr& A, const Patches& P, PatchRecords& R, cudaStream_t s, bool transpose = false);
/// One symmetric wave over the patch records [w0, w1) (one TMA per CTA).
/// x_zero: every x_e of the wave is zero (first wave of a sweep from x = 0).
void gs_wave_rec(const PatchRecords& R, int w0, int w1, const double* b, double* x, cudaStream_t s,
                 bool x_zero = false);
void sweep_trace(long long* out);  // development timeline, 5 x 32768 stamps
/// Additive sweep pieces: d_p = Inv_p r_p for all patches; x += damping * sum_p d_p.
void jacobi_patch(const Bsr& A, const Patches& P, const double* r, double* d, int max_nf, cudaStream_t s);
void jacobi_combine(int nb, int bs, const Patches& P, const double* d, int max_nf, double damping, double* x,
                    cudaStream_t s);

/// Small lowest-order levels (small_levels.cu, symmetric): one CTA runs
/// x = 0 and all pre-smoothing waves, then r = b - A x and rc = P^T r run
/// grid-wide (small_pre, 3 launches); x += P e grid-wide, then one CTA runs
/// all post-smoothing waves (small_post, 2 launches).
/// Passes are (first patch, count) ranges of <= small_pass_patches() patches
/// inside one wave, in forward sweep order.
struct PatchRecords;
int small_pass_patches();
void small_trace(int arm, long long* out);
void gm_trace(int arm, long long* out);  // development timeline of the GMRES loop kernels  // development timeline (clock64 per pass phase)
bool small_level_fits(int nb, int record_stride, int npass);
void small_pre(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& PT,
               const double* b, double* x, double* r, double* rc, cudaStream_t s);
void small_post(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& Pm,
                const double* e, const double* b, double* x, cudaStream_t s);
/// batched one-CTA sweeps (setup): CTA j runs the pre (post) phase on column j
/// of X (leading dimension ld) with b = e_{unit0 + j}
void small_pre_batch(const PatchRecords& R, int nb, const int2* passes, int npass, int sweeps, int ncols, int unit0,
                     double* X, int64_t ld, cudaStream_t s);
void small_post_batch(const PatchRecords& R, int nb, const int2* passes, int npass, int sweeps, int ncols, int unit0,
                      double* X, int64_t ld, cudaStream_t s);
/// dense_level.cu: M1 (row-major n x n) = the level-1 V(1,1) sub-cycle
/// (pre-sweep, residual, P C^-1 P^T, post-sweep) as one linear map; y = M b
void dense_level1(const Bsr& A, const PatchRecords& R, const int2* passes, int npass, int sweeps, const BlockCsr& PT,
                  const BlockCsr& Pm, int n0, const double* coarse_inv, double* M1, double* work, bool sym,
                  cudaStream_t s);
/// doubles of M1's storage: full row-major (sym = false) or symmetric tiles + partials
size_t dense_level1_size(int n, bool sym);
/// y = M1 b (b zero-padded past n, see kVecPad)
void dense_apply(int n, bool sym, const double* M, const double* b, double* y, cudaStream_t s);
size_t dense_level1_work(int n, int n0);  // doubles of dense_level1's scratch
/// M row-major with row stride dense_level1_ld(n) (zero columns past n); b
/// must be readable, and zero, up to that stride (level b buffers are padded)
void dense_rowgemv(int n, const double* M, const double* b, double* y, cudaStream_t s);
int dense_level1_ld(int n);
constexpr int kVecPad = 2048;  // doubles of zero padding after every level's b

/// Device arrays of host::TransferPlan (corrected prolongation structure).
struct TransferDev {
  int nelem = 0, nnz = 0;
  int *nmed = nullptr, *med = nullptr, *ncol = nullptr, *col = nullptr, *pos = nullptr;
  int *avg_ptr = nullptr, *avg_col = nullptr;
  double* avg_val = nullptr;
  double* base = nullptr;  // averaging part in the final pattern [nnz][4]
  int* tperm = nullptr;    // PT block d <- P block tperm[d]
};
constexpr int kTransferColMax = 16;
/// P = averaging + harmonic correction -A_TT^{-1} (A I_avg)_T per coarse
/// element (reference transfer.hpp:95-133) from the fine operator A on the
/// device, into P's fixed pattern; PT by the block permutation.
/// T.base = the averaging transfer's blocks in P's final pattern (zero elsewhere); T.avg_* uploaded
void prolong_base(const BlockCsr& P, const TransferDev& T, cudaStream_t s);
void corrected_prolongation(const Bsr& A, const TransferDev& T, BlockCsr& P, BlockCsr& PT, cudaStream_t s);
void prolong_add(const BlockCsr& P, const double* e, double* x, cudaStream_t s);
void restrict_(const BlockCsr& PT, const double* r, double* rc, cudaStream_t s,
               double* xc_zero = nullptr);  // optionally zeroes xc (same length as rc)
void dense_gemv(int n, const double* inv_colmajor, const double* b, double* x, double* work, cudaStream_t s);
/// D (n x n row-major, n = 2 nb) = the lowest-order operator A, zeros elsewhere
void bsr_to_dense(const Bsr& A, double* D, cudaStream_t s);
size_t dense_gemv_work(int n);  // doubles of dense_gemv's partial-sum scratch
/// Gauss-Jordan inverse with partial pivoting of a dense row-major matrix (setup).
void dense_invert(int n, const double* A_rowmajor, double* inv_colmajor, cudaStream_t s);
/// Gauss-Jordan scratch kept by the context (allocated outside any stream work), so the
/// inversion can be queued asynchronously on a side stream and checked later.
struct DenseInvertWork {
  double *aug = nullptr, *rowk = nullptr, *colk = nullptr;
  int* status = nullptr;
  unsigned* ctl = nullptr;
  void* cand = nullptr;
  int* piv = nullptr;
  int n = 0, grid = 0;
  bool coop = false;
};
void dense_invert_alloc(int n, DenseInvertWork& W);
void dense_invert_free(DenseInvertWork& W);
void dense_invert_async(int n, const double* A_rowmajor, double* inv_colmajor, DenseInvertWork& W, cudaStream_t s);
/// synchronises s and throws on a singular matrix
void dense_invert_check(const DenseInvertWork& W, cudaStream_t s);

// vector kernels (n doubles)
void fill(double* x, double v, int64_t n, cudaStream_t s);
void copy(double* y, const double* x, int64_t n, cudaStream_t s);
void axpy(double* y, double a, const double* x, int64_t n, cudaStream_t s);
void sub(double* y, const double* a, const double* b, int64_t n, cudaStream_t s);  // y = a - b
void dot(const double* a, const double* b, int64_t n, const Reduce& red, double* out, cudaStream_t s);
/// *out = ||u||^2_{L2} of the RT field with compound (flux part, reference
/// layout) and interior [ne][no] coefficients (reference assembly.hpp:487-501)
constexpr int kMaxRt = 64;  // 3(k+1) + k(k+1) = 63 at k = 6 (kernels specialise k <= 3 at 24)
void rt_norm2(const RefT& T, const ElemGeo* geo, int ne, const int* elem_facets, const double* compound,
              const double* interior, const Reduce& red, double* out, cudaStream_t s);
/// Post-processing tables of one order (post.cu; reference inc/postprocess.hpp).
/// a, b: reference x / y derivatives of the orthonormal P^{k+1} modes 1..nh-1.
struct PostT {
  int k = 0, nfd = 1, nrt = 3, no = 0, ns = 1, nh = 3;
  const double* Lv = nullptr;  // [2][nrt] sum_q w v^_{r,i} (assembly rule)
  const double* Kh = nullptr;  // [3][nh-1][nh-1] sum_q w a_s a_t, b_s b_t, a_s b_t + b_s a_t
  const double* Bh = nullptr;  // [2][nh-1][ns]   sum_q w a_s s_m, b_s s_m
  double ref_mean = 0.0;       // int_ref P^{k+1} mode 0
  int nqe = 0;                 // error rule (degree 16)
  const double* ex = nullptr;  // [nqe][2] reference points
  const double* ew = nullptr;  // [nqe]
  const double* eval = nullptr;   // [nqe][2][nrt]
  const double* ediv = nullptr;   // [nqe][nrt]
  const double* escal = nullptr;  // [nqe][ns]
  const double* ehi = nullptr;    // [nqe][nh]
};
/// u* in [P^{k+1}]^2 per element (reference postprocess.hpp:24-80): post [ne][2 nh]
/// (x modes then y modes); grad [ne][4 ns] as recover() writes it.
void postprocess(const PostT& P, const ElemGeo* geo, int ne, const int* elem_facets, double nu, const double* compound,
                 const double* interior, const double* grad, double* post, cudaStream_t s);
/// out4 = (e_u, e_L, e_ustar, div_u) (reference postprocess.hpp:140-188) against
/// exact flow `kind` (1 manufactured, 2 linear) or, kind 0, host-tabulated
/// values ue [ne][nqe][2], ge [ne][nqe][4] at the error rule; x0 [ne][2] the
/// element origins; partial [4][kRedBlocks] scratch.
void measure_errors(const PostT& P, const ElemGeo* geo, const double* x0, int ne, const int* elem_facets, double nu,
                    const double* compound, const double* interior, const double* grad, const double* post, int kind,
                    const double* ue, const double* ge, double* partial, double* out4, cudaStream_t s);
/// PCG update: alpha = sc[i_num]/sc[i_den]; x += alpha p; r -= alpha Ap; sc[i_rr] = |r|^2
void pcg_update(double* x, double* r, const double* p, const double* Ap, int64_t n, double* sc, int i_num, int i_den,
                const Reduce& red, int i_rr, cudaStream_t s);
/// p = z + (sc[i_new]/sc[i_old]) p ; then sc[i_old] = sc[i_new]
void pcg_direction(double* p, const double* z, int64_t n, double* sc, int i_new, int i_old, cudaStream_t s);

/// Device-resident Krylov loops: scalar slots of the context's sc[] array
/// (shared with context.cu) and loop states.
enum : int {
  kScRZ = 0, kScRZn = 1, kScPAp = 2, kScRR = 3, kScBB = 4,
  kScIt = 9, kScStatus = 10, kScTarget = 11, kScMaxIt = 12, kScBeta = 13
};
constexpr double kLoopRunning = 0.0, kLoopConverged = 1.0, kLoopNaPAp = 2.0, kLoopNaRZ = 3.0, kLoopMaxIt = 4.0,
                 kLoopLast = 5.0;
void pcg_loop_init(double* sc, double target, double max_it, cudaStream_t s);
/// the update with the count / stop test, r.z with the positivity test and beta
void pcg_loop_update(double* x, double* r, double* p, const double* z, const double* Ap, int64_t n, int dir,
                     double* sc, const Reduce& red, cudaGraphConditionalHandle h_loop, cudaStream_t s);
/// Ap = A p', p'.Ap into sc[kScPAp], p' = z + beta p (dir) or p, p untouched
void pcg_spmv_dir(const Bsr& A, const double* p, const double* z, double* Ap, int dir, double* sc, const Reduce& red,
                  cudaStream_t s);
void pcg_loop_rz(const double* r, const double* z, int64_t n, double* sc, const Reduce& red,
                 cudaGraphConditionalHandle h_loop, cudaStream_t s);
void pcg_loop_direction(double* p, const double* z, int64_t n, const double* sc, cudaStream_t s);
void loop_continue(const double* sc, cudaGraphConditionalHandle h_loop, cudaStream_t s);
void loop_countdown(double* c, cudaGraphConditionalHandle h_loop, cudaStream_t s);

/// Device GMRES state: basis slab V[(cap+1)][ldv], Hessenberg columns
/// H[cap][ldh = cap+1], rotations, g, y, and scalar state st[].
struct GmDev {
  double* V = nullptr;
  int64_t ldv = 0;
  double* H = nullptr;
  int ldh = 0;
  double *cs = nullptr, *sn = nullptr, *g = nullptr, *y = nullptr, *st = nullptr;
  double* part = nullptr;  // [2][kRedBlocks] per-CTA partials of the Gram-Schmidt steps (parity of the step)
};
enum : int { kGmBeta = 0, kGmJ = 1, kGmI = 2, kGmHappy = 3, kGmStalled = 4, kGmHn = 5, kGmCap = 6, kGmM = 7,
             kGmI2 = 8, kGmSlots = 16 };
void gm_init(double* sc, const GmDev& G, double target, double max_it, int cap, cudaStream_t s);
void gm_start(double* sc, const GmDev& G, cudaGraphConditionalHandle h_cyc, cudaGraphConditionalHandle h_inner,
              cudaStream_t s);
/// V[0] = r / beta (and into u, the preconditioner input); arms the MGS loop
void gm_v0(const GmDev& G, const double* r, double* u, int64_t n, cudaGraphConditionalHandle h_mgs, cudaStream_t s);
/// MGS step u (0..7) of a loop body of eight
void mgs_step(const GmDev& G, double* w, int64_t n, int u, cudaGraphConditionalHandle h_mgs, cudaStream_t s);
/// last MGS axpy and the partials of |w|^2
void mgs_tail(const GmDev& G, double* w, int64_t n, cudaStream_t s);
/// h(j+1), the breakdown test, V[j+1] = w / h(j+1) (and into u), then the
/// Givens step and the loop decisions (h_inner; re-arms h_mgs for the next column)
void gm_arnoldi_close(double* sc, const GmDev& G, const double* w, double* u, int64_t n, const Reduce& red,
                      cudaGraphConditionalHandle h_inner, cudaGraphConditionalHandle h_mgs, cudaStream_t s);
void gm_update(const GmDev& G, double* u, int64_t n, cudaStream_t s);
void gm_end(double* sc, const GmDev& G, cudaStream_t s);
/// y = a * x + b * y with device scalars sc[ia] (or 1 if ia < 0), factor fa
void scal_axpby(double* y, const double* x, int64_t n, const double* sc, int ia, double fa, double fb, cudaStream_t s);

// layout permutations between the reference free order and the block layout
void to_blocks(int nb, int nfd, const double* ref, double* blk, cudaStream_t s);
void to_reference(int nb, int nfd, const double* blk, double* ref, cudaStream_t s);
/// to_blocks + zero[0..n) = 0 in one pass (the drop-in apply's first kernel)
void to_blocks_zero(int nb, int nfd, const double* ref, double* blk, double* zero, cudaStream_t s);
/// points the io graph's first (to_blocks_zero) and last (to_reference) kernel nodes at new buffers
void set_io_nodes(cudaGraphExec_t ge, cudaGraphNode_t in_node, cudaGraphNode_t out_node, int nb, int nfd,
                  const double* ref_in, double* blk_in, double* zero, const double* blk_out, double* ref_out);

// augmented-Lagrangian Uzawa pieces (uzawa.hpp:69-82)
void uzawa_rhs(int nb, int bs, const double* rhs0, const int* row_elems, const ElemGeo* geo, const double* p,
               double* rhs, cudaStream_t s);
void uzawa_div(int ne, int bs, const int* elem_facets, const int* facet_block, const double* g_fac, const double* u,
               const ElemGeo* geo, double* div, cudaStream_t s);
void uzawa_pressure(int ne, const double* div, const ElemGeo* geo, double inv_eps, double* p, int enclosed,
                    const Reduce& red, double* sc, int i_s, int i_a, int i_max, cudaStream_t s);

}  // namespace dev
}  // namespace hpmg
