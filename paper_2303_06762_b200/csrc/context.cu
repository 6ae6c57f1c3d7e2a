// hpmg context: owns every device structure of one hp-MG preconditioner and
// implements the C ABI of include/hpmg/capi.h. Setup builds the mesh
// hierarchy and bookkeeping on the host, condenses every level on the GPU,
// inverts the patch blocks on the GPU, builds the CR-GMG transfers on the host
// and uploads them; apply/spmv/pcg/gmres/uzawa run entirely on the device
// (host syncs only to read convergence scalars).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/hpmg/capi.h"
#include "host/basis.hpp"
#include "host/plan.hpp"
#include "host/transfer.hpp"
#include "host/wind.hpp"
#include "kernels/kernels.hpp"

using namespace hpmg;

#define CK(x)                                                                                              \
  do {                                                                                                     \
    cudaError_t e__ = (x);                                                                                 \
    if (e__ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e__)); \
  } while (0)

namespace {

thread_local std::string g_last_error;

inline void dfree(void* p);

/// Owning device buffer for the temporaries of one C-ABI call (freed on every
/// exit path, including a CUDA error thrown half-way).
struct DevTemps {
  std::vector<void*> ptrs;
  DevTemps() = default;
  DevTemps(const DevTemps&) = delete;
  DevTemps& operator=(const DevTemps&) = delete;
  ~DevTemps() {
    for (void* p : ptrs) dfree(p);
  }
  template <typename T>
  T* add(T* p) {
    ptrs.push_back(p);
    return p;
  }
};

/// development: time spent in device allocations / uploads (HPMG_SETUP_TRACE)
inline double& g_alloc_s() {
  static double t = 0;
  return t;
}
inline double& g_upload_s() {
  static double t = 0;
  return t;
}
/// Device allocations come from a process-wide stream-ordered memory pool
/// that keeps freed memory (release threshold = max): a context built after
/// another one was destroyed (NS re-linearisation drivers, repeated setups)
/// reuses the pages instead of paying cudaMalloc's page mapping again.
cudaStream_t alloc_stream() {
  static cudaStream_t q = [] {
    cudaStream_t t;
    CK(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    return t;
  }();
  return q;
}
cudaMemPool_t alloc_pool() {
  static cudaMemPool_t mp = [] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t m;
    CK(cudaMemPoolCreate(&m, &props));
    uint64_t thr = ~uint64_t(0);
    CK(cudaMemPoolSetAttribute(m, cudaMemPoolAttrReleaseThreshold, &thr));
    return m;
  }();
  return mp;
}
/// Frees a dalloc'ed buffer back to the pool once all device work is done.
inline void dfree(void* p) {
  if (!p) return;
  cudaDeviceSynchronize();  // what cudaFree implied: no kernel may still use p
  cudaFreeAsync(p, alloc_stream());
}
template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaMallocFromPoolAsync(&p, n * sizeof(T), alloc_pool(), alloc_stream()));
  CK(cudaStreamSynchronize(alloc_stream()));  // usable from any stream
  g_alloc_s() += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // HPMG_POISON=1: every allocation starts as NaN / -1 bytes (uninitialised-read check)
  static const bool poison = std::getenv("HPMG_POISON") != nullptr;
  if (poison) {
    CK(cudaMemset(p, 0xff, n * sizeof(T)));
    CK(cudaDeviceSynchronize());  // ordered before any non-blocking-stream use
  }
  return static_cast<T*>(p);
}
template <typename T, typename Alloc>
T* dupload(const std::vector<T, Alloc>& v, cudaStream_t s) {
  (void)s;
  T* p = dalloc<T>(v.size());
  const auto t0 = std::chrono::steady_clock::now();
  // on the (otherwise idle) allocation stream: a pageable copy synchronises
  // with its stream first, and on the context stream that meant waiting for
  // every kernel queued before it; the buffer is fresh, so nothing queued
  // there can read it, and the copy is complete when dupload returns
  if (!v.empty()) {
    CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, alloc_stream()));
    CK(cudaStreamSynchronize(alloc_stream()));
  }
  g_upload_s() += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return p;
}

// device scalar slots
enum { S_RZ0 = 0, S_RZ1, S_PAP, S_RR, S_BB, S_TMP, S_PS, S_PA, S_PMAX, S_H0 = 16, S_COUNT = 16 + 520 };

struct DevRef {
  RefT T{};
  std::vector<void*> owned;
};

struct Level {
  host::LevelPlan plan;
  int k = 0, bs = 2, nb = 0;
  int64_t n = 0;
  dev::Bsr A, AT;
  dev::Bsr A0;  // order-k head: the mode-0 rows of A's blocks, contiguous (cols shared with A)
  int* tslot = nullptr;
  dev::Patches P;
  int max_nf = 0;
  std::vector<int> wave_ptr;
  int* d_wave_ptr = nullptr;
  dev::PatchRecords rec;
  dev::PatchRecords srec;  // full-inverse records of the one-CTA path
  dev::PatchRecords rect;  // A^T / S_p^T records of the transposed sweep (advected operators)
  bool small = false;      // whole pre/post phase in one CTA (small_levels.cu)
  int2* d_passes = nullptr;
  int npass = 0;
  dev::BlockCsr Pm, PT;  // from level l-1 to l (lowest-order levels l >= 1)
  dev::TransferDev tdev;  // structure of Pm for its device construction
  double *x = nullptr, *b = nullptr, *r = nullptr, *y = nullptr, *bw = nullptr, *xw = nullptr, *dbuf = nullptr;
  int steps = 1;
  ElemGeo* geo = nullptr;
  bool geo_shared = false;  // the head's geometry is its mesh level's (same mesh): not freed twice
  int ne = 0;
  std::vector<double> Ahost;  // BSR values mirror (filled on demand)
  // finest-system extras
  int* row_elems = nullptr;
  int* elem_facets = nullptr;
  int* facet_block = nullptr;
  int* block_facet = nullptr;
  int* gath = nullptr;  // assembly gather lists (kept for re-linearisation)
  bool finest = false;
  double bytes_sweep = 0, bytes_spmv = 0, p_nnz = 0;
  double bytes_stream = 0;  // one sweep as this implementation moves it: records + b/x rows + x_e gathers
};

}  // namespace

struct hpmg_ctx {
  cudaStream_t s = nullptr;
  std::string err;
  hpmg_options opt{};
  bool advected = false;
  int L = 0;  // finest lowest-order level index
  std::vector<host::TriMesh> mesh;
  std::vector<host::Refinement> ref;
  std::vector<std::unique_ptr<Level>> lv;
  std::unique_ptr<Level> head;  // order-k system (k >= 1)
  DevRef ref0, refk;
  DevRef post;  // post-processing tables (built on first use); post.T unused
  dev::PostT post_t{};
  const double* post_x0 = nullptr;  // finest element origins [ne][2]
  double* post_red = nullptr;       // error partials [4][kRedBlocks] + result [4]
  double* coarse_inv = nullptr;
  double* m1 = nullptr;  // level-1 V(1,1) sub-cycle as one dense map (dense_level.cu), or null
  int m1_n = 0;
  bool m1_sym = true;  // symmetric tile storage (HPMG_DENSE_L1=2: the full row-major map)
  double* coarse_dense = nullptr;  // level-0 operator, dense row-major (setup scratch of the inverse)
  dev::DenseInvertWork gj;         // Gauss-Jordan scratch of the coarse inverse
  cudaStream_t s_coarse = nullptr; // setup: the coarse inverse runs beside the finer levels' work
  double* gemv_work = nullptr;
  int n0 = 0;
  dev::Reduce red;
  double* sc = nullptr;
  double* sc_host = nullptr;  // pinned mirror
  double* rhs = nullptr;      // finest rhs, block layout
  double* g_fac = nullptr;    // finest Dirichlet data per facet (bs each)
  char* facet_dir = nullptr;
  std::vector<double> g_full;  // reference compound order
  std::vector<int64_t> free_to_full;
  // krylov workspace (block layout, finest system)
  double *kx = nullptr, *kb = nullptr, *kr = nullptr, *kz = nullptr, *kp = nullptr, *kAp = nullptr, *ktmp = nullptr;
  double *io_a = nullptr, *io_b = nullptr;  // reference-order staging
  // pipelined batch apply (hpmg_apply_batch): copy streams, double-buffered staging
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  double *bin[2] = {nullptr, nullptr}, *bout[2] = {nullptr, nullptr};
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
              ev_out[2] = {nullptr, nullptr}, ev_start = nullptr;
  std::vector<double*> gm_basis;
  // uzawa
  double *pres = nullptr, *div = nullptr, *urhs = nullptr;
  // finest-system load and condensation parameters (recover_locals)
  double lin_parts[4] = {0, 0, 0, 0};  // last linearisation: patch inverses, transfers, coarse, condensation [s]
  double* acr = nullptr;               // condensed element blocks (scratch of the linearisation)
  size_t acr_cap = 0;
  double* fine_load = nullptr;
  double* fine_wind = nullptr;  // finest-system local wind / mass field (recovery)
  double* fine_mass = nullptr;
  int fine_lstride = 0;
  CondenseParams fine_prm{};
  bool enclosed = true;
  int launches_per_apply = 0;      // kernels of the apply graph (z = M r on block-order kr / kz)
  int io_launches = 0;             // kernels of the drop-in hpmg_apply's io graph
  bool counting = false;
  double setup_parts[8] = {0};
  // CUDA graph of apply(kr -> kz)
  cudaGraphExec_t apply_graph = nullptr;
  // drop-in apply: reference-order input -> blocks (+ x = 0), the cycle,
  // blocks -> reference order, one graph; the end nodes are re-pointed at the
  // caller's device buffers (or the io staging buffers) per call
  cudaGraph_t io_tmpl = nullptr;
  cudaGraphExec_t io_graph = nullptr;
  cudaGraphNode_t io_in = nullptr, io_out = nullptr;
  const double* io_in_cur = nullptr;
  double* io_out_cur = nullptr;
  // MG residual trace (MGOptions::trace, reference multigrid.hpp:18-33): set
  // only during hpmg_apply_trace, which runs the cycle outside the graph
  struct TraceEntry {
    int level, entering;
    double residual;
  };
  std::vector<TraceEntry>* trace = nullptr;
  // device-resident PCG iteration: one graph with a while node (built lazily)
  cudaGraphExec_t pcg_loop = nullptr;
  bool pcg_loop_failed = false;
  cudaStream_t s_nest[4] = {nullptr, nullptr, nullptr, nullptr};  // nested conditional-body captures
  // device-resident GMRES: workspace for `gm_cap` Arnoldi steps per cycle and its loop graph
  dev::GmDev gm;
  int gm_cap = 0, gm_graph_cap = 0;
  cudaGraphExec_t gm_loop = nullptr;
  bool gm_loop_failed = false;

  Level& top() { return opt.k > 0 ? *head : *lv[L]; }
  int64_t nfree() { return top().n; }
};

namespace {

void upload_ref(DevRef& D, const host::RefTensors& T, cudaStream_t s) {
  auto up = [&](const std::vector<double>& v) {
    double* p = dupload(v, s);
    D.owned.push_back(p);
    return p;
  };
  D.T.k = T.k;
  D.T.nfd = T.nfd;
  D.T.nrt = T.nrt;
  D.T.no = T.no;
  D.T.ns = T.ns;
  D.T.nc = T.nc;
  D.T.nv = T.nv;
  D.T.G = up(T.G);
  D.T.Mm = up(T.Mm);
  D.T.Dv = up(T.Dv);
  D.T.Lv = up(T.Lv);
  D.T.Ev = up(T.Ev);
  D.T.Tv = up(T.Tv);
  D.T.vval = up(T.vval);
  D.T.qw = up(T.qw);
  D.T.nq = T.nq;
  D.T.vjac = up(T.vjac);
  D.T.evp = up(T.evp);
  D.T.ew = up(T.ew);
  D.T.eleg = up(T.eleg);
  D.T.nqe = T.nqe;
}

/// Legendre moments of the boundary data on Dirichlet facets, block layout
/// per facet (reference Constraints::build, inc/fespace.hpp:477-515).
std::vector<double> dirichlet_data(const host::TriMesh& m, int k, hpmg_field_fn bc, void* user) {
  const int bs = 2 * (k + 1);
  std::vector<double> g(size_t(m.nf()) * bs, 0.0);
  if (!bc) return g;
  std::vector<double> gx, gw;
  host::gauss(2 * k + 6, gx, gw);
  double L[8], out[2];
  for (int f = 0; f < m.nf(); ++f) {
    if (m.ftag[f] != host::kTagDirichlet) continue;
    double nx, ny, tx, ty;
    m.fnormal(f, nx, ny);
    m.ftan(f, tx, ty);
    for (size_t q = 0; q < gx.size(); ++q) {
      double x, y;
      m.fpoint(f, gx[q], x, y);
      bc(x, y, out, user);
      host::legendre(k, gx[q], L);
      for (int i = 0; i <= k; ++i) {
        const double w = 0.5 * (2 * i + 1) * gw[q] * L[i];
        g[size_t(f) * bs + 2 * i] += w * (out[0] * nx + out[1] * ny);
        g[size_t(f) * bs + 2 * i + 1] += w * (out[0] * tx + out[1] * ty);
      }
    }
  }
  return g;
}

void alloc_level_vectors(Level& V) {
  V.x = dalloc<double>(V.n);
  // zero padding past n: the dense level-1 GEMV reads b up to its row stride
  V.b = dalloc<double>(V.n + dev::kVecPad);
  CK(cudaMemsetAsync(V.b + V.n, 0, sizeof(double) * dev::kVecPad, alloc_stream()));
  CK(cudaStreamSynchronize(alloc_stream()));
  V.r = dalloc<double>(V.n);
  V.y = dalloc<double>(V.n);
  V.bw = dalloc<double>(V.n);
  V.xw = dalloc<double>(V.n);
}

std::vector<int> transpose_slots(const host::LevelPlan& P);

/// Structure of one level: plan (patterns, patches, waves), geometry and every
/// device allocation whose size does not depend on the linearisation state.
/// Development: HPMG_SETUP_TRACE=1 prints setup sub-phase times to stderr.
struct SetupTrace {
  bool on = std::getenv("HPMG_SETUP_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-28s %8.2f ms   (allocs so far %.1f ms, uploads %.1f ms)\n", what,
                 std::chrono::duration<double>(n - t).count() * 1e3, g_alloc_s() * 1e3, g_upload_s() * 1e3);
    t = n;
  }
};

void plan_level(hpmg_ctx& C, Level& V, const host::TriMesh& m, int k, bool finest, host::LevelPlan&& plan,
                ElemGeo* shared_geo = nullptr) {
  cudaStream_t s = C.s;
  V.k = k;
  V.bs = 2 * (k + 1);
  V.finest = finest;
  V.plan = std::move(plan);
  host::set_inverse_layout(V.plan, !C.advected);  // packed symmetric inverses for Stokes
  V.nb = V.plan.nb;
  V.n = V.plan.n();
  V.ne = m.ne();
  if (shared_geo) {  // the order-k head on the finest mesh: the lowest-order level's geometry
    V.geo = shared_geo;
    V.geo_shared = true;
  } else {
    host::BigVec<ElemGeo> geo(m.ne());  // 240 B per element: filled (and first touched) by the plan threads
    host::parallel_for(m.ne(), [&](int e) { geo[e] = host::element_geometry(m, e); });
    V.geo = dupload(geo, s);
  }
  V.A.nb = V.nb;
  V.A.bs = V.bs;
  V.A.val = dalloc<double>(size_t(V.nb) * host::kSlots * V.bs * V.bs);
  V.A.cols = dupload(V.plan.cols, s);
  V.gath = dupload(V.plan.gath, s);
  if (C.advected) {  // A^T rows for the exact transpose (backward) sweeps, multigrid.hpp:84,106
    V.AT = V.A;
    V.AT.val = dalloc<double>(size_t(V.nb) * host::kSlots * V.bs * V.bs);
    V.tslot = dupload(transpose_slots(V.plan), s);
  }
  if (finest) {
    std::vector<int> ef(size_t(m.ne()) * 3);
    for (int e = 0; e < m.ne(); ++e)
      for (int q = 0; q < 3; ++q) ef[size_t(e) * 3 + q] = m.ef[e][q];
    V.elem_facets = dupload(ef, s);
    V.row_elems = dupload(V.plan.row_elems, s);
    V.facet_block = dupload(V.plan.facet_block, s);
    V.block_facet = dupload(V.plan.block_facet, s);
  }
  // patches + explicit inverses
  V.P.n = V.plan.npatch;
  V.max_nf = V.plan.max_patch_f;
  V.P.nf = dupload(V.plan.patch_nf, s);
  V.P.fac = dupload(V.plan.patch_fac, s);
  V.P.off = dupload(V.plan.inv_off, s);
  V.P.inv = dalloc<double>(size_t(V.plan.inv_total));
  V.P.packed = V.plan.packed ? 1 : 0;
  V.P.wave = dupload(V.plan.wave_patch, s);
  V.P.fpatch = dupload(V.plan.facet_patches, s);
  V.wave_ptr = V.plan.wave_ptr;
  V.d_wave_ptr = dupload(V.wave_ptr, s);
  alloc_level_vectors(V);
  V.dbuf = dalloc<double>(size_t(std::max(V.P.n, 1)) * V.max_nf * V.bs);
  // algorithmic bytes, ELL slots counted as stored
  double nnz = 0;
  for (int c : V.plan.cols) nnz += c >= 0 ? double(V.bs) * V.bs : 0.0;
  const double nblk = nnz / (double(V.bs) * V.bs);
  V.bytes_spmv = 8 * nnz + 4 * nblk + 4 * (V.nb + 1.0) + 16.0 * V.n;
  // reference storage accounting: full np^2 patch factors (packing halves the physical bytes)
  V.bytes_sweep = 8.0 * double(V.plan.inv_full_total) + 2 * (8 * nnz + 4 * nblk) + 32.0 * V.n;
}

/// Linearisation-dependent part of one level: condensation about the wind
/// (Oseen / Newton, pseudo-time mass field), assembly into the level's
/// operator arrays in place, A^T, and the finest system's rhs.
void linearise_level(hpmg_ctx& C, Level& V, const host::TriMesh& m, const DevRef& R, const hpmg_problem* prob,
                     double* rhs_out, const host::HdgField* wind = nullptr) {
  cudaStream_t s = C.s;
  const int k = V.k;
  const bool finest = V.finest;
  const int nc = R.T.nc, stride = nc * nc + nc;
  // condensed element blocks: one persistent scratch sized for the largest level
  const size_t need = size_t(m.ne()) * stride;
  if (C.acr_cap < need) {
    if (C.acr) dfree(C.acr);
    C.acr = dalloc<double>(need);
    C.acr_cap = need;
  }
  double* acr = C.acr;
  CondenseParams prm{C.opt.nu, C.opt.beta + C.opt.mass_coef, 0, (prob && prob->newton) ? 1 : 0, C.opt.mass_coef};
  double* dload = nullptr;
  int lstride = 0;
  if (finest && prob) {
    if (prob->structured_load) {
      // seeded per-triangle force on an n x n grid: cell from the centroid,
      // lower triangle (v00, v10, v11) iff (x - i/n) >= (y - j/n) (mesh.hpp:231-232)
      const int sn = prob->structured_n;
      std::vector<double> l(size_t(2) * m.ne());
      for (int e = 0; e < m.ne(); ++e) {
        const auto& v = m.ev[e];
        const double cx = (m.vx[v[0]] + m.vx[v[1]] + m.vx[v[2]]) / 3.0;
        const double cy = (m.vy[v[0]] + m.vy[v[1]] + m.vy[v[2]]) / 3.0;
        const int i = std::min(sn - 1, std::max(0, int(std::floor(cx * sn))));
        const int j = std::min(sn - 1, std::max(0, int(std::floor(cy * sn))));
        const bool lower = (cx - double(i) / sn) >= (cy - double(j) / sn);
        const size_t sidx = (size_t(j) * sn + i) * 2 + (lower ? 0 : 1);
        l[2 * e] = prob->structured_load[2 * sidx];
        l[2 * e + 1] = prob->structured_load[2 * sidx + 1];
      }
      dload = dupload(l, s);
      prm.load_mode = 1;
      lstride = 2;
    } else if (prob->load_per_element) {
      std::vector<double> l(prob->load_per_element, prob->load_per_element + size_t(2) * m.ne());
      dload = dupload(l, s);
      prm.load_mode = 1;
      lstride = 2;
    } else if (prob->load) {
      // pointwise: evaluate the callback at the mapped volume nodes on the host
      const int nq = R.T.nq;
      std::vector<double> qx, qy, qw;
      host::duffy(3 * k + 4, qx, qy, qw);
      std::vector<double> l(size_t(m.ne()) * nq * 2);
      double out[2];
      for (int e = 0; e < m.ne(); ++e) {
        const ElemGeo g = host::element_geometry(m, e);
        const double x0 = m.vx[m.ev[e][0]], y0 = m.vy[m.ev[e][0]];
        for (int q = 0; q < nq; ++q) {
          const double x = x0 + g.J[0] * qx[q] + g.J[1] * qy[q], y = y0 + g.J[2] * qx[q] + g.J[3] * qy[q];
          prob->load(x, y, out, prob->load_user);
          l[(size_t(e) * nq + q) * 2] = out[0];
          l[(size_t(e) * nq + q) * 2 + 1] = out[1];
        }
      }
      dload = dupload(l, s);
      prm.load_mode = 2;
      lstride = 2 * nq;
    }
  }
  double* dwind = nullptr;
  if (wind) dwind = dupload(host::local_wind(m, k, *wind), s);
  double* dmass = nullptr;  // pseudo-time mass field: a load, so on the finest system only
  if (finest && prob && prob->mass_compound) {
    host::HdgField mf;
    mf.k = k;
    mf.compound.assign(prob->mass_compound, prob->mass_compound + C.g_full.size());
    const size_t ni = size_t(m.ne()) * k * (k + 1);
    if (ni) mf.interior.assign(prob->mass_interior, prob->mass_interior + ni);
    dmass = dupload(host::local_wind(m, k, mf), s);
  }
  dev::condense(R.T, V.geo, m.ne(), prm, dload, lstride, acr, s, dwind, dmass);
  dev::assemble_bsr(V.A, k + 1, acr, stride, nc, V.gath, V.geo, C.opt.inv_eps, s);
  if (C.advected) dev::transpose_bsr(V.A, V.tslot, V.AT, s);
  if (k > 0) {  // the head residual's rows, streamed contiguously
    if (!V.A0.val) V.A0.val = dalloc<double>(size_t(V.nb) * host::kSlots * 2 * V.bs);
    V.A0.nb = V.A.nb;
    V.A0.bs = V.A.bs;
    V.A0.cols = V.A.cols;
    dev::extract_mode0(V.A, V.A0, s);
  }
  if (finest)
    dev::assemble_rhs(V.nb, V.bs, k + 1, V.row_elems, V.block_facet, V.elem_facets, C.facet_dir, C.g_fac, acr,
                      stride, nc, V.geo, C.opt.inv_eps, rhs_out, s);
  // no stream synchronisation here: the next level's kernels queue behind
  // these on the same stream; dfree synchronises before releasing a buffer
  if (finest) {  // kept for recover_locals (same linearisation state)
    for (void* p : {(void*)C.fine_load, (void*)C.fine_wind, (void*)C.fine_mass})
      if (p) dfree(p);
    C.fine_wind = dwind;
    C.fine_mass = dmass;
    C.fine_load = dload;
    C.fine_lstride = lstride;
    C.fine_prm = prm;
  } else {
    if (dwind) dfree(dwind);
    if (dload) dfree(dload);
  }
}

void build_patch_inverses(hpmg_ctx& C, Level& V) {
  if (V.P.n == 0) return;
  dev::patch_inverse(V.A, V.P, V.max_nf, C.s);
  // fixed-stride patch records for the TMA sweep (sweep_rec.cu); nonsymmetric
  // operators: full inverses, plus A^T / S_p^T records for the transposed sweep
  // (hpmg_options.sweep_variant = HPMG_SWEEP_DIRECT_NONSYM: the direct-gather
  // correction sweeps of kernels.cu instead)
  const bool nonsym_records = C.opt.sweep_variant != HPMG_SWEEP_DIRECT_NONSYM;
  bool use_records = V.P.packed || nonsym_records;
  if (use_records && !V.P.packed && !V.rec.rec) {
    // nonsymmetric records hold full inverses twice (S_p and S_p^T sets, ~5x the
    // packed footprint at k = 3): where they do not fit next to a safety margin,
    // stay on the direct-gather sweeps (same results) instead of failing setup
    const dev::PatchRecords lay = dev::record_layout(V.bs, V.max_nf, true);
    const double need = 8.0 * double(V.P.n) * double(lay.stride) * (C.advected ? 2.0 : 1.0);
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (need + 0.05 * double(total_b) > double(free_b)) use_records = false;
  }
  if (use_records) {
    // every patch facet couples to at most kExt facets outside the patch (triangle meshes)
    double vec_bytes = 0;
    for (int p = 0; p < V.P.n; ++p)
      for (int lf = 0; lf < V.plan.patch_nf[p]; ++lf) {
        const int f = V.plan.patch_fac[size_t(p) * dev::kMaxPatchF + lf];
        int ne = 0;
        for (int sl = 0; sl < host::kSlots; ++sl) {
          const int c = V.plan.cols[size_t(f) * host::kSlots + sl];
          bool inside = false;
          for (int q = 0; q < V.plan.patch_nf[p]; ++q) inside |= V.plan.patch_fac[size_t(p) * dev::kMaxPatchF + q] == c;
          ne += (c >= 0 && !inside) ? 1 : 0;
        }
        if (ne > dev::kExt) throw std::runtime_error("patch facet with more than 2 external couplings");
        vec_bytes += 8.0 * V.bs * (2 + ne);  // b row read, x row written, x_e blocks gathered
      }
    if (V.rec.rec) {  // re-linearisation: same layout, rebuild the record contents in place
      dev::build_records(V.A, V.P, V.rec, C.s);
      if (V.rect.rec) dev::build_records(V.AT, V.P, V.rect, C.s, true);
      if (V.small) dev::build_records(V.A, V.P, V.srec, C.s);
      return;
    }
    V.rec = dev::record_layout(V.bs, V.max_nf, !V.P.packed);
    V.rec.rec = dalloc<double>(size_t(V.P.n) * V.rec.stride);
    if (C.advected) {
      V.rect = V.rec;
      V.rect.rec = dalloc<double>(size_t(V.P.n) * V.rect.stride);
      dev::build_records(V.AT, V.P, V.rect, C.s, true);
    }
    V.rec.n = V.P.n;
    if (const char* d = std::getenv("HPMG_DBG")) V.rec.dbg = std::atoi(d);
    dev::build_records(V.A, V.P, V.rec, C.s);
    std::vector<int2> passes;
    const int pp = dev::small_pass_patches();
    for (size_t w = 0; w + 1 < V.wave_ptr.size(); ++w)
      for (int a = V.wave_ptr[w]; a < V.wave_ptr[w + 1]; a += pp)
        passes.push_back(make_int2(a, std::min(pp, V.wave_ptr[w + 1] - a)));
    // one-CTA path only where the wave count (not the width) dominates: level 1
    // of a coarse base mesh (26 / 50 waves); refined levels have 9 wide waves
    const int nwaves = int(V.wave_ptr.size()) - 1;
    const dev::PatchRecords full = dev::record_layout(V.bs, V.max_nf, true);
    if (V.P.packed && V.k == 0 && nwaves > 12 && dev::small_level_fits(V.nb, full.stride, int(passes.size()))) {
      V.srec = full;
      V.srec.rowext = 1;
      V.srec.rec = dalloc<double>(size_t(V.P.n) * V.srec.stride);
      dev::build_records(V.A, V.P, V.srec, C.s);
      V.npass = int(passes.size());
      V.d_passes = dupload(passes, C.s);
      V.small = true;
    }
    V.bytes_stream = 8.0 * double(V.P.n) * (V.small ? V.srec.stride : V.rec.stride) + vec_bytes;
  }
}

/// transposed-slot map for A^T in the same ELL pattern (A's pattern is symmetric)
std::vector<int> transpose_slots(const host::LevelPlan& P) {
  std::vector<int> t(P.cols.size(), -1);
  for (int r = 0; r < P.nb; ++r)
    for (int s = 0; s < host::kSlots; ++s) {
      const int c = P.cols[size_t(r) * host::kSlots + s];
      if (c < 0) continue;
      for (int s2 = 0; s2 < host::kSlots; ++s2)
        if (P.cols[size_t(c) * host::kSlots + s2] == r) t[size_t(r) * host::kSlots + s] = s2;
    }
  return t;
}

std::vector<double> download_bsr(hpmg_ctx& C, Level& V) {
  std::vector<double> h(size_t(V.nb) * host::kSlots * V.bs * V.bs);
  CK(cudaMemcpyAsync(h.data(), V.A.val, h.size() * sizeof(double), cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
  return h;
}

/// Block CSR to the device; values uploaded only when `values` (the
/// prolongation's are formed on the device from the averaging base, the
/// restriction's by the block transpose: their host arrays are not sent).
dev::BlockCsr upload_blockcsr(const host::BlockCsrH& H, cudaStream_t s, bool values = true) {
  dev::BlockCsr D;
  D.nrows = H.nrows;
  D.ptr = dupload(H.ptr, s);
  D.col = dupload(H.col, s);
  D.val = values ? dupload(H.val, s) : dalloc<double>(H.col.size() * 4);
  return D;
}

// ------------------------------------------------------------------ cycle
void count(hpmg_ctx& C, int n = 1) {
  if (C.counting) C.launches_per_apply += n;
}

/// x_zero: x = 0 on entry (pre-smoothing inside the cycle): the first wave
/// of the first sweep sees x_e = 0 (and the transposed post sweep's first
/// wave y_e = 0), which gs_wave_rec exploits bitwise-exactly.
void smooth(hpmg_ctx& C, Level& V, double* x, const double* b, bool post, bool x_zero = false) {
  const int nw = int(V.wave_ptr.size()) - 1;
  if (C.opt.smoother == HPMG_SMOOTH_ADDITIVE) {
    for (int s = 0; s < V.steps; ++s) {
      dev::spmv(V.A, x, b, V.r, 1, nullptr, nullptr, C.s);
      dev::jacobi_patch(V.A, V.P, V.r, V.dbuf, V.max_nf, C.s);
      dev::jacobi_combine(V.nb, V.bs, V.P, V.dbuf, V.max_nf, C.opt.jacobi_damping, x, C.s);
      count(C, 3);
    }
    return;
  }
  // L2 prefetch of the next wave's patch inverses (contiguous: patches are numbered in wave order)
  auto next_inv = [&](int w, const void** ptr, size_t* len) {
    *ptr = nullptr;
    *len = 0;
    if (w < 0 || w >= nw || !V.P.packed) return;
    const int64_t a = V.plan.inv_off[V.wave_ptr[w]];
    const int64_t e = V.wave_ptr[w + 1] < V.P.n ? V.plan.inv_off[V.wave_ptr[w + 1]] : V.plan.inv_total;
    const uintptr_t beg = reinterpret_cast<uintptr_t>(V.P.inv + a) & ~uintptr_t(15);
    *ptr = reinterpret_cast<const void*>(beg);
    *len = size_t(reinterpret_cast<uintptr_t>(V.P.inv + e) - beg);
  };
  const void* pf;
  size_t pl;
  if (!post) {
    for (int s = 0; s < V.steps; ++s)
      for (int w = 0; w < nw; ++w) {
        if (V.rec.rec) {
          dev::gs_wave_rec(V.rec, V.wave_ptr[w], V.wave_ptr[w + 1], b, x, C.s, x_zero && s == 0 && w == 0);
        } else {
          next_inv(w + 1 < nw ? w + 1 : (s + 1 < V.steps ? 0 : -1), &pf, &pl);
          dev::gs_wave(V.A, V.P, V.wave_ptr[w], V.wave_ptr[w + 1], b, x, 0, V.max_nf, C.s, pf, pl);
        }
        count(C);
      }
    return;
  }
  if (!C.advected) {
    // symmetric: the exact transpose sweep is the reverse-order sweep on x itself
    for (int s = 0; s < V.steps; ++s)
      for (int w = nw - 1; w >= 0; --w) {
        if (V.P.packed) {
          dev::gs_wave_rec(V.rec, V.wave_ptr[w], V.wave_ptr[w + 1], b, x, C.s);
        } else {
          next_inv(w - 1 >= 0 ? w - 1 : (s + 1 < V.steps ? nw - 1 : -1), &pf, &pl);
          dev::gs_wave(V.A, V.P, V.wave_ptr[w], V.wave_ptr[w + 1], b, x, 0, V.max_nf, C.s, pf, pl);
        }
        count(C);
      }
    return;
  }
  // nonsymmetric: c = b - A x, y = 0, transposed sweep on y with A^T rows, x += y
  dev::spmv(V.A, x, b, V.r, 1, nullptr, nullptr, C.s);
  dev::fill(V.y, 0.0, V.n, C.s);
  count(C, 2);
  for (int s = 0; s < V.steps; ++s)
    for (int w = nw - 1; w >= 0; --w) {
      if (V.rect.rec)
        dev::gs_wave_rec(V.rect, V.wave_ptr[w], V.wave_ptr[w + 1], V.r, V.y, C.s, s == 0 && w == nw - 1);
      else
        dev::gs_wave(V.AT, V.P, V.wave_ptr[w], V.wave_ptr[w + 1], V.r, V.y, 1, V.max_nf, C.s);
      count(C);
    }
  dev::axpy(x, 1.0, V.y, V.n, C.s);
  count(C);
}

void read_scalars(hpmg_ctx& C, int n = 16);

/// Trace entries: |b| on entering a level, |b - A x| on leaving it (the
/// reference's MGTraceEntry, multigrid.hpp:120,126,168-183). Synchronous;
/// only hpmg_apply_trace sets C.trace.
void trace_norm(hpmg_ctx& C, int level, bool entering, const double* v, int64_t n) {
  dev::dot(v, v, n, C.red, C.sc + S_TMP, C.s);
  read_scalars(C, 16);
  C.trace->push_back({level, entering ? 1 : 0, std::sqrt(C.sc_host[S_TMP])});
}
void trace_residual(hpmg_ctx& C, int level, const Level& V, const double* b, const double* x, double* scratch) {
  dev::spmv(V.A, x, b, scratch, 1, nullptr, nullptr, C.s);
  trace_norm(C, level, false, scratch, V.n);
}

/// h_cycle(l, b) -> x (reference inc/multigrid.hpp:166-185)
void h_cycle(hpmg_ctx& C, int l, const double* b, double* x) {
  if (C.trace) trace_norm(C, l, true, b, C.lv[l]->n);
  if (l == 0) {
    dev::dense_gemv(C.n0, C.coarse_inv, b, x, C.gemv_work, C.s);
    count(C);
    if (C.trace) trace_residual(C, 0, *C.lv[0], b, x, C.lv[0]->y);  // y: no smoother on level 0; bw may be b (W-cycle)
    return;
  }
  Level& V = *C.lv[l];
  Level& W = *C.lv[l - 1];
  const int q = C.opt.cycle == HPMG_CYCLE_W ? 2 : 1;
  if (l == 1 && C.m1 && b == V.b && !C.trace && V.small && C.opt.smoother == HPMG_SMOOTH_MULTIPLICATIVE && q == 1) {
    // the whole level-1 sub-cycle (sweeps, transfers, coarse solve) as one
    // dense map formed at setup (dense_level.cu): one HBM-bound GEMV
    dev::dense_apply(int(V.n), C.m1_sym, C.m1, b, x, C.s);
    count(C);
    return;
  }
  if (V.small && C.opt.smoother == HPMG_SMOOTH_MULTIPLICATIVE && q == 1) {
    // whole-level sweeps in one persistent CTA (small_levels.cu)
    dev::small_pre(V.A, V.srec, V.d_passes, V.npass, V.steps, V.PT, b, x, V.r, W.b, C.s);
    count(C, 3);
    h_cycle(C, l - 1, W.b, W.x);
    dev::small_post(V.A, V.srec, V.d_passes, V.npass, V.steps, V.Pm, W.x, b, x, C.s);
    count(C, 2);
    if (C.trace) trace_residual(C, l, V, b, x, V.r);
    return;
  }
  // x = 0 was written by the kernel that produced b (restriction / E^T injection)
  smooth(C, V, x, b, false, true);
  dev::spmv(V.A, x, b, V.r, 1, nullptr, nullptr, C.s);
  dev::restrict_(V.PT, V.r, W.b, C.s, l - 1 > 0 ? W.x : nullptr);
  count(C, 2);
  h_cycle(C, l - 1, W.b, W.x);
  for (int i = 1; i < q; ++i) {
    dev::spmv(W.A, W.x, W.b, W.bw, 1, nullptr, nullptr, C.s);
    count(C);
    if (l - 1 > 0) {  // h_cycle expects x = 0 on entry
      dev::fill(W.xw, 0.0, W.n, C.s);
      count(C);
    }
    h_cycle(C, l - 1, W.bw, W.xw);
    dev::axpy(W.x, 1.0, W.xw, W.n, C.s);
    count(C);
  }
  dev::prolong_add(V.Pm, W.x, x, C.s);
  count(C);
  smooth(C, V, x, b, true);
  if (C.trace) trace_residual(C, l, V, b, x, V.r);
}

/// apply(b) -> x on the finest system, block layout (inc/multigrid.hpp:117-128)
void apply_blocks(hpmg_ctx& C, const double* b, double* x, bool x_zeroed = false) {
  if (C.opt.k == 0) {
    if (!x_zeroed && C.L > 0 && !(C.lv[C.L]->small && C.opt.smoother == HPMG_SMOOTH_MULTIPLICATIVE &&
                                  C.opt.cycle != HPMG_CYCLE_W)) {
      dev::fill(x, 0.0, C.lv[C.L]->n, C.s);  // h_cycle expects x = 0 on entry (restriction zeroes it below)
      count(C);
    }
    h_cycle(C, C.L, b, x);
    return;
  }
  Level& H = *C.head;
  Level& F = *C.lv[C.L];
  if (C.trace) trace_norm(C, C.L + 1, true, b, H.n);  // the head is reported one index above the finest mesh level
  if (!x_zeroed) {
    dev::fill(x, 0.0, H.n, C.s);
    count(C);
  }
  smooth(C, H, x, b, false, true);
  dev::inject_residual(H.A0, x, b, F.b, C.s, F.x);
  count(C);
  h_cycle(C, C.L, F.b, F.x);
  dev::embed_add(H.nb, H.bs, F.x, x, C.s);
  count(C);
  smooth(C, H, x, b, true);
  if (C.trace) trace_residual(C, C.L + 1, H, b, x, C.ktmp);
}

void build_apply_graph(hpmg_ctx& C) {
  cudaGraph_t g;
  C.launches_per_apply = 0;
  C.counting = true;
  CK(cudaStreamBeginCapture(C.s, cudaStreamCaptureModeThreadLocal));
  apply_blocks(C, C.kr, C.kz);
  CK(cudaStreamEndCapture(C.s, &g));
  C.counting = false;
  CK(cudaGraphInstantiate(&C.apply_graph, g, 0));
  cudaGraphDestroy(g);
}

void apply_graph(hpmg_ctx& C) { CK(cudaGraphLaunch(C.apply_graph, C.s)); }

/// the node the last captured launch on s created
cudaGraphNode_t last_captured(cudaStream_t s) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &ndeps));
  if (ndeps != 1) throw std::runtime_error("io graph: unexpected capture fan-in");
  return deps[0];
}

void destroy_io_graph(hpmg_ctx& C) {
  if (C.io_graph) cudaGraphExecDestroy(C.io_graph);
  if (C.io_tmpl) cudaGraphDestroy(C.io_tmpl);
  C.io_graph = nullptr;
  C.io_tmpl = nullptr;
  C.io_in = C.io_out = nullptr;
  C.io_in_cur = nullptr;
  C.io_out_cur = nullptr;
}

void build_io_graph(hpmg_ctx& C) {
  Level& T = C.top();
  CK(cudaStreamBeginCapture(C.s, cudaStreamCaptureModeThreadLocal));
  try {
    dev::to_blocks_zero(T.nb, T.k + 1, C.io_a, C.kr, C.kz, C.s);
    C.io_in = last_captured(C.s);
    apply_blocks(C, C.kr, C.kz, true);
    dev::to_reference(T.nb, T.k + 1, C.kz, C.io_b, C.s);
    C.io_out = last_captured(C.s);
  } catch (...) {
    cudaGraph_t tmp;
    cudaStreamEndCapture(C.s, &tmp);
    if (tmp) cudaGraphDestroy(tmp);
    throw;
  }
  CK(cudaStreamEndCapture(C.s, &C.io_tmpl));
  CK(cudaGraphInstantiate(&C.io_graph, C.io_tmpl, 0));
  size_t nn = 0;
  CK(cudaGraphGetNodes(C.io_tmpl, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CK(cudaGraphGetNodes(C.io_tmpl, nodes.data(), &nn));
  C.io_launches = 0;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    CK(cudaGraphNodeGetType(nd, &ty));
    C.io_launches += ty == cudaGraphNodeTypeKernel;
  }
  C.io_in_cur = C.io_a;
  C.io_out_cur = C.io_b;
}

/// z = M r through the io graph; r / z on the device (stream-ordered) or the
/// io staging buffers after / before the host copies
void apply_io(hpmg_ctx& C, const double* r_dev, double* z_dev) {
  if (!C.io_graph) build_io_graph(C);
  if (r_dev != C.io_in_cur || z_dev != C.io_out_cur) {
    Level& T = C.top();
    dev::set_io_nodes(C.io_graph, C.io_in, C.io_out, T.nb, T.k + 1, r_dev, C.kr, C.kz, C.kz, z_dev);
    C.io_in_cur = r_dev;
    C.io_out_cur = z_dev;
  }
  CK(cudaGraphLaunch(C.io_graph, C.s));
}

void read_scalars(hpmg_ctx& C, int n) {
  CK(cudaMemcpyAsync(C.sc_host, C.sc, sizeof(double) * n, cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
}

// ---------------------------------------------------------------- boundary
void in_vec(hpmg_ctx& C, const double* src, double* dst_blk, int flags) {
  Level& T = C.top();
  const double* ref = src;
  if (!(flags & HPMG_DEVICE_PTRS)) {
    CK(cudaMemcpyAsync(C.io_a, src, sizeof(double) * T.n, cudaMemcpyHostToDevice, C.s));
    ref = C.io_a;
  }
  dev::to_blocks(T.nb, T.k + 1, ref, dst_blk, C.s);
}
void out_vec(hpmg_ctx& C, const double* src_blk, double* dst, int flags) {
  Level& T = C.top();
  if (flags & HPMG_DEVICE_PTRS) {  // stream-ordered: the caller synchronises hpmg_stream(ctx) as needed
    dev::to_reference(T.nb, T.k + 1, src_blk, dst, C.s);
    return;
  }
  dev::to_reference(T.nb, T.k + 1, src_blk, C.io_b, C.s);
  CK(cudaMemcpyAsync(dst, C.io_b, sizeof(double) * T.n, cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
}

// ---------------------------------------------------------------- solvers
// ------------------------------------------------ conditional-graph capture
struct GraphError {
  cudaError_t e;
};
inline void GK(cudaError_t e) {
  if (e != cudaSuccess) throw GraphError{e};
}
/// Appends a conditional node after the work captured so far on `s`; later
/// captured work depends on it. Returns the node's body graph.
cudaGraph_t add_conditional(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t capg;
  GK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &capg, &deps, &ndeps));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  GK(cudaGraphAddNode(&node, capg, deps, ndeps, &p));
  GK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  return p.conditional.phGraph_out[0];
}
/// Captures fn() into `body` on nesting stream `depth`, with C.s pointing at
/// that stream meanwhile (the V-cycle helpers launch on C.s).
template <class F>
void capture_body(hpmg_ctx& C, cudaGraph_t body, int depth, F fn) {
  if (!C.s_nest[depth]) GK(cudaStreamCreateWithFlags(&C.s_nest[depth], cudaStreamNonBlocking));
  cudaStream_t q = C.s_nest[depth], saved = C.s;
  GK(cudaStreamBeginCaptureToGraph(q, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  C.s = q;
  try {
    fn();
  } catch (...) {
    C.s = saved;
    cudaGraph_t tmp;
    cudaStreamEndCapture(q, &tmp);
    throw;
  }
  C.s = saved;
  cudaGraph_t tmp;
  GK(cudaStreamEndCapture(q, &tmp));
}

/// The PCG iterations (reference krylov.hpp:44-70) as one CUDA graph with no
/// host round trip: the first iteration's
///   Ap = A p, p.Ap | x += a p, r -= a Ap, r.r, count, stop test
/// then a while node whose body is
///   z = M r (the V-cycle launch sequence) | r.z, positivity test, beta
///   | Ap = A p' with p' = z + beta p formed on the fly, p'.Ap
///   | p = p', x += a p, r -= a Ap, r.r, count, stop test.
/// The loop predicate is set on the device (cudaGraphSetConditional) by the
/// kernel that decides to stop; the kernels after it in the same body are
/// no-ops then. No if node: the V-cycle sits directly in the loop body.
/// Returns false (and the host loop is used) where the driver cannot build it.
bool build_pcg_loop(hpmg_ctx& C) {
  Level& T = C.top();
  const int64_t n = T.n;
  cudaGraph_t g = nullptr;
  try {
    GK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop;
    GK(cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault));
    capture_body(C, g, 0, [&] {
      dev::pcg_spmv_dir(T.A, C.kp, C.kz, C.kAp, 0, C.sc, C.red, C.s);  // p = z0 (pcg_device)
      dev::pcg_loop_update(C.kx, C.kr, C.kp, C.kz, C.kAp, n, 0, C.sc, C.red, h_loop, C.s);
      cudaGraph_t body = add_conditional(C.s, h_loop, cudaGraphCondTypeWhile);
      capture_body(C, body, 1, [&] {
        apply_blocks(C, C.kr, C.kz);  // z = M r
        dev::pcg_loop_rz(C.kr, C.kz, n, C.sc, C.red, h_loop, C.s);
        dev::pcg_spmv_dir(T.A, C.kp, C.kz, C.kAp, 1, C.sc, C.red, C.s);
        dev::pcg_loop_update(C.kx, C.kr, C.kp, C.kz, C.kAp, n, 1, C.sc, C.red, h_loop, C.s);
      });
    });
    GK(cudaGraphInstantiate(&C.pcg_loop, g, 0));
  } catch (const GraphError& e) {
    if (g) cudaGraphDestroy(g);
    C.pcg_loop = nullptr;
    cudaGetLastError();
    if (std::getenv("HPMG_DEBUG_GRAPH")) std::fprintf(stderr, "pcg loop graph: %s\n", cudaGetErrorString(e.e));
    return false;
  } catch (const std::exception& e) {
    if (g) cudaGraphDestroy(g);
    C.pcg_loop = nullptr;
    cudaGetLastError();
    if (std::getenv("HPMG_DEBUG_GRAPH")) std::fprintf(stderr, "pcg loop graph: %s\n", e.what());
    return false;
  }
  cudaGraphDestroy(g);
  return true;
}

/// PCG on the device (reference inc/krylov.hpp:30-73); x/b in kx/kb. The
/// setup (r0, z0, r0.z0) syncs twice per solve; the iterations run as one
/// graph launch (build_pcg_loop) unless HPMG_KRYLOV_HOST=1 or the graph is
/// unavailable, where a host loop with two syncs per iteration does the same
/// arithmetic in the same order.
hpmg_solve_stats pcg_device(hpmg_ctx& C, const hpmg_krylov_opts& o) {
  hpmg_solve_stats st{0, 0, 0, 0.0};
  Level& T = C.top();
  const int64_t n = T.n;
  dev::dot(C.kb, C.kb, n, C.red, C.sc + S_BB, C.s);
  dev::spmv(T.A, C.kx, C.kb, C.kr, 1, nullptr, nullptr, C.s);
  dev::dot(C.kr, C.kr, n, C.red, C.sc + S_RR, C.s);
  read_scalars(C);
  const double target = std::max(o.rel_tol * std::sqrt(C.sc_host[S_BB]), o.abs_tol);
  st.residual = std::sqrt(C.sc_host[S_RR]);
  if (st.residual <= target) {
    st.converged = 1;
    return st;
  }
  apply_graph(C);  // kz = M kr
  int cur = S_RZ0, nxt = S_RZ1;
  dev::dot(C.kr, C.kz, n, C.red, C.sc + cur, C.s);
  read_scalars(C);
  if (!(C.sc_host[cur] > 0)) {
    st.not_applicable = 1;
    return st;
  }
  dev::copy(C.kp, C.kz, n, C.s);
  if (o.max_iterations <= 0) return st;
  static const bool host_loop = std::getenv("HPMG_KRYLOV_HOST") && std::atoi(std::getenv("HPMG_KRYLOV_HOST"));
  if (!host_loop && !C.pcg_loop && !C.pcg_loop_failed) C.pcg_loop_failed = !build_pcg_loop(C);
  if (!host_loop && C.pcg_loop) {
    dev::pcg_loop_init(C.sc, target, double(o.max_iterations), C.s);
    CK(cudaGraphLaunch(C.pcg_loop, C.s));
    read_scalars(C);
    const double status = C.sc_host[dev::kScStatus];
    st.iterations = int(C.sc_host[dev::kScIt]);
    st.residual = std::sqrt(C.sc_host[S_RR]);
    st.converged = status == dev::kLoopConverged;
    st.not_applicable = status == dev::kLoopNaPAp || status == dev::kLoopNaRZ;
    return st;
  }
  for (int it = 0; it < o.max_iterations; ++it) {
    dev::spmv(T.A, C.kp, nullptr, C.kAp, 0, &C.red, C.sc + S_PAP, C.s);
    dev::pcg_update(C.kx, C.kr, C.kp, C.kAp, n, C.sc, cur, S_PAP, C.red, S_RR, C.s);
    read_scalars(C);
    if (!(C.sc_host[S_PAP] > 0)) {  // pcg_update skipped x and r on the device
      st.not_applicable = 1;
      return st;
    }
    st.iterations = it + 1;
    st.residual = std::sqrt(C.sc_host[S_RR]);
    if (st.residual <= target) {
      st.converged = 1;
      return st;
    }
    apply_graph(C);
    dev::dot(C.kr, C.kz, n, C.red, C.sc + nxt, C.s);
    read_scalars(C);
    if (!(C.sc_host[nxt] > 0)) {
      st.not_applicable = 1;
      return st;
    }
    dev::pcg_direction(C.kp, C.kz, n, C.sc, nxt, cur, C.s);
    std::swap(cur, nxt);
  }
  return st;
}


/// GMRES workspace for `cap` Arnoldi steps per cycle (grows only).
void gm_workspace(hpmg_ctx& C, int cap) {
  if (cap <= C.gm_cap) return;
  for (void* p : {(void*)C.gm.V, (void*)C.gm.H, (void*)C.gm.cs, (void*)C.gm.sn, (void*)C.gm.g, (void*)C.gm.y})
    if (p) dfree(p);
  const int64_t n = C.top().n;
  C.gm.ldv = (n + 31) & ~int64_t(31);
  C.gm.ldh = cap + 1;
  C.gm.V = dalloc<double>(size_t(cap + 1) * size_t(C.gm.ldv));
  C.gm.H = dalloc<double>(size_t(cap) * size_t(cap + 1));
  C.gm.cs = dalloc<double>(cap);
  C.gm.sn = dalloc<double>(cap);
  C.gm.g = dalloc<double>(cap + 1);
  C.gm.y = dalloc<double>(cap);
  if (!C.gm.st) C.gm.st = dalloc<double>(dev::kGmSlots);
  if (!C.gm.part) C.gm.part = dalloc<double>(2 * size_t(dev::kRedBlocks));
  C.gm_cap = cap;
  if (C.gm_loop) cudaGraphExecDestroy(C.gm_loop);
  C.gm_loop = nullptr;
}

/// The whole restarted GMRES (reference krylov.hpp:79-144) as one graph:
///   while (running):                                  -- restart cycles
///     r = b - A x, r.r, true-residual test
///     if (not converged):
///       V0 = r / beta
///       while (Arnoldi continues):                    -- steps j
///         kr = V[j]; kz = M kr (V-cycle); w = A kz
///         while (i <= j): w -= h(i-1) V[i-1]; h(i) = w.V[i]   (fused MGS)
///         w -= h(j) V[j], |w|; V[j+1] = w / h(j+1); Givens, g, stop test
///       y = H \ g; kr = sum y_i V[i]; kz = M kr; x += kz
///       r = b - A x, r.r; converged / stalled / out of iterations
/// Every predicate is set on the device.
bool build_gm_loop(hpmg_ctx& C) {
  Level& T = C.top();
  const int64_t n = T.n;
  const dev::GmDev G = C.gm;
  cudaGraph_t g = nullptr;
  try {
    GK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_outer, h_cyc, h_inner, h_mgs;
    GK(cudaGraphConditionalHandleCreate(&h_outer, g, 1, cudaGraphCondAssignDefault));
    GK(cudaGraphConditionalHandleCreate(&h_cyc, g, 0, cudaGraphCondAssignDefault));
    GK(cudaGraphConditionalHandleCreate(&h_inner, g, 0, cudaGraphCondAssignDefault));
    GK(cudaGraphConditionalHandleCreate(&h_mgs, g, 0, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_outer;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    GK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
    capture_body(C, wp.conditional.phGraph_out[0], 0, [&] {
      dev::spmv(T.A, C.kx, C.kb, C.kr, 1, nullptr, nullptr, C.s);
      dev::dot(C.kr, C.kr, n, C.red, C.sc + S_RR, C.s);
      dev::gm_start(C.sc, G, h_cyc, h_inner, C.s);
      cudaGraph_t cyc = add_conditional(C.s, h_cyc, cudaGraphCondTypeIf);
      capture_body(C, cyc, 1, [&] {
        dev::gm_v0(G, C.kr, C.kr, n, h_mgs, C.s);  // V[0] = r / beta, in place as z's input
        cudaGraph_t inner = add_conditional(C.s, h_inner, cudaGraphCondTypeWhile);
        capture_body(C, inner, 2, [&] {
          apply_blocks(C, C.kr, C.kz);                                  // z = M v_j
          dev::spmv(T.A, C.kz, nullptr, C.ktmp, 0, nullptr, nullptr, C.s);  // w = A z
          cudaGraph_t mgs = add_conditional(C.s, h_mgs, cudaGraphCondTypeWhile);
          // eight MGS steps per loop-body iteration (steps past j return at once)
          capture_body(C, mgs, 3, [&] {
            for (int u = 0; u < 8; ++u) dev::mgs_step(G, C.ktmp, n, u, h_mgs, C.s);
          });
          dev::mgs_tail(G, C.ktmp, n, C.s);
          dev::gm_arnoldi_close(C.sc, G, C.ktmp, C.kr, n, C.red, h_inner, h_mgs, C.s);
        });
        dev::gm_update(G, C.kr, n, C.s);  // u = V y into the preconditioner's input
        apply_blocks(C, C.kr, C.kz);
        dev::axpy(C.kx, 1.0, C.kz, n, C.s);
        dev::spmv(T.A, C.kx, C.kb, C.kr, 1, nullptr, nullptr, C.s);
        dev::dot(C.kr, C.kr, n, C.red, C.sc + S_RR, C.s);
        dev::gm_end(C.sc, G, C.s);
      });
      dev::loop_continue(C.sc, h_outer, C.s);
    });
    GK(cudaGraphInstantiate(&C.gm_loop, g, 0));
  } catch (const GraphError& e) {
    if (g) cudaGraphDestroy(g);
    C.gm_loop = nullptr;
    cudaGetLastError();
    if (std::getenv("HPMG_DEBUG_GRAPH")) std::fprintf(stderr, "gmres loop graph: %s\n", cudaGetErrorString(e.e));
    return false;
  } catch (const std::exception& e) {
    if (g) cudaGraphDestroy(g);
    C.gm_loop = nullptr;
    cudaGetLastError();
    if (std::getenv("HPMG_DEBUG_GRAPH")) std::fprintf(stderr, "gmres loop graph: %s\n", e.what());
    return false;
  }
  cudaGraphDestroy(g);
  C.gm_graph_cap = C.gm_cap;
  return true;
}

double* gm_vec(hpmg_ctx& C, int i) {
  while (int(C.gm_basis.size()) <= i) C.gm_basis.push_back(dalloc<double>(C.top().n));
  return C.gm_basis[i];
}

/// Right-preconditioned MGS GMRES on the device, Givens on the host
/// (reference inc/krylov.hpp:79-144); `restart` > 0 caps the cycle length.
hpmg_solve_stats gmres_device(hpmg_ctx& C, const hpmg_krylov_opts& o) {
  hpmg_solve_stats st{0, 0, 0, 0.0};
  Level& T = C.top();
  const int64_t n = T.n;
  dev::dot(C.kb, C.kb, n, C.red, C.sc + S_BB, C.s);
  read_scalars(C);
  const double target = std::max(o.rel_tol * std::sqrt(C.sc_host[S_BB]), o.abs_tol);
  static const bool host_loop = std::getenv("HPMG_KRYLOV_HOST") && std::atoi(std::getenv("HPMG_KRYLOV_HOST"));
  if (!host_loop && o.max_iterations > 0 && !C.gm_loop_failed) {
    // one graph launch for the whole solve (build_gm_loop)
    const int want = o.restart > 0 ? std::min(o.restart, o.max_iterations) : o.max_iterations;
    gm_workspace(C, want);
    if (!C.gm_loop || C.gm_graph_cap != C.gm_cap) {
      C.gm_loop_failed = !build_gm_loop(C);
    }
    if (C.gm_loop) {
      dev::gm_init(C.sc, C.gm, target, double(o.max_iterations), want, C.s);
      CK(cudaGraphLaunch(C.gm_loop, C.s));
      read_scalars(C);
      st.iterations = int(C.sc_host[dev::kScIt]);
      st.residual = std::sqrt(C.sc_host[S_RR]);
      st.converged = C.sc_host[dev::kScStatus] == dev::kLoopConverged;
      return st;
    }
  }
  const double breakdown = 1e-14;
  const int cap = o.restart > 0 ? o.restart : (1 << 30);
  while (st.iterations < o.max_iterations) {
    dev::spmv(T.A, C.kx, C.kb, C.kr, 1, nullptr, nullptr, C.s);
    dev::dot(C.kr, C.kr, n, C.red, C.sc + S_RR, C.s);
    read_scalars(C);
    st.residual = std::sqrt(C.sc_host[S_RR]);
    if (st.residual <= target) {
      st.converged = 1;
      return st;
    }
    const double beta = st.residual;
    dev::scal_axpby(gm_vec(C, 0), C.kr, n, nullptr, -1, 1.0 / beta, 0.0, C.s);
    std::vector<std::vector<double>> hc;
    std::vector<double> cs, sn, g{beta};
    bool stalled = false;
    for (int j = 0; st.iterations < o.max_iterations && j < cap; ++j) {
      dev::copy(C.kr, gm_vec(C, j), n, C.s);
      apply_graph(C);                                                        // kz = M v_j
      dev::spmv(T.A, C.kz, nullptr, C.ktmp, 0, nullptr, nullptr, C.s);      // w = A M v_j
      for (int i = 0; i <= j; ++i) {                                          // modified Gram-Schmidt
        dev::dot(C.ktmp, gm_vec(C, i), n, C.red, C.sc + S_H0 + i, C.s);
        dev::scal_axpby(C.ktmp, gm_vec(C, i), n, C.sc, S_H0 + i, -1.0, 1.0, C.s);
      }
      dev::dot(C.ktmp, C.ktmp, n, C.red, C.sc + S_H0 + j + 1, C.s);
      read_scalars(C, S_H0 + j + 2);
      std::vector<double> h(j + 2);
      for (int i = 0; i <= j; ++i) h[i] = C.sc_host[S_H0 + i];
      h[j + 1] = std::sqrt(C.sc_host[S_H0 + j + 1]);
      const bool happy = h[j + 1] <= breakdown * beta;
      if (!happy) dev::scal_axpby(gm_vec(C, j + 1), C.ktmp, n, nullptr, -1, 1.0 / h[j + 1], 0.0, C.s);
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
      }
      const double rho = std::hypot(h[j], h[j + 1]);
      cs.push_back(h[j] / rho);
      sn.push_back(h[j + 1] / rho);
      h[j] = rho;
      h[j + 1] = 0;
      g.push_back(-sn.back() * g[j]);
      g[j] *= cs.back();
      hc.push_back(h);
      ++st.iterations;
      if (std::abs(g.back()) <= target || happy) {
        stalled = happy && std::abs(g.back()) > target;
        break;
      }
    }
    const int m = int(hc.size());
    std::vector<double> y(m);
    for (int i = m - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < m; ++l) s -= hc[l][i] * y[l];
      y[i] = s / hc[i][i];
    }
    dev::fill(C.kr, 0.0, n, C.s);
    for (int i = 0; i < m; ++i) dev::axpy(C.kr, y[i], gm_vec(C, i), n, C.s);
    apply_graph(C);
    dev::axpy(C.kx, 1.0, C.kz, n, C.s);
    dev::spmv(T.A, C.kx, C.kb, C.kr, 1, nullptr, nullptr, C.s);
    dev::dot(C.kr, C.kr, n, C.red, C.sc + S_RR, C.s);
    read_scalars(C);
    st.residual = std::sqrt(C.sc_host[S_RR]);
    if (st.residual <= target) {
      st.converged = 1;
      return st;
    }
    if (stalled) return st;
  }
  return st;
}

void linearise(hpmg_ctx& C, const hpmg_problem* prob, const host::RefTensors* Tk);

void setup(hpmg_ctx& C, const hpmg_mesh_desc* md, const hpmg_options* opt, const hpmg_problem* prob) {
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("no CUDA device: hpmg has no CPU fallback");
  if (opt->k < 0 || opt->k > 6) throw std::invalid_argument("order k must be in 0..6");
  if (opt->sweep_variant != HPMG_SWEEP_RECORDS && opt->sweep_variant != HPMG_SWEEP_DIRECT_NONSYM)
    throw std::invalid_argument("unknown sweep variant");
  if (md->levels < 1) throw std::invalid_argument("levels must be >= 1");
  C.opt = *opt;
  C.advected = prob && (prob->wind_compound || prob->wind);
  if (prob && prob->newton && !(prob->wind_compound || prob->wind))
    throw std::invalid_argument("a Newton linearisation needs the advection state (wind)");
  if (prob && prob->mass_compound && (opt->k > 0 && !prob->mass_interior))
    throw std::invalid_argument("mass field needs its interior coefficients at k > 0");
  CK(cudaStreamCreateWithFlags(&C.s, cudaStreamNonBlocking));
  // mesh hierarchy
  host::TriMesh base;
  for (int v = 0; v < md->n_vertices; ++v) {
    base.vx.push_back(md->xy[2 * v]);
    base.vy.push_back(md->xy[2 * v + 1]);
  }
  for (int e = 0; e < md->n_elements; ++e)
    base.ev.push_back({md->elements[3 * e], md->elements[3 * e + 1], md->elements[3 * e + 2]});
  base.build_facets();
  if (md->n_tag_overrides > 0) {
    std::unordered_map<uint64_t, int> tags = base.tag_map();
    for (int i = 0; i < md->n_tag_overrides; ++i) {
      int a = md->tag_overrides[3 * i], b = md->tag_overrides[3 * i + 1];
      if (a > b) std::swap(a, b);
      tags[(uint64_t(uint32_t(a)) << 32) | uint32_t(b)] = md->tag_overrides[3 * i + 2];
    }
    base.build_facets(&tags);
  }
  C.mesh.push_back(std::move(base));
  for (int l = 1; l < md->levels; ++l) {
    host::Refinement R;
    host::TriMesh f = host::refine(C.mesh[l - 1], R);
    C.mesh.push_back(std::move(f));
    C.ref.push_back(std::move(R));
  }
  C.L = md->levels - 1;
  SetupTrace tr;
  tr.mark("mesh hierarchy");
  const host::TriMesh& fine = C.mesh[C.L];
  for (int f = 0; f < fine.nf(); ++f)
    if (fine.ftag[f] == host::kTagOutflow) C.enclosed = false;
  const int k = opt->k;
  auto tT0 = host::build_ref_tensors(0);
  upload_ref(C.ref0, *tT0, C.s);
  std::unique_ptr<host::RefTensors> tTk;
  if (k > 0) {
    tTk = host::build_ref_tensors(k);
    upload_ref(C.refk, *tTk, C.s);
  }
  tr.mark("reference tensors");
  // reductions and scalars
  C.red.partial = dalloc<double>(dev::kRedBlocks);
  C.red.counter = dalloc<unsigned>(1);
  CK(cudaMemsetAsync(C.red.counter, 0, sizeof(unsigned), C.s));
  C.sc = dalloc<double>(S_COUNT);
  CK(cudaMemsetAsync(C.sc, 0, sizeof(double) * S_COUNT, C.s));
  CK(cudaMallocHost(&C.sc_host, sizeof(double) * S_COUNT));
  // Dirichlet data and constraints of the finest system
  const std::vector<double> gfac = dirichlet_data(fine, k, prob ? prob->bc : nullptr, prob ? prob->bc_user : nullptr);
  C.g_fac = dupload(gfac, C.s);
  std::vector<char> dir(fine.nf());
  for (int f = 0; f < fine.nf(); ++f) dir[f] = fine.ftag[f] == host::kTagDirichlet;
  C.facet_dir = dupload(dir, C.s);
  {
    const int nfd = k + 1, bs = 2 * nfd;
    const int64_t nflux = int64_t(fine.nf()) * nfd;
    C.g_full.assign(2 * nflux, 0.0);
    for (int f = 0; f < fine.nf(); ++f)
      for (int i = 0; i < nfd; ++i) {
        C.g_full[int64_t(f) * nfd + i] = gfac[size_t(f) * bs + 2 * i];
        C.g_full[nflux + int64_t(f) * nfd + i] = gfac[size_t(f) * bs + 2 * i + 1];
      }
    for (int f = 0; f < fine.nf(); ++f)
      if (!dir[f])
        for (int i = 0; i < nfd; ++i) C.free_to_full.push_back(int64_t(f) * nfd + i);
    for (int f = 0; f < fine.nf(); ++f)
      if (!dir[f])
        for (int i = 0; i < nfd; ++i) C.free_to_full.push_back(nflux + int64_t(f) * nfd + i);
  }
  auto t1 = clk::now();
  // structure of every level
  C.lv.resize(C.L + 1);
  {
    // host plans of all levels (and the order-k head) on concurrent threads
    std::vector<host::LevelPlan> plans(C.L + 2);
    std::vector<std::string> errs(C.L + 2);
    std::vector<std::thread> pool;
    for (int l = 0; l <= C.L + (k > 0 ? 1 : 0); ++l)
      pool.emplace_back([&, l] {
        try {
          plans[l] = l <= C.L ? host::make_level(C.mesh[l], 0) : host::make_level(fine, k);
        } catch (const std::exception& e) {
          errs[l] = e.what();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    tr.mark("dirichlet + level plans");
    for (int l = 0; l <= C.L; ++l) {
      C.lv[l] = std::make_unique<Level>();
      Level& V = *C.lv[l];
      const bool finest = (k == 0 && l == C.L);
      plan_level(C, V, C.mesh[l], 0, finest, std::move(plans[l]));
      V.steps = opt->cycle == HPMG_CYCLE_VARIABLE_V ? (opt->smooth_steps << (C.L - l)) : opt->smooth_steps;
      tr.mark("level upload");
    }
    if (k > 0) {
      C.head = std::make_unique<Level>();
      plan_level(C, *C.head, fine, k, true, std::move(plans[C.L + 1]), C.lv[C.L]->geo);
      C.head->steps = opt->smooth_steps;
    }
  }
  tr.mark("level uploads");
  C.rhs = dalloc<double>(int64_t(C.free_to_full.size()));
  // everything that depends on the linearisation state
  const auto t_lin = clk::now();
  linearise(C, prob, k > 0 ? tTk.get() : tT0.get());
  auto t2 = clk::now();
  (void)t2;
  C.setup_parts[2] = C.lin_parts[0];
  C.setup_parts[3] = C.lin_parts[1];
  C.setup_parts[4] = C.lin_parts[2];
  auto t5 = clk::now();
  // solver workspace
  Level& T = C.top();
  for (double** p : {&C.kx, &C.kb, &C.kr, &C.kz, &C.kp, &C.kAp, &C.ktmp, &C.io_a, &C.io_b}) *p = dalloc<double>(T.n);
  C.pres = dalloc<double>(fine.ne());
  C.div = dalloc<double>(fine.ne());
  C.urhs = dalloc<double>(T.n);
  build_apply_graph(C);
  CK(cudaStreamSynchronize(C.s));
  tr.mark("workspace + graph");
  auto t6 = clk::now();
  auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  C.setup_parts[0] = sec(t0, t1);                      // mesh + tables
  // plans + level uploads (host) + condensation (device); parts [2..4] are
  // device times of phases that overlap the host's transfer uploads, so the
  // parts need not add up to the total
  C.setup_parts[1] = sec(t1, t_lin) + C.lin_parts[3];
  C.setup_parts[5] = sec(t5, t6);                      // workspace + graph
  C.setup_parts[6] = sec(t0, t6);
}

/// Everything that depends on the linearisation state (the reference rebuilds
/// the whole MGPreconditioner per Picard / Newton step, ns.hpp:84): the wind
/// chain (multigrid.hpp:58-66), condensation and assembly of every level, the
/// The level-1 V(1,1) sub-cycle as one dense map (dense_level.cu) where the
/// one-CTA level path would run it: V-cycle (or variable V), multiplicative
/// smoother, level 1 small, n1 <= 8192 (M1 <= 512 MB; past that the GEMV
/// costs more than the sweeps). HPMG_DENSE_L1=0 keeps the sweeps.
void build_dense_level1(hpmg_ctx& C) {
  const char* env = std::getenv("HPMG_DENSE_L1");
  const bool want = !(env && env[0] == '0') && C.L >= 1 && C.lv[1]->small &&
                    C.opt.smoother == HPMG_SMOOTH_MULTIPLICATIVE && C.opt.cycle != HPMG_CYCLE_W && C.lv[1]->n <= 8192 &&
                    C.L >= 2;  // level 1's input is then always its own (padded) b
  if (!want) {
    if (C.m1) dfree(C.m1);
    C.m1 = nullptr;
    C.m1_n = 0;
    return;
  }
  Level& V = *C.lv[1];
  const bool sym = !(env && env[0] == '2');
  if (!C.m1 || C.m1_n != int(V.n) || C.m1_sym != sym) {
    if (C.m1) dfree(C.m1);
    C.m1 = dalloc<double>(dev::dense_level1_size(int(V.n), sym));
    C.m1_n = int(V.n);
    C.m1_sym = sym;
  }
  // scratch from the context pool: stream-ordered, reused by the next context
  void* w = nullptr;
  CK(cudaMallocFromPoolAsync(&w, sizeof(double) * dev::dense_level1_work(int(V.n), C.n0), alloc_pool(), C.s));
  dev::dense_level1(V.A, V.srec, V.d_passes, V.npass, V.steps, V.PT, V.Pm, C.n0, C.coarse_inv, C.m1,
                    static_cast<double*>(w), C.m1_sym, C.s);
  CK(cudaFreeAsync(w, C.s));
}

/// patch inverses, the corrected prolongations and the coarse inverse.
void linearise(hpmg_ctx& C, const hpmg_problem* prob, const host::RefTensors* Tk) {
  using clk = std::chrono::steady_clock;
  auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  SetupTrace tr;
  const int k = C.opt.k;
  const host::TriMesh& fine = C.mesh[C.L];
  std::vector<host::HdgField> adv;
  host::HdgField wind_k;
  if (C.advected) {
    if (prob->wind) {
      wind_k = host::interpolate_hdg(fine, k, *Tk, [&](double x, double y, double* o) {
        prob->wind(x, y, o, prob->wind_user);
      });
    } else {
      wind_k.k = k;
      wind_k.compound.assign(prob->wind_compound, prob->wind_compound + C.g_full.size());
      const size_t ni = size_t(fine.ne()) * k * (k + 1);
      if (ni) wind_k.interior.assign(prob->wind_interior, prob->wind_interior + ni);
    }
    adv.resize(C.L + 1);
    adv[C.L] = k > 0 ? host::lowest_order(fine, wind_k) : wind_k;
    for (int l = C.L; l > 0; --l) adv[l - 1] = host::restrict_wind(C.mesh[l - 1], C.mesh[l], C.ref[l - 1], adv[l]);
  }
  // transfer structure (host, first linearisation only) on a helper thread
  // while the condensation, patch inverses and coarse inverse run on the device
  static_assert(host::TransferPlan::kColMax == dev::kTransferColMax, "transfer column capacity");
  const bool need_tp = C.L >= 1 && !C.lv[1]->tdev.base;
  std::vector<host::TransferPlan> tp(C.L + 1);
  std::vector<std::string> tp_errs(C.L + 1);
  std::thread tp_thread;
  if (need_tp)
    tp_thread = std::thread([&] {
      std::vector<std::thread> pool;
      for (int l = 1; l <= C.L; ++l)
        pool.emplace_back([&, l] {
          try {
            tp[l] = host::transfer_plan(C.lv[l - 1]->plan, C.lv[l]->plan, C.ref[l - 1]);
          } catch (const std::exception& e) {
            tp_errs[l] = e.what();
          }
        });
      for (auto& t : pool) t.join();
    });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{tp_thread};
  // the condensation scratch sized once for the largest level (a regrowth
  // between levels would synchronise the device)
  {
    size_t need = 0;
    for (int l = 0; l <= C.L; ++l) need = std::max(need, size_t(C.mesh[l].ne()) * (C.ref0.T.nc * C.ref0.T.nc + C.ref0.T.nc));
    if (k > 0) need = std::max(need, size_t(fine.ne()) * (C.refk.T.nc * C.refk.T.nc + C.refk.T.nc));
    if (C.acr_cap < need) {
      if (C.acr) dfree(C.acr);
      C.acr = dalloc<double>(need);
      C.acr_cap = need;
    }
  }
  // The device work below is queued without host synchronisation (phase
  // times from events on the stream), so the host joins and uploads the
  // transfer structure while the condensation and the patch inverses run.
  struct Events {  // released on every exit path (setup errors throw)
    cudaEvent_t e[8] = {};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } evs;
  cudaEvent_t* ev = evs.e;
  for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&ev[i]));
  // coarse-inverse buffers first: allocations stay out of the queued work
  Level& V0 = *C.lv[0];
  C.n0 = int(V0.n);
  if (!C.coarse_inv) C.coarse_inv = dalloc<double>(size_t(C.n0) * C.n0);
  if (!C.coarse_dense) C.coarse_dense = dalloc<double>(size_t(C.n0) * C.n0);
  dev::dense_invert_alloc(C.n0, C.gj);
  if (!C.s_coarse) CK(cudaStreamCreateWithFlags(&C.s_coarse, cudaStreamNonBlocking));
  CK(cudaEventRecord(ev[0], C.s));
  linearise_level(C, V0, C.mesh[0], C.ref0, prob, V0.finest ? C.rhs : nullptr, C.advected ? &adv[0] : nullptr);
  // the coarse dense inverse (Gauss-Jordan with partial pivoting, kernels.cu
  // dense_invert_async) of the level-0 operator, densified on the device, on
  // a side stream: its latency-bound pivot steps run beside the finer levels'
  // condensation and patch inverses
  CK(cudaEventRecord(ev[5], C.s));
  CK(cudaStreamWaitEvent(C.s_coarse, ev[5], 0));
  CK(cudaEventRecord(ev[6], C.s_coarse));
  dev::bsr_to_dense(V0.A, C.coarse_dense, C.s_coarse);
  dev::dense_invert_async(C.n0, C.coarse_dense, C.coarse_inv, C.gj, C.s_coarse);
  CK(cudaEventRecord(ev[7], C.s_coarse));
  for (int l = 1; l <= C.L; ++l)
    linearise_level(C, *C.lv[l], C.mesh[l], C.ref0, prob, C.lv[l]->finest ? C.rhs : nullptr,
                    C.advected ? &adv[l] : nullptr);
  if (k > 0) linearise_level(C, *C.head, fine, C.refk, prob, C.rhs, C.advected ? &wind_k : nullptr);
  CK(cudaEventRecord(ev[1], C.s));
  if (tr.on) CK(cudaStreamSynchronize(C.s));
  tr.mark("condense + assemble");
  for (int l = 1; l <= C.L; ++l) build_patch_inverses(C, *C.lv[l]);
  if (k > 0) build_patch_inverses(C, *C.head);
  CK(cudaEventRecord(ev[2], C.s));
  if (tr.on) CK(cudaStreamSynchronize(C.s));
  tr.mark("patch inverses + records");
  // transfers: structure once (the helper thread above), uploaded while the
  // device works; the harmonic correction from the current fine operators
  const auto t_tp = clk::now();
  if (need_tp) {
    tp_thread.join();
    tr.mark("transfer plans (host wait)");
    for (int l = 1; l <= C.L; ++l) {
      if (!tp_errs[l].empty()) throw std::runtime_error(tp_errs[l]);
      Level& V = *C.lv[l];
      const host::TransferPlan& T = tp[l];
      V.Pm = upload_blockcsr(T.P, C.s, false);  // P = base + correction (corrected_prolongation)
      V.PT = upload_blockcsr(T.PT, C.s, false);
      V.Pm.nnz = V.PT.nnz = int(T.P.col.size());
      dev::TransferDev& D = V.tdev;
      D.nelem = T.nelem;
      D.nnz = int(T.P.col.size());
      D.nmed = dupload(T.nmed, C.s);
      D.med = dupload(T.med, C.s);
      D.ncol = dupload(T.ncol, C.s);
      D.col = dupload(T.col, C.s);
      D.pos = dupload(T.pos, C.s);
      D.avg_ptr = dupload(T.avg.ptr, C.s);
      D.avg_col = dupload(T.avg.col, C.s);
      D.avg_val = dupload(T.avg.val, C.s);
      D.base = dalloc<double>(T.P.col.size() * 4);
      dev::prolong_base(V.Pm, D, C.s);  // the averaging values in P's pattern
      D.tperm = dupload(T.tperm, C.s);
      V.p_nnz = 4.0 * double(T.P.col.size());
    }
  }
  const double t_upload = sec(t_tp, clk::now());
  for (int l = 1; l <= C.L; ++l) dev::corrected_prolongation(C.lv[l]->A, C.lv[l]->tdev, C.lv[l]->Pm, C.lv[l]->PT, C.s);
  CK(cudaEventRecord(ev[3], C.s));
  tr.mark("transfer upload + correction");
  // join the coarse inverse
  CK(cudaStreamWaitEvent(C.s, ev[7], 0));
  if (!C.gemv_work) {
    C.gemv_work = dalloc<double>(dev::dense_gemv_work(C.n0));
    CK(cudaMemsetAsync(C.gemv_work, 0, sizeof(double) * dev::dense_gemv_work(C.n0), C.s));  // arrival counters
  }
  CK(cudaEventRecord(ev[4], C.s));
  dev::dense_invert_check(C.gj, C.s_coarse);  // synchronises the side stream; throws if singular
  CK(cudaStreamSynchronize(C.s));
  tr.mark("coarse inverse (joined)");
  auto el = [&](int a, int b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return 1e-3 * double(ms);
  };
  C.lin_parts[0] = el(1, 2);             // patch inverses + records (device)
  C.lin_parts[1] = t_upload + el(2, 3);  // transfer join + uploads (host) + correction (device)
  C.lin_parts[2] = el(6, 7);             // coarse densify + inverse (device, side stream, overlapped)
  C.lin_parts[3] = el(0, 1);             // condensation + assembly (device)
  build_dense_level1(C);
  tr.mark("dense level-1 cycle");

}

template <typename F>
int guarded(hpmg_ctx* C, F&& f) {
  try {
    f();
    return HPMG_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    if (C) C->err = e.what();
    return HPMG_ERR_ARG;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (C) C->err = e.what();
    return std::string(e.what()).find("CUDA") != std::string::npos || std::string(e.what()).find("cuda") != std::string::npos
               ? HPMG_ERR_CUDA
               : HPMG_ERR_SETUP;
  }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* hpmg_last_error(void) { return g_last_error.c_str(); }
void hpmg_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
const char* hpmg_ctx_error(const hpmg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int hpmg_create(hpmg_ctx** out, const hpmg_mesh_desc* mesh, const hpmg_options* opt, const hpmg_problem* prob) {
  if (!out || !mesh || !opt) {
    g_last_error = "null argument";
    return HPMG_ERR_ARG;
  }
  auto* C = new hpmg_ctx();
  int rc = guarded(C, [&] { setup(*C, mesh, opt, prob); });
  if (rc != HPMG_OK) {
    delete C;  // device memory is reclaimed with the process / context
    *out = nullptr;
    return rc;
  }
  *out = C;
  return HPMG_OK;
}

int hpmg_update(hpmg_ctx* ctx, const hpmg_options* opt, const hpmg_problem* prob) {
  return guarded(ctx, [&] {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    hpmg_ctx& C = *ctx;
    const bool advected = prob && (prob->wind_compound || prob->wind);
    if (opt->k != C.opt.k || opt->cycle != C.opt.cycle || opt->smoother != C.opt.smoother ||
        opt->smooth_steps != C.opt.smooth_steps || opt->sweep_variant != C.opt.sweep_variant || advected != C.advected)
      throw std::invalid_argument("hpmg_update changes only the linearisation state (wind, Newton, mass terms, nu, "
                                  "beta, inv_eps); order, cycle, smoother and symmetry need a new context");
    if (prob && prob->newton && !advected)
      throw std::invalid_argument("a Newton linearisation needs the advection state (wind)");
    C.opt.nu = opt->nu;
    C.opt.beta = opt->beta;
    C.opt.mass_coef = opt->mass_coef;
    C.opt.inv_eps = opt->inv_eps;
    C.opt.jacobi_damping = opt->jacobi_damping;
    // Dirichlet data of the (possibly new) boundary function, same constraint pattern
    const int k = C.opt.k;
    const host::TriMesh& fine = C.mesh[C.L];
    const std::vector<double> gfac = dirichlet_data(fine, k, prob ? prob->bc : nullptr, prob ? prob->bc_user : nullptr);
    CK(cudaMemcpyAsync(C.g_fac, gfac.data(), sizeof(double) * gfac.size(), cudaMemcpyHostToDevice, C.s));
    {
      const int nfd = k + 1, bs = 2 * nfd;
      const int64_t nflux = int64_t(fine.nf()) * nfd;
      for (int f = 0; f < fine.nf(); ++f)
        for (int i = 0; i < nfd; ++i) {
          C.g_full[int64_t(f) * nfd + i] = gfac[size_t(f) * bs + 2 * i];
          C.g_full[nflux + int64_t(f) * nfd + i] = gfac[size_t(f) * bs + 2 * i + 1];
        }
    }
    CK(cudaStreamSynchronize(C.s));
    std::unique_ptr<host::RefTensors> Tk;
    if (prob && prob->wind) Tk = host::build_ref_tensors(k);
    linearise(C, prob, Tk.get());
    if (C.apply_graph) cudaGraphExecDestroy(C.apply_graph);
    C.apply_graph = nullptr;
    destroy_io_graph(C);
    if (C.pcg_loop) cudaGraphExecDestroy(C.pcg_loop);
    C.pcg_loop = nullptr;
    if (C.gm_loop) cudaGraphExecDestroy(C.gm_loop);
    C.gm_loop = nullptr;
    build_apply_graph(C);
    CK(cudaStreamSynchronize(C.s));
    C.setup_parts[1] = C.lin_parts[3];
    C.setup_parts[2] = C.lin_parts[0];
    C.setup_parts[3] = C.lin_parts[1];
    C.setup_parts[4] = C.lin_parts[2];
    C.setup_parts[0] = C.setup_parts[5] = 0.0;
    C.setup_parts[6] = std::chrono::duration<double>(clk::now() - t0).count();
  });
}

void hpmg_destroy(hpmg_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->s);
  if (ctx->apply_graph) cudaGraphExecDestroy(ctx->apply_graph);
  destroy_io_graph(*ctx);
  if (ctx->pcg_loop) cudaGraphExecDestroy(ctx->pcg_loop);
  if (ctx->gm_loop) cudaGraphExecDestroy(ctx->gm_loop);
  for (cudaStream_t q : ctx->s_nest)
    if (q) cudaStreamDestroy(q);
  for (void* p : {(void*)ctx->gm.V, (void*)ctx->gm.H, (void*)ctx->gm.cs, (void*)ctx->gm.sn, (void*)ctx->gm.g,
                  (void*)ctx->gm.y, (void*)ctx->gm.st, (void*)ctx->gm.part})
    if (p) dfree(p);
  auto fr = [](void* p) { if (p) dfree(p); };
  auto free_level = [&](Level* V) {
    if (!V) return;
    for (void* p : {(void*)V->A.val, (void*)V->A.cols, (void*)V->A0.val, (void*)V->AT.val, (void*)V->tslot, (void*)V->P.nf,
                    (void*)V->P.fac, (void*)V->P.off, (void*)V->P.inv, (void*)V->P.wave, (void*)V->P.fpatch,
                    (void*)V->Pm.ptr, (void*)V->Pm.col, (void*)V->Pm.val, (void*)V->PT.ptr, (void*)V->PT.col,
                    (void*)V->PT.val, (void*)V->x, (void*)V->b, (void*)V->r, (void*)V->y, (void*)V->bw, (void*)V->xw,
                    (void*)V->dbuf, (void*)(V->geo_shared ? nullptr : V->geo), (void*)V->row_elems, (void*)V->elem_facets, (void*)V->facet_block,
                    (void*)V->d_wave_ptr, (void*)V->rec.rec, (void*)V->srec.rec, (void*)V->rect.rec,
                    (void*)V->d_passes, (void*)V->gath,
                    (void*)V->block_facet, (void*)V->tdev.nmed, (void*)V->tdev.med, (void*)V->tdev.ncol,
                    (void*)V->tdev.col, (void*)V->tdev.pos, (void*)V->tdev.avg_ptr, (void*)V->tdev.avg_col,
                    (void*)V->tdev.avg_val, (void*)V->tdev.base, (void*)V->tdev.tperm})
      fr(p);
  };
  for (auto& V : ctx->lv) free_level(V.get());
  free_level(ctx->head.get());
  for (void* p : ctx->ref0.owned) fr(p);
  for (void* p : ctx->refk.owned) fr(p);
  for (void* p : ctx->post.owned) fr(p);
  for (int i = 0; i < 2; ++i) {
    fr(ctx->bin[i]);
    fr(ctx->bout[i]);
    for (cudaEvent_t e : {ctx->ev_in[i], ctx->ev_used[i], ctx->ev_done[i], ctx->ev_out[i]})
      if (e) cudaEventDestroy(e);
  }
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
  for (double* p : ctx->gm_basis) fr(p);
  dev::dense_invert_free(ctx->gj);
  if (ctx->s_coarse) cudaStreamDestroy(ctx->s_coarse);
  for (void* p : {(void*)ctx->m1, (void*)ctx->coarse_inv, (void*)ctx->coarse_dense, (void*)ctx->gemv_work, (void*)ctx->red.partial, (void*)ctx->red.counter,
                  (void*)ctx->sc, (void*)ctx->rhs, (void*)ctx->g_fac, (void*)ctx->facet_dir, (void*)ctx->kx,
                  (void*)ctx->kb, (void*)ctx->kr, (void*)ctx->kz, (void*)ctx->kp, (void*)ctx->kAp, (void*)ctx->ktmp,
                  (void*)ctx->io_a, (void*)ctx->io_b, (void*)ctx->pres, (void*)ctx->div, (void*)ctx->urhs,
                  (void*)ctx->fine_load, (void*)ctx->fine_wind, (void*)ctx->fine_mass, (void*)ctx->acr})
    fr(p);
  if (ctx->sc_host) cudaFreeHost(ctx->sc_host);
  if (ctx->s) cudaStreamDestroy(ctx->s);
  delete ctx;
}

int64_t hpmg_n(const hpmg_ctx* ctx) { return int64_t(ctx->free_to_full.size()); }
int64_t hpmg_n_full(const hpmg_ctx* ctx) { return int64_t(ctx->g_full.size()); }
int hpmg_ne(const hpmg_ctx* ctx) { return ctx->mesh.back().ne(); }
int hpmg_num_levels(const hpmg_ctx* ctx) { return int(ctx->lv.size()); }
int64_t hpmg_level_n(const hpmg_ctx* ctx, int level) {
  auto& C = *const_cast<hpmg_ctx*>(ctx);
  if (level < 0) return C.top().n;
  if (level >= int(C.lv.size())) return -1;
  return C.lv[level]->n;
}
int hpmg_level_patches(const hpmg_ctx* ctx, int level) {
  auto& C = *const_cast<hpmg_ctx*>(ctx);
  if (level < 0) return C.top().P.n;
  if (level >= int(C.lv.size())) return -1;
  return C.lv[level]->P.n;
}
int hpmg_symmetric(const hpmg_ctx* ctx) { return ctx->advected ? 0 : 1; }
double hpmg_penalty(const hpmg_ctx* ctx) { return ctx->opt.inv_eps; }
int hpmg_free_to_full(const hpmg_ctx* ctx, int64_t* out) {
  std::memcpy(out, ctx->free_to_full.data(), sizeof(int64_t) * ctx->free_to_full.size());
  return HPMG_OK;
}
int hpmg_g_full(const hpmg_ctx* ctx, double* out) {
  std::memcpy(out, ctx->g_full.data(), sizeof(double) * ctx->g_full.size());
  return HPMG_OK;
}
int hpmg_rhs(hpmg_ctx* ctx, double* out, int flags) {
  return guarded(ctx, [&] { out_vec(*ctx, ctx->rhs, out, flags); });
}

int hpmg_matrix_csr(hpmg_ctx* ctx, int level, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val) {
  return guarded(ctx, [&] {
    Level& V = level < 0 ? ctx->top() : *ctx->lv.at(level);
    const int nfd = V.k + 1, bs = V.bs, nb = V.nb;
    auto ref_of = [&](int blk, int ii) -> int64_t {
      const int i = ii >> 1, t = ii & 1;
      return (t ? int64_t(nb) * nfd : 0) + int64_t(blk) * nfd + i;
    };
    std::vector<double> A = download_bsr(*ctx, V);
    // rows in reference order
    std::vector<std::vector<std::pair<int64_t, double>>> rows(V.n);
    for (int r = 0; r < nb; ++r)
      for (int s = 0; s < host::kSlots; ++s) {
        const int c = V.plan.cols[size_t(r) * host::kSlots + s];
        if (c < 0) continue;
        for (int ii = 0; ii < bs; ++ii)
          for (int jj = 0; jj < bs; ++jj) {
            const double v = A[((size_t(r) * host::kSlots + s) * bs + ii) * bs + jj];
            rows[ref_of(r, ii)].push_back({ref_of(c, jj), v});
          }
      }
    int64_t tot = 0;
    for (auto& rw : rows) tot += int64_t(rw.size());
    *nnz = tot;
    if (!ptr) return;
    int64_t q = 0;
    for (int64_t i = 0; i < V.n; ++i) {
      ptr[i] = q;
      std::sort(rows[i].begin(), rows[i].end());
      for (auto& e : rows[i]) {
        idx[q] = e.first;
        val[q] = e.second;
        ++q;
      }
    }
    ptr[V.n] = q;
  });
}

int hpmg_write_matrix_market(hpmg_ctx* ctx, int level, const char* path) {
  int64_t nnz = 0;
  if (int rc = hpmg_matrix_csr(ctx, level, &nnz, nullptr, nullptr, nullptr)) return rc;
  const int64_t n = level < 0 ? ctx->top().n : ctx->lv.at(level)->n;
  std::vector<int64_t> ptr(n + 1), idx(nnz);
  std::vector<double> val(nnz);
  if (int rc = hpmg_matrix_csr(ctx, level, &nnz, ptr.data(), idx.data(), val.data())) return rc;
  return guarded(ctx, [&] {
    // column by column, rows ascending: the order of a column-major Eigen
    // SparseMatrix walked by write_matrix_market (io.hpp:74-81)
    std::vector<int64_t> cptr(n + 1, 0), order(nnz);
    for (int64_t q = 0; q < nnz; ++q) ++cptr[idx[q] + 1];
    for (int64_t c = 0; c < n; ++c) cptr[c + 1] += cptr[c];
    std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1), rowof(nnz);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t q = ptr[r]; q < ptr[r + 1]; ++q) {
        const int64_t d = fill[idx[q]]++;
        order[d] = q;
        rowof[d] = r;
      }
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)n, (long long)n,
                 (long long)nnz);
    for (int64_t c = 0; c < n; ++c)
      for (int64_t d = cptr[c]; d < cptr[c + 1]; ++d)
        std::fprintf(f, "%lld %lld %.17g\n", (long long)(rowof[d] + 1), (long long)(c + 1), val[order[d]]);
    if (std::fclose(f) != 0) throw std::runtime_error(std::string("write failed: ") + path);
  });
}

int hpmg_spmv(hpmg_ctx* ctx, const double* x, double* y, int flags) {
  return guarded(ctx, [&] {
    in_vec(*ctx, x, ctx->kp, flags);
    dev::spmv(ctx->top().A, ctx->kp, nullptr, ctx->kAp, 0, nullptr, nullptr, ctx->s);
    out_vec(*ctx, ctx->kAp, y, flags);
  });
}

int hpmg_apply(hpmg_ctx* ctx, const double* r, double* z, int flags) {
  return guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    const size_t bytes = sizeof(double) * C.top().n;
    if (flags & HPMG_DEVICE_PTRS) {  // stream-ordered: the caller synchronises hpmg_stream(ctx) as needed
      apply_io(C, r, z);
      return;
    }
    CK(cudaMemcpyAsync(C.io_a, r, bytes, cudaMemcpyHostToDevice, C.s));
    apply_io(C, C.io_a, C.io_b);
    CK(cudaMemcpyAsync(z, C.io_b, bytes, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

int hpmg_apply_trace(hpmg_ctx* ctx, const double* r, double* z, int flags, int cap, int* level, int* entering,
                     double* residual, int* count_out) {
  return guarded(ctx, [&] {
    if (cap < 0 || (cap > 0 && (!level || !entering || !residual))) throw std::invalid_argument("apply_trace: bad buffers");
    hpmg_ctx& C = *ctx;
    std::vector<hpmg_ctx::TraceEntry> tr;
    in_vec(C, r, C.kr, flags);
    C.trace = &tr;
    try {
      apply_blocks(C, C.kr, C.kz);  // the cycle outside the graph, with the norms of every level
    } catch (...) {
      C.trace = nullptr;
      throw;
    }
    C.trace = nullptr;
    out_vec(C, C.kz, z, flags);
    CK(cudaStreamSynchronize(C.s));
    for (int i = 0; i < int(tr.size()) && i < cap; ++i) {
      level[i] = tr[i].level;
      entering[i] = tr[i].entering;
      residual[i] = tr[i].residual;
    }
    if (count_out) *count_out = int(tr.size());
  });
}

int hpmg_apply_batch(hpmg_ctx* ctx, int m, const double* const* r, double* const* z) {
  return guarded(ctx, [&] {
    if (m < 0 || (m > 0 && (!r || !z))) throw std::invalid_argument("apply_batch: bad vector list");
    if (m == 0) return;
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const size_t bytes = sizeof(double) * T.n;
    if (!C.s_h2d) {
      CK(cudaStreamCreateWithFlags(&C.s_h2d, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&C.s_d2h, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        C.bin[i] = dalloc<double>(T.n);
        C.bout[i] = dalloc<double>(T.n);
        for (cudaEvent_t* e : {&C.ev_in[i], &C.ev_used[i], &C.ev_done[i], &C.ev_out[i]})
          CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&C.ev_start, cudaEventDisableTiming));
    }
    // everything below is ordered after the work already queued on the context stream
    CK(cudaEventRecord(C.ev_start, C.s));
    CK(cudaStreamWaitEvent(C.s_h2d, C.ev_start, 0));
    CK(cudaStreamWaitEvent(C.s_d2h, C.ev_start, 0));
    for (int i = 0; i < m; ++i) {
      const int j = i & 1;
      // H2D of vector i into staging j once apply i-2 has consumed it
      if (i >= 2) CK(cudaStreamWaitEvent(C.s_h2d, C.ev_used[j], 0));
      CK(cudaMemcpyAsync(C.bin[j], r[i], bytes, cudaMemcpyHostToDevice, C.s_h2d));
      CK(cudaEventRecord(C.ev_in[j], C.s_h2d));
      // V-cycle i on the context stream (the io graph: permutations + cycle)
      CK(cudaStreamWaitEvent(C.s, C.ev_in[j], 0));
      if (i >= 2) CK(cudaStreamWaitEvent(C.s, C.ev_out[j], 0));  // D2H of result i-2 left bout[j]
      apply_io(C, C.bin[j], C.bout[j]);
      CK(cudaEventRecord(C.ev_used[j], C.s));
      CK(cudaEventRecord(C.ev_done[j], C.s));
      // D2H of result i
      CK(cudaStreamWaitEvent(C.s_d2h, C.ev_done[j], 0));
      CK(cudaMemcpyAsync(z[i], C.bout[j], bytes, cudaMemcpyDeviceToHost, C.s_d2h));
      CK(cudaEventRecord(C.ev_out[j], C.s_d2h));
    }
    // the context stream ends after the last copy-out (callers time on it)
    CK(cudaStreamWaitEvent(C.s, C.ev_out[(m - 1) & 1], 0));
    CK(cudaStreamSynchronize(C.s));
  });
}

int hpmg_smooth(hpmg_ctx* ctx, int level, int which, double* x, const double* b, int sweeps, int flags) {
  return guarded(ctx, [&] {
    Level& V = level < 0 ? ctx->top() : *ctx->lv.at(level);
    if (level >= 0 && level == 0) throw std::invalid_argument("level 0 has no smoother");
    const int n = int(V.n);
    // level vectors are exchanged in the level's own reference order
    std::vector<double> hx(n), hb(n);
    double* dx = ctx->kx;
    double* db = ctx->kb;
    if (level >= 0 && V.n > ctx->top().n) throw std::invalid_argument("level larger than workspace");
    const double* sx = x;
    const double* sb = b;
    double *ta = ctx->io_a, *tb = ctx->io_b;
    if (!(flags & HPMG_DEVICE_PTRS)) {
      CK(cudaMemcpyAsync(ta, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s));
      CK(cudaMemcpyAsync(tb, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s));
      sx = ta;
      sb = tb;
    }
    dev::to_blocks(V.nb, V.k + 1, sx, dx, ctx->s);
    dev::to_blocks(V.nb, V.k + 1, sb, db, ctx->s);
    const int saved = V.steps;
    V.steps = sweeps;
    if (which == 2) {
      const int sm = ctx->opt.smoother;
      ctx->opt.smoother = HPMG_SMOOTH_ADDITIVE;
      smooth(*ctx, V, dx, db, false);
      ctx->opt.smoother = sm;
    } else {
      const int sm = ctx->opt.smoother;
      ctx->opt.smoother = HPMG_SMOOTH_MULTIPLICATIVE;
      smooth(*ctx, V, dx, db, which == 1);
      ctx->opt.smoother = sm;
    }
    V.steps = saved;
    if (flags & HPMG_DEVICE_PTRS) {
      dev::to_reference(V.nb, V.k + 1, dx, x, ctx->s);
    } else {
      dev::to_reference(V.nb, V.k + 1, dx, ta, ctx->s);
      CK(cudaMemcpyAsync(x, ta, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->s));
    }
    CK(cudaStreamSynchronize(ctx->s));
    (void)hx;
    (void)hb;
  });
}

int hpmg_pcg(hpmg_ctx* ctx, const double* b, double* x, const hpmg_krylov_opts* o, hpmg_solve_stats* st, int flags) {
  return guarded(ctx, [&] {
    in_vec(*ctx, b, ctx->kb, flags);
    in_vec(*ctx, x, ctx->kx, flags);
    *st = pcg_device(*ctx, *o);
    out_vec(*ctx, ctx->kx, x, flags);
  });
}

int hpmg_gmres(hpmg_ctx* ctx, const double* b, double* x, const hpmg_krylov_opts* o, hpmg_solve_stats* st, int flags) {
  return guarded(ctx, [&] {
    in_vec(*ctx, b, ctx->kb, flags);
    in_vec(*ctx, x, ctx->kx, flags);
    *st = gmres_device(*ctx, *o);
    out_vec(*ctx, ctx->kx, x, flags);
  });
}

int hpmg_uzawa(hpmg_ctx* ctx, const hpmg_uzawa_opts* o, double* velocity, double* pressure, hpmg_uzawa_report* rep) {
  return guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const int ne = T.ne;
    std::memset(rep, 0, sizeof(*rep));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, C.s));
    dev::fill(C.pres, 0.0, ne, C.s);
    if (o->initial_velocity) {  // warm start: Constraints::to_free of the given full velocity
      std::vector<double> u0(T.n);
      for (size_t i = 0; i < C.free_to_full.size(); ++i) u0[i] = o->initial_velocity[C.free_to_full[i]];
      in_vec(C, u0.data(), C.kx, 0);
      CK(cudaStreamSynchronize(C.s));  // u0 is a host temporary
    } else {
      dev::fill(C.kx, 0.0, T.n, C.s);
    }
    rep->converged = 1;
    for (int it = 0; it < o->outer_iterations && it < 64; ++it) {
      dev::uzawa_rhs(T.nb, T.bs, C.rhs, T.row_elems, T.geo, C.pres, C.kb, C.s);
      hpmg_solve_stats st = C.advected ? gmres_device(C, o->krylov) : pcg_device(C, o->krylov);
      rep->inner_iterations[it] = st.iterations;
      rep->n_outer = it + 1;
      if (st.not_applicable) {
        rep->not_applicable = 1;
        rep->converged = 0;
        break;
      }
      rep->converged = rep->converged && st.converged;
      dev::uzawa_div(ne, T.bs, T.elem_facets, T.facet_block, C.g_fac, C.kx, T.geo, C.div, C.s);
      dev::uzawa_pressure(ne, C.div, T.geo, C.opt.inv_eps, C.pres, C.enclosed ? 1 : 0, C.red, C.sc, S_PS, S_PA,
                          S_PMAX, C.s);
      read_scalars(C);
      rep->divergence_history[it] = C.sc_host[S_PMAX];
    }
    CK(cudaEventRecord(e1, C.s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    rep->seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rep->n_outer > 0) rep->final_divergence = rep->divergence_history[rep->n_outer - 1];
    // velocity: g_full with free entries overwritten (Constraints::to_full)
    std::vector<double> u(T.n);
    dev::to_reference(T.nb, T.k + 1, C.kx, C.io_b, C.s);
    CK(cudaMemcpyAsync(u.data(), C.io_b, sizeof(double) * T.n, cudaMemcpyDeviceToHost, C.s));
    CK(cudaMemcpyAsync(pressure, C.pres, sizeof(double) * ne, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    std::memcpy(velocity, C.g_full.data(), sizeof(double) * C.g_full.size());
    for (size_t i = 0; i < C.free_to_full.size(); ++i) velocity[C.free_to_full[i]] = u[i];
  });
}

int hpmg_interpolate_hdg(hpmg_ctx* ctx, hpmg_field_fn field, void* user, double* compound_full, double* interior) {
  return guarded(ctx, [&] {
    if (!field) throw std::invalid_argument("interpolate_hdg needs a field");
    hpmg_ctx& C = *ctx;
    const int k = C.opt.k;
    auto T = host::build_ref_tensors(k);
    const host::HdgField u = host::interpolate_hdg(C.mesh.back(), k, *T, [&](double x, double y, double* o) {
      field(x, y, o, user);
    });
    std::memcpy(compound_full, u.compound.data(), sizeof(double) * u.compound.size());
    if (!u.interior.empty()) std::memcpy(interior, u.interior.data(), sizeof(double) * u.interior.size());
  });
}

double hpmg_rt_l2_norm(hpmg_ctx* ctx, const double* compound_full, const double* interior) {
  double out = -1.0;
  const int rc = guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const DevRef& R = C.opt.k > 0 ? C.refk : C.ref0;
    const size_t nfull = C.g_full.size(), ni = size_t(T.ne) * R.T.no;
    DevTemps tmp;
    double* comp = tmp.add(dalloc<double>(nfull));
    double* di = tmp.add(dalloc<double>(std::max<size_t>(ni, 1)));
    CK(cudaMemcpyAsync(comp, compound_full, sizeof(double) * nfull, cudaMemcpyHostToDevice, C.s));
    if (ni) CK(cudaMemcpyAsync(di, interior, sizeof(double) * ni, cudaMemcpyHostToDevice, C.s));
    dev::rt_norm2(R.T, T.geo, T.ne, T.elem_facets, comp, di, C.red, C.sc + S_TMP, C.s);
    read_scalars(C);
    out = std::sqrt(C.sc_host[S_TMP]);
  });
  return rc == 0 ? out : -1.0;
}

/// Process-wide pinned staging buffer for the large host <-> device copies of
/// the host-pointer API (grow-only, kept across contexts like the device
/// pool): a pageable copy runs through the driver's small staging buffers at
/// a fraction of the link rate; here the DMA runs at full rate and host
/// threads move the data between the staging buffer and the caller's arrays.
struct PinnedStage {
  std::mutex m;
  char* p = nullptr;
  size_t cap = 0;
  char* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      CK(cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocDefault));
      cap = bytes;
    }
    return p;
  }
};
PinnedStage& pinned_stage() {
  static PinnedStage st;
  return st;
}
/// memcpy on up to 8 host threads (large copies are limited per thread by
/// page faults on the destination and by a single core's bandwidth)
void par_memcpy(void* dst, const void* src, size_t bytes) {
  const int nt = int(std::min<size_t>(8, bytes >> 22) + 1);
  if (nt == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([=] {
      const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
      std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
  for (auto& x : th) x.join();
}

int hpmg_recover(hpmg_ctx* ctx, const double* velocity_full, double* interior, double* p_ortho, double* grad) {
  return guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const DevRef& R = C.opt.k > 0 ? C.refk : C.ref0;
    const int ne = T.ne, no = R.T.no, np = R.T.ns - 1, ng = 4 * R.T.ns;
    const size_t nfull = C.g_full.size();
    DevTemps tmp;
    double* comp = tmp.add(dalloc<double>(nfull));
    double* di = tmp.add(dalloc<double>(size_t(ne) * std::max(no, 1)));
    double* dp = tmp.add(dalloc<double>(size_t(ne) * std::max(np, 1)));
    double* dg = tmp.add(dalloc<double>(size_t(ne) * ng));
    const size_t bi = sizeof(double) * size_t(ne) * no, bp = sizeof(double) * size_t(ne) * np,
                 bg = sizeof(double) * size_t(ne) * ng, bv = sizeof(double) * nfull;
    PinnedStage& st = pinned_stage();
    std::lock_guard<std::mutex> lock(st.m);
    char* h = st.get(std::max(bv, bi + bp + bg));
    par_memcpy(h, velocity_full, bv);
    CK(cudaMemcpyAsync(comp, h, bv, cudaMemcpyHostToDevice, C.s));
    dev::recover(R.T, T.geo, ne, C.fine_prm, C.fine_load, C.fine_lstride, T.elem_facets, (long long)(nfull / 2), comp,
                 di, dp, dg, C.s, C.fine_wind, C.fine_mass);
    // the staging buffer is reused for the results only after the upload has
    // been consumed: the copies below queue behind the recovery kernel
    if (no) CK(cudaMemcpyAsync(h, di, bi, cudaMemcpyDeviceToHost, C.s));
    if (np) CK(cudaMemcpyAsync(h + bi, dp, bp, cudaMemcpyDeviceToHost, C.s));
    CK(cudaMemcpyAsync(h + bi + bp, dg, bg, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    if (no) par_memcpy(interior, h, bi);
    if (np) par_memcpy(p_ortho, h + bi, bp);
    par_memcpy(grad, h + bi + bp, bg);
  });
}

namespace {

/// Post-processing tables and element origins of the finest mesh, on first use.
const dev::PostT& post_tables(hpmg_ctx& C) {
  if (C.post_t.Lv) return C.post_t;
  const int k = C.opt.k;
  const DevRef& R = k > 0 ? C.refk : C.ref0;
  auto T = host::build_ref_tensors(k);
  const host::PostTables H = host::build_post_tables(*T);
  auto up = [&](const std::vector<double>& v) {
    double* p = dupload(v, C.s);
    C.post.owned.push_back(p);
    return (const double*)p;
  };
  const host::TriMesh& M = C.mesh.back();
  std::vector<double> x0(size_t(2) * M.ne());
  for (int e = 0; e < M.ne(); ++e) {
    x0[2 * e] = M.vx[M.ev[e][0]];
    x0[2 * e + 1] = M.vy[M.ev[e][0]];
  }
  dev::PostT P;
  P.k = k;
  P.nfd = R.T.nfd;
  P.nrt = R.T.nrt;
  P.no = R.T.no;
  P.ns = R.T.ns;
  P.nh = H.nh;
  P.Lv = R.T.Lv;
  P.Kh = up(H.Kh);
  P.Bh = up(H.Bh);
  P.ref_mean = H.ref_mean;
  P.nqe = H.nqe;
  P.ex = up(H.ex);
  P.ew = up(H.ew);
  P.eval = up(H.eval);
  P.ediv = up(H.ediv);
  P.escal = up(H.escal);
  P.ehi = up(H.ehi);
  C.post_x0 = up(x0);
  C.post_red = const_cast<double*>(up(std::vector<double>(size_t(4) * dev::kRedBlocks + 4, 0.0)));
  CK(cudaStreamSynchronize(C.s));
  C.post_t = P;
  return C.post_t;
}

}  // namespace

int hpmg_postprocess(hpmg_ctx* ctx, const double* velocity_full, const double* interior, const double* grad,
                     double* post) {
  return guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const dev::PostT& P = post_tables(C);
    const int ne = T.ne;
    const size_t nfull = C.g_full.size(), ni = size_t(ne) * P.no, ng = size_t(ne) * 4 * P.ns, np = size_t(ne) * 2 * P.nh;
    DevTemps tmp;
    double* comp = tmp.add(dalloc<double>(nfull));
    double* di = tmp.add(dalloc<double>(std::max<size_t>(ni, 1)));
    double* dg = tmp.add(dalloc<double>(ng));
    double* dp = tmp.add(dalloc<double>(np));
    CK(cudaMemcpyAsync(comp, velocity_full, sizeof(double) * nfull, cudaMemcpyHostToDevice, C.s));
    if (ni) CK(cudaMemcpyAsync(di, interior, sizeof(double) * ni, cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpyAsync(dg, grad, sizeof(double) * ng, cudaMemcpyHostToDevice, C.s));
    dev::postprocess(P, T.geo, ne, T.elem_facets, C.opt.nu, comp, di, dg, dp, C.s);
    CK(cudaMemcpyAsync(post, dp, sizeof(double) * np, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

int hpmg_measure_errors(hpmg_ctx* ctx, const double* velocity_full, const double* interior, const double* grad,
                        const double* post, hpmg_field_fn u_exact, void* u_user, hpmg_tensor_fn grad_exact,
                        void* g_user, double* out) {
  return guarded(ctx, [&] {
    if (!u_exact || !grad_exact) throw std::invalid_argument("measure_errors needs the exact velocity and gradient");
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    const dev::PostT& P = post_tables(C);
    const int ne = T.ne;
    // the library's own analytic flows are evaluated on the device
    int kind = 0;
    if (u_exact == hpmg_field_mms_velocity && grad_exact == hpmg_tensor_mms_gradient) kind = 1;
    if (u_exact == hpmg_field_linear_flow && grad_exact == hpmg_tensor_linear_flow_gradient) kind = 2;
    const size_t nfull = C.g_full.size(), ni = size_t(ne) * P.no, ng = size_t(ne) * 4 * P.ns, np = size_t(ne) * 2 * P.nh;
    DevTemps tmp;
    auto alloc = [&](size_t n) { return tmp.add(dalloc<double>(std::max<size_t>(n, 1))); };
    double *comp = alloc(nfull), *di = alloc(ni), *dg = alloc(ng), *dp = alloc(np), *ue = nullptr, *ge = nullptr;
    CK(cudaMemcpyAsync(comp, velocity_full, sizeof(double) * nfull, cudaMemcpyHostToDevice, C.s));
    if (ni) CK(cudaMemcpyAsync(di, interior, sizeof(double) * ni, cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpyAsync(dg, grad, sizeof(double) * ng, cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpyAsync(dp, post, sizeof(double) * np, cudaMemcpyHostToDevice, C.s));
    std::vector<double> hu, hg;
    if (kind == 0) {  // user callbacks: tabulate at the physical error-rule points
      const host::TriMesh& M = C.mesh.back();
      auto T0 = host::build_ref_tensors(C.opt.k);
      const host::PostTables H = host::build_post_tables(*T0);
      hu.resize(size_t(ne) * H.nqe * 2);
      hg.resize(size_t(ne) * H.nqe * 4);
      for (int e = 0; e < ne; ++e) {
        const auto& v = M.ev[e];
        const double x0 = M.vx[v[0]], y0 = M.vy[v[0]];
        const double j00 = M.vx[v[1]] - x0, j10 = M.vy[v[1]] - y0, j01 = M.vx[v[2]] - x0, j11 = M.vy[v[2]] - y0;
        for (int q = 0; q < H.nqe; ++q) {
          const double xh = H.ex[2 * q], yh = H.ex[2 * q + 1];
          const double x = x0 + j00 * xh + j01 * yh, y = y0 + j10 * xh + j11 * yh;
          const size_t o = size_t(e) * H.nqe + q;
          u_exact(x, y, &hu[2 * o], u_user);
          grad_exact(x, y, &hg[4 * o], g_user);
        }
      }
      ue = alloc(hu.size());
      ge = alloc(hg.size());
      CK(cudaMemcpyAsync(ue, hu.data(), sizeof(double) * hu.size(), cudaMemcpyHostToDevice, C.s));
      CK(cudaMemcpyAsync(ge, hg.data(), sizeof(double) * hg.size(), cudaMemcpyHostToDevice, C.s));
    }
    double* partial = C.post_red;
    dev::measure_errors(P, T.geo, C.post_x0, ne, T.elem_facets, C.opt.nu, comp, di, dg, dp, kind, ue, ge, partial,
                        partial + 4 * dev::kRedBlocks, C.s);
    CK(cudaMemcpyAsync(out, partial + 4 * dev::kRedBlocks, sizeof(double) * 4, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

void* hpmg_stream(hpmg_ctx* ctx) { return ctx->s; }

double hpmg_spmv_bytes(const hpmg_ctx* ctx) {
  const Level& T = const_cast<hpmg_ctx*>(ctx)->top();
  return T.bytes_spmv;
}

double hpmg_vcycle_bytes(const hpmg_ctx* ctx, double* parts) {
  auto& C = *const_cast<hpmg_ctx*>(ctx);
  double p[8] = {0};
  const int q = C.opt.cycle == HPMG_CYCLE_W ? 2 : 1;
  if (C.opt.k > 0) {
    const Level& H = *C.head;
    p[0] = 2.0 * H.steps * H.bytes_sweep;
    // mode-0 rows of the head residual: 2 of bs rows per block
    p[1] = H.bytes_spmv * 2.0 / H.bs + 32.0 * C.lv[C.L]->n;
  }
  // visits of level l: q^(L-l)
  for (int l = C.L; l >= 1; --l) {
    const Level& V = *C.lv[l];
    const double visits = std::pow(double(q), C.L - l);
    p[2] += visits * 2.0 * V.steps * V.bytes_sweep;
    p[3] += visits * (V.bytes_spmv + 8.0 * V.n);
    // B_P = 12 nnz(P) + 16 n_l, for P and for P^T
    p[4] += visits * 2.0 * (12.0 * V.p_nnz + 16.0 * V.n);
  }
  p[5] = std::pow(double(q), C.L) * 8.0 * double(C.n0) * C.n0;
  double tot = 0;
  for (int i = 0; i < 6; ++i) tot += p[i];
  // streamed bytes of this implementation's sweeps (records, not in `tot`)
  auto stream = [](const Level& V) { return V.bytes_stream > 0 ? V.bytes_stream : V.bytes_sweep; };
  if (C.opt.k > 0) p[6] = 2.0 * C.head->steps * stream(*C.head);
  for (int l = C.L; l >= 1; --l)
    p[7] += std::pow(double(q), C.L - l) * 2.0 * C.lv[l]->steps * stream(*C.lv[l]);
  if (parts)
    for (int i = 0; i < 8; ++i) parts[i] = p[i];
  return tot;
}

double hpmg_time_spmv(hpmg_ctx* ctx, int reps, double* bytes) {
  double ms_per = -1;
  guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    Level& T = C.top();
    if (bytes) {  // as stored: ELL-BSR values + slot columns, x read once, y written
      bytes[0] = double(T.nb) * host::kSlots * T.bs * T.bs * 8.0 + double(T.nb) * host::kSlots * 4.0 + 16.0 * T.n;
      bytes[1] = T.bytes_spmv;  // SURVEY 8(d) reference CSR accounting
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) dev::spmv(T.A, C.kp, nullptr, C.kAp, 0, nullptr, nullptr, C.s);
    CK(cudaEventRecord(e0, C.s));
    for (int i = 0; i < reps; ++i) dev::spmv(T.A, C.kp, nullptr, C.kAp, 0, nullptr, nullptr, C.s);
    CK(cudaEventRecord(e1, C.s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_per = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
  return ms_per;
}

double hpmg_time_apply(hpmg_ctx* ctx, int reps, double* phase_ms) {
  double ms_per = -1;
  guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) apply_graph(C);
    CK(cudaEventRecord(e0, C.s));
    for (int i = 0; i < reps; ++i) apply_graph(C);
    CK(cudaEventRecord(e1, C.s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_per = ms / reps;
    if (phase_ms && C.opt.k > 0) {
      // each phase captured as a graph of its own and timed over `reps`
      // launches: head pre-sweep (from x = 0), head residual (E^T injection),
      // the lowest-order h-cycle with the embedding, head post-sweep
      for (int i = 0; i < 8; ++i) phase_ms[i] = 0;
      Level& H = *C.head;
      Level& F = *C.lv[C.L];
      auto phase = [&](auto fn) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(C.s, cudaStreamCaptureModeThreadLocal));
        fn();
        CK(cudaStreamEndCapture(C.s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, C.s));
        CK(cudaEventRecord(e0, C.s));
        for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, C.s));
        CK(cudaEventRecord(e1, C.s));
        CK(cudaEventSynchronize(e1));
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        cudaGraphExecDestroy(ge);
        return double(t) / reps;
      };
      phase_ms[0] = phase([&] {
        dev::fill(C.kz, 0.0, H.n, C.s);
        smooth(C, H, C.kz, C.kr, false, true);
      });
      phase_ms[1] = phase([&] { dev::inject_residual(H.A0, C.kz, C.kr, F.b, C.s, F.x); });
      phase_ms[2] = phase([&] {
        h_cycle(C, C.L, F.b, F.x);
        dev::embed_add(H.nb, H.bs, F.x, C.kz, C.s);
      });
      phase_ms[3] = phase([&] { smooth(C, H, C.kz, C.kr, true); });
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
  return ms_per;
}

int hpmg_kernel_launches_per_apply(const hpmg_ctx* ctx) {
  return ctx->io_launches > 0 ? ctx->io_launches : ctx->launches_per_apply;
}

/// Development hook: arm (1) / disarm (0) the one-CTA sweep timeline and copy
/// it out (4096 clock64 stamps: per pass start, data ready, residual done, end).
void hpmg_debug_small_trace(int arm, long long* out) { dev::small_trace(arm, out); }
void hpmg_debug_gm_trace(int arm, long long* out) { dev::gm_trace(arm, out); }
void hpmg_debug_sweep_trace(long long* out) { dev::sweep_trace(out); }

/// Event-instrumented V-cycle (no graph): out[2l], out[2l+1] = pre/post part
/// of level l (l = 1..L) in ms, out[0] = coarse solve, out[2(L+1)..+2] = head
/// pre-sweep, residual+embed, post-sweep. Returns the number of entries.
double hpmg_debug_loop_probe(hpmg_ctx* ctx, int mode, int iters) {
  double ms_per = -1;
  guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    double* c = C.sc + 15;
    try {
      GK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h, hi = 0;
      GK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      const int pm = mode >= 32 ? mode - 32 : -1;  // PCG-shaped body, parts by bit
      if (mode == 2 || (pm >= 0 && (pm & 4)))
        GK(cudaGraphConditionalHandleCreate(&hi, g, (pm >= 0 && (pm & 2)) ? 0 : 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams wp = {};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      cudaGraphNode_t wnode;
      GK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
      capture_body(C, wp.conditional.phGraph_out[0], 0, [&] {
        if (mode == 1) apply_blocks(C, C.kr, C.kz);
        if (mode == 2) {
          cudaGraph_t br = add_conditional(C.s, hi, cudaGraphCondTypeIf);
          capture_body(C, br, 1, [&] { apply_blocks(C, C.kr, C.kz); });
        }
        if (mode == 3) {
          cudaGraph_t child;
          GK(cudaGraphCreate(&child, 0));
          capture_body(C, child, 1, [&] { apply_blocks(C, C.kr, C.kz); });
          cudaStreamCaptureStatus cs;
          const cudaGraphNode_t* deps = nullptr;
          size_t ndeps = 0;
          cudaGraph_t capg;
          GK(cudaStreamGetCaptureInfo(C.s, &cs, nullptr, &capg, &deps, &ndeps));
          cudaGraphNode_t cn;
          GK(cudaGraphAddChildGraphNode(&cn, capg, deps, ndeps, child));
          GK(cudaStreamUpdateCaptureDependencies(C.s, &cn, 1, cudaStreamSetCaptureDependencies));
          cudaGraphDestroy(child);
        }
        if (pm >= 0 && (pm & 64)) {  // the round-2 PCG body: V-cycle | r.z | A p' | update
          const int64_t n = C.top().n;
          apply_blocks(C, C.kr, C.kz);
          if (pm & 8) dev::pcg_loop_rz(C.kr, C.kz, n, C.sc, C.red, h, C.s);
          if (pm & 1) dev::pcg_spmv_dir(C.top().A, C.kp, C.kz, C.kAp, 1, C.sc, C.red, C.s);
          if (pm & 2) dev::pcg_loop_update(C.kx, C.kr, C.kp, C.kz, C.kAp, n, 1, C.sc, C.red, h, C.s);
        } else if (pm >= 0) {
          const int64_t n = C.top().n;
          if (pm & 1) dev::pcg_spmv_dir(C.top().A, C.kp, C.kz, C.kAp, 1, C.sc, C.red, C.s);
          if (pm & 2) dev::pcg_loop_update(C.kx, C.kr, C.kp, C.kz, C.kAp, n, 1, C.sc, C.red, h, C.s);
          auto branch = [&] {
            apply_blocks(C, C.kr, C.kz);
            if (pm & 8) dev::pcg_loop_rz(C.kr, C.kz, n, C.sc, C.red, h, C.s);
            if (pm & 16) dev::pcg_loop_direction(C.kp, C.kz, n, C.sc, C.s);
          };
          if (pm & 4) {
            cudaGraph_t br = add_conditional(C.s, hi, cudaGraphCondTypeIf);
            capture_body(C, br, 1, branch);
          } else {
            if (pm & 8) dev::pcg_loop_rz(C.kr, C.kz, n, C.sc, C.red, h, C.s);
            if (pm & 16) dev::pcg_loop_direction(C.kp, C.kz, n, C.sc, C.s);
          }
        }
        dev::loop_countdown(c, h, C.s);
      });
      GK(cudaGraphInstantiate(&ge, g, 0));
    } catch (const GraphError& e) {
      if (g) cudaGraphDestroy(g);
      throw std::runtime_error(std::string("loop probe: ") + cudaGetErrorString(e.e));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    if (mode >= 32) {  // a live PCG state: r = b, p = z = M r, target 0
      const int64_t nn = C.top().n;
      dev::copy(C.kr, C.kb, nn, C.s);
      dev::fill(C.kx, 0.0, nn, C.s);
      apply_blocks(C, C.kr, C.kz);
      dev::copy(C.kp, C.kz, nn, C.s);
      dev::dot(C.kr, C.kz, nn, C.red, C.sc + dev::kScRZ, C.s);
      dev::pcg_loop_init(C.sc, 0.0, 1e9, C.s);
    }
    const double warm = 3.0, n = double(iters);
    CK(cudaMemcpyAsync(c, &warm, sizeof(double), cudaMemcpyHostToDevice, C.s));
    CK(cudaGraphLaunch(ge, C.s));
    CK(cudaMemcpyAsync(c, &n, sizeof(double), cudaMemcpyHostToDevice, C.s));
    CK(cudaEventRecord(e0, C.s));
    CK(cudaGraphLaunch(ge, C.s));
    CK(cudaEventRecord(e1, C.s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_per = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  });
  return ms_per;
}

int hpmg_profile_levels(hpmg_ctx* ctx, int reps, double* out) {
  int nout = 0;
  guarded(ctx, [&] {
    hpmg_ctx& C = *ctx;
    const int L = C.L;
    nout = 2 * (L + 1) + 3;
    for (int i = 0; i < nout; ++i) out[i] = 0;
    std::vector<cudaEvent_t> ev(2 * (L + 1) + 8);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    auto el = [&](int a, int b) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[a], ev[b]);
      return double(ms);
    };
    for (int r = 0; r < reps; ++r) {
      // walk down: pre parts, record an event after each level's pre part
      const double* b = C.opt.k > 0 ? C.lv[L]->b : C.kr;
      double* x = C.opt.k > 0 ? C.lv[L]->x : C.kz;
      int e = 0;
      CK(cudaEventRecord(ev[e++], C.s));  // 0
      if (C.opt.k > 0) {
        Level& H = *C.head;
        dev::fill(C.kz, 0.0, H.n, C.s);
        smooth(C, H, C.kz, C.kr, false);
        CK(cudaEventRecord(ev[e++], C.s));  // 1
        dev::inject_residual(H.A0, C.kz, C.kr, C.lv[L]->b, C.s);
        CK(cudaEventRecord(ev[e++], C.s));  // 2
      }
      const int ebase = e;
      std::vector<const double*> bs(L + 1);
      std::vector<double*> xs(L + 1);
      bs[L] = b;
      xs[L] = x;
      for (int l = L; l >= 1; --l) {
        Level& V = *C.lv[l];
        Level& W = *C.lv[l - 1];
        if (V.small) {
          dev::small_pre(V.A, V.srec, V.d_passes, V.npass, V.steps, V.PT, bs[l], xs[l], V.r, W.b, C.s);
        } else {
          dev::fill(xs[l], 0.0, V.n, C.s);
          smooth(C, V, xs[l], bs[l], false);
          dev::spmv(V.A, xs[l], bs[l], V.r, 1, nullptr, nullptr, C.s);
          dev::restrict_(V.PT, V.r, W.b, C.s);
        }
        bs[l - 1] = W.b;
        xs[l - 1] = W.x;
        CK(cudaEventRecord(ev[e++], C.s));
      }
      dev::dense_gemv(C.n0, C.coarse_inv, bs[0], xs[0], C.gemv_work, C.s);
      CK(cudaEventRecord(ev[e++], C.s));
      for (int l = 1; l <= L; ++l) {
        Level& V = *C.lv[l];
        Level& W = *C.lv[l - 1];
        if (V.small) {
          dev::small_post(V.A, V.srec, V.d_passes, V.npass, V.steps, V.Pm, W.x, bs[l], xs[l], C.s);
        } else {
          dev::prolong_add(V.Pm, W.x, xs[l], C.s);
          smooth(C, V, xs[l], bs[l], true);
        }
        CK(cudaEventRecord(ev[e++], C.s));
      }
      if (C.opt.k > 0) {
        Level& H = *C.head;
        dev::embed_add(H.nb, H.bs, C.lv[L]->x, C.kz, C.s);
        smooth(C, H, C.kz, C.kr, true);
        CK(cudaEventRecord(ev[e++], C.s));
      }
      CK(cudaEventSynchronize(ev[e - 1]));
      // pre part of level l: between consecutive events going down
      int idx = ebase;
      for (int l = L; l >= 1; --l, ++idx) out[2 * l] += el(idx - 1, idx) / reps;
      out[0] += el(idx - 1, idx) / reps;  // coarse
      ++idx;
      for (int l = 1; l <= L; ++l, ++idx) out[2 * l + 1] += el(idx - 1, idx) / reps;
      if (C.opt.k > 0) {
        out[2 * (L + 1)] += el(0, 1) / reps;
        out[2 * (L + 1) + 1] += el(1, 2) / reps;
        out[2 * (L + 1) + 2] += el(idx - 1, idx) / reps;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
  return nout;
}

double hpmg_setup_seconds(const hpmg_ctx* ctx, double* parts) {
  if (parts)
    for (int i = 0; i < 8; ++i) parts[i] = ctx->setup_parts[i];
  return ctx->setup_parts[6];
}

void hpmg_field_config5_wind(double x, double y, double* out, void*) {
  const double s = std::sin(M_PI * x), t = std::sin(M_PI * y);
  out[0] = M_PI * s * s * std::sin(2 * M_PI * y);
  out[1] = -M_PI * std::sin(2 * M_PI * x) * t * t;
}
void hpmg_field_rotation(double x, double y, double* out, void*) {
  out[0] = y - 0.5;
  out[1] = 0.5 - x;
}
// manufactured flow (reference inc/manufactured.hpp:16-65): bump G(s) = s^2 (s-1)^2
namespace {
inline double mb(double s) { return s * s * (s - 1.0) * (s - 1.0); }
inline double mb1(double s) { return 2.0 * s * (s - 1.0) * (2.0 * s - 1.0); }
inline double mb2(double s) { return 12.0 * s * s - 12.0 * s + 2.0; }
inline double mb3(double s) { return 24.0 * s - 12.0; }
void mms_parts(double x, double y, double* u, double* g, double* lap, double* gp) {
  u[0] = -mb(x) * mb1(y);
  u[1] = mb1(x) * mb(y);
  g[0] = -mb1(x) * mb1(y);
  g[1] = -mb(x) * mb2(y);
  g[2] = mb2(x) * mb(y);
  g[3] = mb1(x) * mb1(y);
  lap[0] = -mb2(x) * mb1(y) - mb(x) * mb3(y);
  lap[1] = mb3(x) * mb(y) + mb1(x) * mb2(y);
  gp[0] = (1.0 - 2.0 * x) * (1.0 - y);
  gp[1] = x * x - x;
}
}  // namespace
void hpmg_field_mms_velocity(double x, double y, double* out, void*) {
  out[0] = -mb(x) * mb1(y);
  out[1] = mb1(x) * mb(y);
}
void hpmg_tensor_mms_gradient(double x, double y, double* out, void*) {
  out[0] = -mb1(x) * mb1(y);
  out[1] = -mb(x) * mb2(y);
  out[2] = mb2(x) * mb(y);
  out[3] = mb1(x) * mb1(y);
}
double hpmg_mms_pressure(double x, double y) { return x * (1.0 - x) * (1.0 - y) - 1.0 / 12.0; }
void hpmg_field_mms_stokes_load(double x, double y, double* out, void* user) {
  const double* p = static_cast<const double*>(user);
  const double nu = p[0], beta = p[1];
  double u[2], g[4], l[2], gp[2];
  mms_parts(x, y, u, g, l, gp);
  out[0] = -nu * l[0] + beta * u[0] + gp[0];
  out[1] = -nu * l[1] + beta * u[1] + gp[1];
}
void hpmg_field_mms_ns_load(double x, double y, double* out, void* user) {
  const double nu = *static_cast<const double*>(user);
  double u[2], g[4], l[2], gp[2];
  mms_parts(x, y, u, g, l, gp);
  out[0] = -nu * l[0] + (g[0] * u[0] + g[1] * u[1]) + gp[0];
  out[1] = -nu * l[1] + (g[2] * u[0] + g[3] * u[1]) + gp[1];
}
void hpmg_field_linear_flow(double x, double y, double* out, void*) {
  out[0] = 1 + 2 * y + 3 * x;
  out[1] = 4 - 3 * y + 5 * x;
}
void hpmg_tensor_linear_flow_gradient(double, double, double* out, void*) {
  out[0] = 3;
  out[1] = 2;
  out[2] = 5;
  out[3] = -3;
}
void hpmg_field_linear_flow_load(double x, double y, double* out, void*) {
  hpmg_field_linear_flow(x, y, out, nullptr);
  out[0] = 2.0 * out[0] + 1.0;
  out[1] = 2.0 * out[1] + 1.0;
}
void hpmg_field_lid_unit(double x, double y, double* out, void*) {
  out[0] = y > 1.0 - 1e-12 ? 1.0 : 0.0;
  out[1] = 0.0;
  (void)x;
}

void hpmg_seeded_load(int n, unsigned seed, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> d(lo, hi);
  for (size_t i = 0; i < size_t(4) * n * n; ++i) out[i] = d(rng);
}

int hpmg_structured_to_elements(const hpmg_ctx* ctx, int n, const double* S, double* out) {
  const host::TriMesh& m = ctx->mesh.back();
  for (int e = 0; e < m.ne(); ++e) {
    const auto& v = m.ev[e];
    const double cx = (m.vx[v[0]] + m.vx[v[1]] + m.vx[v[2]]) / 3.0, cy = (m.vy[v[0]] + m.vy[v[1]] + m.vy[v[2]]) / 3.0;
    int i = int(std::floor(cx * n)), j = int(std::floor(cy * n));
    i = std::min(n - 1, std::max(0, i));
    j = std::min(n - 1, std::max(0, j));
    const bool lower = (cx - double(i) / n) >= (cy - double(j) / n);
    const size_t s = (size_t(j) * n + i) * 2 + (lower ? 0 : 1);
    out[2 * e] = S[2 * s];
    out[2 * e + 1] = S[2 * s + 1];
  }
  return HPMG_OK;
}

namespace {
thread_local std::vector<double> t_xy;
thread_local std::vector<int> t_el, t_tags;
int fill_desc(const host::TriMesh& m, int levels, hpmg_mesh_desc* out) {
  t_xy.clear();
  t_el.clear();
  t_tags.clear();
  for (int v = 0; v < m.nv(); ++v) {
    t_xy.push_back(m.vx[v]);
    t_xy.push_back(m.vy[v]);
  }
  for (int e = 0; e < m.ne(); ++e)
    for (int q = 0; q < 3; ++q) t_el.push_back(m.ev[e][q]);
  for (int f = 0; f < m.nf(); ++f)
    if (m.ftag[f] == host::kTagOutflow) {
      t_tags.push_back(m.fa[f]);
      t_tags.push_back(m.fb[f]);
      t_tags.push_back(host::kTagOutflow);
    }
  out->n_vertices = m.nv();
  out->xy = t_xy.data();
  out->n_elements = m.ne();
  out->elements = t_el.data();
  out->n_tag_overrides = int(t_tags.size() / 3);
  out->tag_overrides = t_tags.data();
  out->levels = levels;
  return HPMG_OK;
}
}  // namespace

int hpmg_unit_square_mesh(int n, int levels, hpmg_mesh_desc* out) { return fill_desc(host::unit_square(n), levels, out); }

int hpmg_plan_check(const hpmg_mesh_desc* md, int k, int level, int64_t* out, int out_len) {
  try {
    host::TriMesh m;
    for (int v = 0; v < md->n_vertices; ++v) {
      m.vx.push_back(md->xy[2 * v]);
      m.vy.push_back(md->xy[2 * v + 1]);
    }
    for (int e = 0; e < md->n_elements; ++e)
      m.ev.push_back({md->elements[3 * e], md->elements[3 * e + 1], md->elements[3 * e + 2]});
    m.build_facets();
    const int target = level < 0 ? md->levels - 1 : level;
    for (int l = 0; l < target; ++l) {
      host::Refinement R;
      m = host::refine(m, R);
    }
    host::LevelPlan P = host::make_level(m, level < 0 ? k : 0);
    // double cover
    std::vector<int> seen(P.nb, 0);
    for (int p = 0; p < P.npatch; ++p)
      for (int q = 0; q < P.patch_nf[p]; ++q) seen[P.patch_fac[size_t(p) * host::kMaxPatchF + q]]++;
    bool cover = true;
    for (int c : seen) cover = cover && c == 2;
    // independence inside a wave: no shared block, no coupling between blocks
    std::vector<int> owner(P.nb, -1), wave_of(P.npatch, -1);
    bool indep = true;
    for (int w = 0; w + 1 < int(P.wave_ptr.size()); ++w) {
      std::vector<int> touched;
      for (int p = P.wave_ptr[w]; p < P.wave_ptr[w + 1]; ++p) {
        wave_of[p] = w;
        for (int q = 0; q < P.patch_nf[p]; ++q) {
          const int f = P.patch_fac[size_t(p) * host::kMaxPatchF + q];
          if (owner[f] >= 0 && owner[f] != p) indep = false;
          owner[f] = p;
          touched.push_back(f);
        }
      }
      for (int p = P.wave_ptr[w]; p < P.wave_ptr[w + 1]; ++p)
        for (int q = 0; q < P.patch_nf[p]; ++q) {
          const int f = P.patch_fac[size_t(p) * host::kMaxPatchF + q];
          for (int s = 0; s < host::kSlots; ++s) {
            const int c = P.cols[size_t(f) * host::kSlots + s];
            if (c >= 0 && owner[c] >= 0 && owner[c] != p) indep = false;
          }
        }
      for (int f : touched) owner[f] = -1;
    }
    // ordering: two coupled patches must run in ascending vertex order; the
    // facet's two patches are stored (lower vertex, higher vertex)
    bool order = true;
    for (int f = 0; f < P.nb; ++f) {
      const int a = P.facet_patches[size_t(f) * 2], b = P.facet_patches[size_t(f) * 2 + 1];
      if (a >= 0 && b >= 0 && !(wave_of[a] < wave_of[b])) order = false;
    }
    int64_t vals[7] = {P.n(), P.npatch, P.nwaves(), cover, indep, order, P.max_patch_f};
    int w = 0;
    for (; w < 7 && w < out_len; ++w) out[w] = vals[w];
    for (int i = 0; i < P.nwaves() && w < out_len; ++i, ++w) out[w] = P.wave_ptr[i + 1] - P.wave_ptr[i];
    for (int i = 0; i < P.nwaves() && w < out_len; ++i, ++w) out[w] = P.asap_sizes[i];
    return w;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1;
  }
}
int hpmg_step_mesh(int n, int levels, hpmg_mesh_desc* out) { return fill_desc(host::step_domain(n), levels, out); }

}  // extern "C"
