/* hpmg C ABI: B200-native hp-multigrid preconditioned Krylov solve for the
 * statically condensed H(div)-HDG Stokes/Oseen operator.
 *
 * Drop-in boundary for the reference (hdivmg) operator API. Each entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/hdivmg):
 *
 *   hpmg_create / hpmg_destroy  <- MGPreconditioner::MGPreconditioner(hier, k, bc,
 *                                  fine_opt, inv_eps, mg)          multigrid.hpp:45-114
 *   hpmg_apply                  <- MGPreconditioner::apply / as_operator
 *                                                                  multigrid.hpp:117-131
 *   hpmg_apply_batch            <- apply() over independent right-hand sides, copies overlapped
 *   hpmg_spmv                   <- the LinearOperator [&B](v){ return B.matrix()*v; }
 *                                                                  uzawa.hpp:42, krylov.hpp:10
 *   hpmg_matrix_csr, hpmg_rhs,  <- matrix(), rhs(), constraints(), symmetric(), penalty()
 *   hpmg_free_to_full, ...                                          multigrid.hpp:133-146
 *   hpmg_write_matrix_market    <- write_matrix_market(os, B.matrix()) io.hpp:74-81
 *   hpmg_pcg / hpmg_gmres       <- pcg(A, M, b, x, opt) / gmres(...)  krylov.hpp:30-144
 *   hpmg_uzawa                  <- uzawa_solve(B, opt)             uzawa.hpp:51-91
 *   hpmg_recover                <- recover_locals(mesh, V, opt, u) assembly.hpp:513-549
 *   hpmg_smooth                 <- PatchSmoother::forward/backward/jacobi
 *                                                                  smoother.hpp:53-80
 *   hpmg_postprocess            <- postprocess_velocity(mesh, V, nu, u, grad) postprocess.hpp:29-80
 *   hpmg_measure_errors         <- measure_errors(..., exact_velocity, exact_gradient)
 *                                                                  postprocess.hpp:142-188
 *
 * Conventions (identical to the reference):
 *  - Vectors crossing the boundary are in the reference FREE order
 *    (Constraints::free_to_full, fespace.hpp:508-513): all free normal-flux
 *    coefficients (facet-major, mode-minor) then all free tangential ones.
 *    Internally the device uses a facet-major block layout; the permutation
 *    is applied inside the call.
 *  - Pointers are host memory unless HPMG_DEVICE_PTRS is passed in `flags`,
 *    in which case they are device pointers (still reference order) and the
 *    call is stream-ordered on hpmg_stream(ctx): inputs must be ready on that
 *    stream, outputs are complete once it is synchronised (or waited on).
 *  - Errors: setup errors return a nonzero status and hpmg_last_error()
 *    describes them (the C++ adapter rethrows them as the reference's
 *    exception types); solver breakdown / indefiniteness is reported in-band
 *    (hpmg_solve_stats.not_applicable), never as an error.
 *  - One context is bound to one CUDA stream and is not thread-safe.
 *  - No CPU fallback: without a usable CUDA device every call fails with
 *    HPMG_ERR_CUDA.
 */
#ifndef HPMG_CAPI_H
#define HPMG_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpmg_ctx hpmg_ctx;

enum { HPMG_OK = 0, HPMG_ERR_ARG = 1, HPMG_ERR_CUDA = 2, HPMG_ERR_SETUP = 3, HPMG_ERR_LOGIC = 4 };
enum { HPMG_CYCLE_V = 0, HPMG_CYCLE_W = 1, HPMG_CYCLE_VARIABLE_V = 2 };        /* CycleKind */
enum { HPMG_SMOOTH_MULTIPLICATIVE = 0, HPMG_SMOOTH_ADDITIVE = 1 };            /* SmootherKind */
enum { HPMG_TAG_INTERIOR = 0, HPMG_TAG_DIRICHLET = 1, HPMG_TAG_OUTFLOW = 2 };  /* bc:: tags */
enum { HPMG_DEVICE_PTRS = 1 };

/* Point callback: out[0..1] = field(x, y) (VelocityBC::g, AssemblyOptions::load). */
typedef void (*hpmg_field_fn)(double x, double y, double* out, void* user);

/* Base mesh of the hierarchy (the reference Mesh before MeshHierarchy::build).
 * Elements are counter-clockwise vertex triples; facets are discovered from
 * them exactly as Mesh::finalize does; boundary facets default to Dirichlet
 * and `tag_overrides` (a, b, tag) triples retag facets (e.g. outflow). */
typedef struct {
  int n_vertices;
  const double* xy;        /* 2 * n_vertices */
  int n_elements;
  const int* elements;     /* 3 * n_elements */
  int n_tag_overrides;
  const int* tag_overrides; /* 3 * n_tag_overrides */
  int levels;              /* MeshHierarchy::build(base, levels) */
} hpmg_mesh_desc;

/* AssemblyOptions + inv_eps + MGOptions (assembly.hpp:69-77, multigrid.hpp:24-34). */
typedef struct {
  int k;                   /* order 0..6 (the reference accepts 0..3, fespace.hpp:115; 4..6 are
                              this library's extension, parity unpinned) */
  double nu, beta, mass_coef, inv_eps;
  int cycle, smoother, smooth_steps;
  double jacobi_damping;
  int sweep_variant;       /* multiplicative sweeps (one launch per independent wave, identical
                              results to the reference's sequential order):
                              HPMG_SWEEP_RECORDS (0, default): every level streams patch records,
                              x_p = S_p (b_p - A_pe x_e) without reading A_pp;
                              HPMG_SWEEP_DIRECT_NONSYM (1): nonsymmetric (advected) levels use the
                              direct-gather correction x_p += S_p (b - A x)_p instead, whose error
                              scales with the residual rather than with x_p (closer iteration counts
                              in long unrestarted GMRES runs; ~2.3x slower V-cycle at config 5) */
} hpmg_options;
enum { HPMG_SWEEP_RECORDS = 0, HPMG_SWEEP_DIRECT_NONSYM = 1 };

/* Problem data: boundary values, load and (Oseen) advection state. */
typedef struct {
  hpmg_field_fn bc;           /* NULL: homogeneous Dirichlet data */
  void* bc_user;
  hpmg_field_fn load;         /* point load, evaluated on the host at the quadrature points */
  void* load_user;
  const double* load_per_element; /* alternative: constant force per finest element (2*ne) */
  const double* wind_compound;    /* advection HDGVelocity on the finest mesh at order k: */
  const double* wind_interior;    /*   compound (n_full) and interior (ne*k(k+1)); NULL = Stokes */
  int newton;                     /* Newton linearisation about the wind (AssemblyOptions::newton) */
  const double* structured_load;  /* alternative: seeded structured force (hpmg_seeded_load layout) */
  int structured_n;               /*   on an n x n unit-square grid, mapped onto the finest elements */
  hpmg_field_fn wind;             /* alternative advection state: a wind field, interpolated into   */
  void* wind_user;                /*   the hybrid RT_k space as interpolate_hdg does (Oseen/Picard) */
  const double* mass_compound;    /* pseudo-time mass field (AssemblyOptions::mass_field): HDG     */
  const double* mass_interior;    /*   velocity at order k, load += mass_coef (m, v); NULL = none   */
} hpmg_problem;

/* Analytic fields usable as hpmg_field_fn (no host-language callback cost):
 * BASELINE config 5 wind w = curl of sin^2(pi x) sin^2(pi y), i.e.
 * (pi sin^2(pi x) sin(2 pi y), -pi sin(2 pi x) sin^2(pi y)); the rotation
 * (y - 1/2, 1/2 - x) of the reference tests; the unit lid (1, 0) on y = 1. */
void hpmg_field_config5_wind(double x, double y, double* out, void* user);
void hpmg_field_rotation(double x, double y, double* out, void* user);
void hpmg_field_lid_unit(double x, double y, double* out, void* user);

/* Point callback of a 2x2 tensor field, row-major: out = {d u0/dx, d u0/dy,
 * d u1/dx, d u1/dy} (measure_errors' exact_gradient). */
typedef void (*hpmg_tensor_fn)(double x, double y, double* out, void* user);
/* The manufactured flow of the reference convergence tests (manufactured.hpp:
 * 16-65): u = curl of -G(x)G(y), G(s) = s^2 (s-1)^2; p = x(1-x)(1-y) - 1/12.
 * Loads: stokes_load user = double[2] {nu, beta} (-nu lap u + beta u + grad p);
 * ns_load user = double* nu (-nu lap u + (grad u) u + grad p). The linear flow
 * u = (1 + 2y + 3x, 4 - 3y + 5x) with load 2u + (1, 1) (nu = 1/2, beta = 2,
 * p = x + y - 1) of the reference exactness test (test_postprocess.cpp:120-157).
 * Passing the library's own velocity/gradient pair to hpmg_measure_errors
 * evaluates it on the device. */
void hpmg_field_mms_velocity(double x, double y, double* out, void* user);
void hpmg_tensor_mms_gradient(double x, double y, double* out, void* user);
double hpmg_mms_pressure(double x, double y);
void hpmg_field_mms_stokes_load(double x, double y, double* out, void* user);
void hpmg_field_mms_ns_load(double x, double y, double* out, void* user);
void hpmg_field_linear_flow(double x, double y, double* out, void* user);
void hpmg_tensor_linear_flow_gradient(double x, double y, double* out, void* user);
void hpmg_field_linear_flow_load(double x, double y, double* out, void* user);

typedef struct {
  double rel_tol, abs_tol;    /* KrylovOptions (krylov.hpp:12-16): 1e-8, 1e-10 */
  int max_iterations;         /* 500 */
  int restart;                /* GMRes only: 0 = reference semantics (no cap); m = GMRes(m) */
} hpmg_krylov_opts;

typedef struct {
  int iterations, converged, not_applicable;
  double residual;
} hpmg_solve_stats;

typedef struct {
  int outer_iterations;       /* UzawaOptions (uzawa.hpp:9-21): 2 */
  hpmg_krylov_opts krylov;
  const double* initial_velocity; /* warm start, full compound (host); NULL = zero */
} hpmg_uzawa_opts;

typedef struct {
  int n_outer;
  int inner_iterations[64];
  double divergence_history[64];
  int converged, not_applicable;
  double final_divergence;
  double seconds;             /* device time of the whole outer loop */
} hpmg_uzawa_report;

/* ---- lifecycle ---- */
int hpmg_create(hpmg_ctx** out, const hpmg_mesh_desc* mesh, const hpmg_options* opt, const hpmg_problem* prob);
void hpmg_destroy(hpmg_ctx* ctx);
/* Re-linearise in place (the reference rebuilds MGPreconditioner per
 * Picard/Newton step, ns.hpp:84): new wind / Newton flag / mass field / load /
 * boundary data and nu, beta, mass_coef, inv_eps; the mesh hierarchy, plans,
 * patch structure, wave schedules and allocations are kept. Order, cycle,
 * smoother, sweep variant and the symmetric/advected class must not change. */
int hpmg_update(hpmg_ctx* ctx, const hpmg_options* opt, const hpmg_problem* prob);
const char* hpmg_last_error(void);
void hpmg_set_last_error(const char* msg); /* for drivers layered on this ABI (hpmg_ns_solve) */
const char* hpmg_ctx_error(const hpmg_ctx* ctx);

/* ---- sizes and host mirrors ---- */
int64_t hpmg_n(const hpmg_ctx* ctx);            /* free DOFs of the finest system */
int64_t hpmg_n_full(const hpmg_ctx* ctx);       /* compound DOFs */
int hpmg_ne(const hpmg_ctx* ctx);               /* finest elements */
int hpmg_num_levels(const hpmg_ctx* ctx);
int64_t hpmg_level_n(const hpmg_ctx* ctx, int level); /* free DOFs of level l (-1: finest system) */
int hpmg_level_patches(const hpmg_ctx* ctx, int level); /* vertex patches of level l (-1: finest system) */
int hpmg_symmetric(const hpmg_ctx* ctx);
double hpmg_penalty(const hpmg_ctx* ctx);
int hpmg_free_to_full(const hpmg_ctx* ctx, int64_t* out);
int hpmg_g_full(const hpmg_ctx* ctx, double* out);
int hpmg_rhs(hpmg_ctx* ctx, double* out, int flags);
/* CSR of the finest operator (level -1) or of lowest-order level l, reference
 * order: call with NULL arrays to get nnz through *nnz. */
int hpmg_matrix_csr(hpmg_ctx* ctx, int level, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val);
/* write_matrix_market (io.hpp:72-81) of the same operator: MatrixMarket
 * coordinate real general, 1-based, %.17g, column by column. */
int hpmg_write_matrix_market(hpmg_ctx* ctx, int level, const char* path);

/* ---- operators ---- */
int hpmg_spmv(hpmg_ctx* ctx, const double* x, double* y, int flags);
int hpmg_apply(hpmg_ctx* ctx, const double* r, double* z, int flags);
/* apply() with the reference's optional residual trace (MGOptions::trace /
 * MGTraceEntry, multigrid.hpp:18-33,120,126,168-183): for every level visit,
 * (level, entering = 1, |b|) on entry and (level, 0, |b - A x|) on exit, in
 * the reference's order; the order-k head is level L+1. Writes up to `cap`
 * entries and the total count. A debugging path: the cycle runs outside the
 * CUDA graph with a host read per norm. Same z as hpmg_apply. */
int hpmg_apply_trace(hpmg_ctx* ctx, const double* r, double* z, int flags, int cap, int* level, int* entering,
                     double* residual, int* count);
/* z[i] = apply(r[i]) for m independent host vectors (reference order; pinned
 * memory for overlap): copy-in of vector i+1 and copy-out of result i-1 run on
 * two copy streams while V-cycle i runs, so PCIe transfers hide behind the
 * device work. Results are identical to m hpmg_apply calls. */
int hpmg_apply_batch(hpmg_ctx* ctx, int m, const double* const* r, double* const* z);
/* which: 0 forward, 1 backward, 2 additive (jacobi) on level l (-1 = order-k head) */
int hpmg_smooth(hpmg_ctx* ctx, int level, int which, double* x, const double* b, int sweeps, int flags);

/* ---- solvers ---- */
int hpmg_pcg(hpmg_ctx* ctx, const double* b, double* x, const hpmg_krylov_opts* o, hpmg_solve_stats* st, int flags);
int hpmg_gmres(hpmg_ctx* ctx, const double* b, double* x, const hpmg_krylov_opts* o, hpmg_solve_stats* st, int flags);
/* velocity: full compound (n_full), pressure: element means (ne); host pointers */
int hpmg_uzawa(hpmg_ctx* ctx, const hpmg_uzawa_opts* o, double* velocity, double* pressure, hpmg_uzawa_report* rep);
/* rt_l2_norm (assembly.hpp:487-501) of the finest-space RT field given by its
 * full compound and interior ([ne][k(k+1)]) coefficients; host pointers */
double hpmg_rt_l2_norm(hpmg_ctx* ctx, const double* compound_full, const double* interior);
/* interpolate_hdg (assembly.hpp:40-62) of a field into the finest space at
 * order k in this library's interior basis: compound (n_full), interior (ne*k(k+1)) */
int hpmg_interpolate_hdg(hpmg_ctx* ctx, hpmg_field_fn field, void* user, double* compound_full, double* interior);

/* ---- stationary Navier-Stokes driver (ns.hpp:10-149) ---- */
typedef struct {
  double picard_tol;          /* 1e-4: Picard ends when ||u_n - u_{n-1}||_L2 < picard_tol */
  double newton_rel_tol;      /* 1e-8 */
  double newton_abs_tol;      /* 1e-10: Newton ends when the update < max(rel |u|, abs) */
  int max_picard;             /* 60 */
  int max_newton;             /* 25 */
  double pseudo_time_inv;     /* 0: backward-Euler pseudo time step 1/pseudo_time_inv in Picard */
  hpmg_uzawa_opts uzawa;      /* every linearised step (initial_velocity is set by the driver) */
} hpmg_ns_opts;

typedef struct {
  int picard_iterations, newton_iterations;
  int n_picard_inner, n_newton_inner;
  int picard_inner[512];      /* Krylov counts of every Picard Uzawa step */
  int newton_inner[256];
  double picard_diffs[128];   /* consecutive velocity difference norms */
  double newton_diffs[64];
  int converged, not_applicable;
  double final_divergence;
  double seconds;             /* wall time of the whole driver */
  double setup_seconds;       /* of which: preconditioner setups (one per linearised step) */
} hpmg_ns_report;

/* Stokes initial guess, Picard steps about the previous velocity, then
 * total-update Newton steps; each step rebuilds the hp-MG hierarchy around the
 * current velocity and warm-starts the AL-Uzawa solve from it. `opt` supplies
 * k, nu, inv_eps and the MG options (beta and mass_coef are ignored as in the
 * reference driver); `prob` supplies bc and load (its wind fields are ignored).
 * Outputs: final velocity (full compound n_full), interior (ne*k(k+1), this
 * library's interior basis), pressure (ne) and, if non-NULL, the recovered
 * locals of the final state (LocalSolution: p_ortho ne*(ns-1), grad ne*4ns,
 * ns = (k+1)(k+2)/2); host pointers. */
int hpmg_ns_solve(const hpmg_mesh_desc* mesh, const hpmg_options* opt, const hpmg_problem* prob,
                  const hpmg_ns_opts* ns, double* velocity, double* interior, double* pressure,
                  hpmg_ns_report* rep, double* p_ortho, double* grad);
/* recover_locals on the finest system: interior (ne*k(k+1)), p_ortho (ne*(ns-1)),
 * grad (ne*4*ns, element-major); interior coefficients refer to this library's
 * interior RT basis (same span as the reference's). */
int hpmg_recover(hpmg_ctx* ctx, const double* velocity_full, double* interior, double* p_ortho, double* grad);

/* ---- post-processing (postprocess.hpp:16-188) ---- */
/* postprocess_velocity: u* in [P^{k+1}]^2 per element from a velocity (full
 * compound + this library's interior coefficients) and its gradient variable
 * (grad as hpmg_recover writes it); post [ne][2 ns_hi] (x modes then y modes of
 * the orthonormal order-(k+1) basis, ns_hi = (k+2)(k+3)/2; the reference's
 * PostprocessedVelocity::coeffs column e). Host pointers. */
int hpmg_postprocess(hpmg_ctx* ctx, const double* velocity_full, const double* interior, const double* grad,
                     double* post);
/* measure_errors: out[4] = (e_u, e_L, e_ustar, div_u), the L2 errors of the
 * velocity, of the gradient variable against -nu grad u, of u*, and the L2
 * norm of div u_h, at the degree-16 rule. Host pointers. */
int hpmg_measure_errors(hpmg_ctx* ctx, const double* velocity_full, const double* interior, const double* grad,
                        const double* post, hpmg_field_fn u_exact, void* u_user, hpmg_tensor_fn grad_exact,
                        void* g_user, double* out);

/* ---- measurement hooks (bench.py) ---- */
void* hpmg_stream(hpmg_ctx* ctx);               /* cudaStream_t the context launches on */
/* Algorithmic bytes of one apply() / one spmv() in the reference storage
 * accounting; `parts` (optional, 8 doubles) splits the
 * V-cycle: head sweeps, head residual, level sweeps, level residuals, transfers, coarse;
 * parts[6] / parts[7] = head / level sweep bytes as this implementation streams
 * them (patch records + vector rows, not part of the returned total). */
double hpmg_vcycle_bytes(const hpmg_ctx* ctx, double* parts);
double hpmg_spmv_bytes(const hpmg_ctx* ctx);
/* Device-resident timing of `reps` applies (graph-launched) on device buffers
 * already in the internal layout; returns ms per apply. phase_ms (optional,
 * 8 doubles) receives per-phase averages from an event-instrumented pass. */
double hpmg_time_apply(hpmg_ctx* ctx, int reps, double* phase_ms);
/* Kernels one hpmg_apply launches (its graph: reference-order input -> blocks
 * with x = 0, the cycle, blocks -> reference order) once hpmg_apply has run;
 * before that, the kernels of the cycle graph alone. */
int hpmg_kernel_launches_per_apply(const hpmg_ctx* ctx);
/* Device-resident timing of `reps` finest-operator applies (k_spmv, stream-ordered,
 * no graph); returns ms per spmv. bytes (optional, 2 doubles): [0] bytes one
 * spmv streams as stored (ELL-BSR values + columns, x, y), [1] the SURVEY 8(d)
 * reference CSR accounting. */
double hpmg_time_spmv(hpmg_ctx* ctx, int reps, double* bytes);
/* Per-level split of one V-cycle (event-instrumented, no graph): out[0] coarse
 * solve, out[2l] / out[2l+1] pre / post part of level l, out[2L+2..2L+4] head
 * pre-sweep, head residual, head post-sweep (ms). Returns the entry count. */
int hpmg_profile_levels(hpmg_ctx* ctx, int reps, double* out);
/* Development probe of the device-loop cost: ms per iteration of a graph while
 * loop whose body is (mode 0) a countdown kernel only, (1) the V-cycle +
 * countdown, (2) an if-node holding the V-cycle, then the countdown (the
 * nesting of round 2's first PCG loop), (3) the V-cycle launched as a
 * child-graph node + countdown; 32 + bits: PCG-shaped body (1 operator apply
 * with the folded direction update, 2 update, 4 if-node, 8 r.z, 16 direction). */
double hpmg_debug_loop_probe(hpmg_ctx* ctx, int mode, int iters);
/* Development hook: clock64 timeline of the one-CTA small-level sweep. */
void hpmg_debug_small_trace(int arm, long long* out);
/* development: (kernel id, step, globaltimer) at the start of the GMRES loop's
 * Gram-Schmidt / tail / new-vector kernels; out[0] = count, then triples */
void hpmg_debug_gm_trace(int arm, long long* out);
/* development: per-CTA globaltimer stamps of the last wave-sweep launches (HPMG_DBG=4) */
void hpmg_debug_sweep_trace(long long* out);
double hpmg_setup_seconds(const hpmg_ctx* ctx, double* parts);

/* Seeded per-triangle force of the BASELINE configs: std::mt19937(seed) and
 * uniform_real_distribution(lo, hi) drawn in structured (j, i, lower/upper,
 * (fx, fy)) order for an n x n unit-square mesh; map_structured_load turns it
 * into per-element values for the finest mesh of a hierarchy. */
void hpmg_seeded_load(int n, unsigned seed, double lo, double hi, double* out);
int hpmg_structured_to_elements(const hpmg_ctx* ctx, int n, const double* structured, double* per_element);

/* Host-only (no GPU needed): builds the hierarchy and the level-`level` plan
 * (-1: order-k head on the finest mesh) and checks the wave schedule.
 * out[0] free DOFs, out[1] patches, out[2] waves, out[3] 1 if every free DOF
 * lies in exactly two patches (smoother.hpp:13-28), out[4] 1 if no two
 * patches of a wave share a facet or an operator coupling, out[5] 1 if the
 * waves respect every ascending-order dependency, out[6] max patch facets,
 * out[7..7+waves) wave sizes of the device schedule (balanced levelling),
 * out[7+waves..7+2*waves) the as-soon-as-possible wave sizes
 * (up to out_len). Returns entries written. */
int hpmg_plan_check(const hpmg_mesh_desc* mesh, int k, int level, int64_t* out, int out_len);

/* Base meshes of the reference (mesh.hpp:220-279): fills a descriptor whose
 * arrays stay valid until the next call from the same thread. */
int hpmg_unit_square_mesh(int n, int levels, hpmg_mesh_desc* out);
int hpmg_step_mesh(int n, int levels, hpmg_mesh_desc* out);

#ifdef __cplusplus
}
#endif
#endif
