"""ctypes binding of the CPU oracle (oracle/_build/liborc.so).

TEST INFRASTRUCTURE ONLY: the oracle is the checker for parity tests and the
CPU baseline; the product (paper_2303_06762_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "_build", "liborc.so")

# enums shared with oracle/orc_capi.cpp
BC_NONE, BC_LID_TOP, BC_LID_ALL, BC_INLET, BC_LID_UNIT, BC_CONST, BC_ZERO, BC_LINEAR_FLOW = range(8)
LOAD_NONE, LOAD_ARRAY, LOAD_SMOOTH_UZAWA, LOAD_SIN_ADV, LOAD_EQUIV, LOAD_ASSEMBLY = range(6)
# manufactured Stokes load (nu, beta of the problem), manufactured NS load (nu),
# the linear flow's load 2u + (1, 1) (reference tests/test_postprocess.cpp)
LOAD_MMS_STOKES, LOAD_MMS_NS, LOAD_LINEAR_FLOW = 6, 7, 8
EXACT_MMS, EXACT_LINEAR = 1, 2
WIND_NONE, WIND_ROT, WIND_CURL = range(3)
CYCLE_V, CYCLE_W, CYCLE_VARV = range(3)
SM_MULT, SM_ADD = range(2)


class Problem(C.Structure):
    _fields_ = [
        ("mesh_kind", C.c_int), ("base_n", C.c_int), ("levels", C.c_int), ("k", C.c_int),
        ("nu", C.c_double), ("beta", C.c_double), ("mass_coef", C.c_double), ("inv_eps", C.c_double),
        ("bc_kind", C.c_int), ("load_kind", C.c_int), ("load", C.POINTER(C.c_double)),
        ("wind_kind", C.c_int), ("cycle", C.c_int), ("smoother", C.c_int), ("smooth_steps", C.c_int),
        ("jacobi_damping", C.c_double), ("newton", C.c_int), ("mass_field", C.c_int),
    ]


class NSOpts(C.Structure):
    _fields_ = [("picard_tol", C.c_double), ("newton_rel_tol", C.c_double), ("newton_abs_tol", C.c_double),
                ("max_picard", C.c_int), ("max_newton", C.c_int), ("pseudo_time_inv", C.c_double),
                ("outer_iterations", C.c_int), ("rel_tol", C.c_double), ("abs_tol", C.c_double),
                ("max_iterations", C.c_int)]


class NSReport(C.Structure):
    _fields_ = [("picard_iterations", C.c_int), ("newton_iterations", C.c_int), ("n_picard_inner", C.c_int),
                ("n_newton_inner", C.c_int), ("picard_inner", C.c_int * 512), ("newton_inner", C.c_int * 256),
                ("picard_diffs", C.c_double * 128), ("newton_diffs", C.c_double * 64),
                ("converged", C.c_int), ("not_applicable", C.c_int), ("final_divergence", C.c_double),
                ("seconds", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("not_applicable", C.c_int),
                ("residual", C.c_double)]


REF_LIB_PATH = os.path.join(ORACLE_DIR, "_ref", "libref.so")

_lib = None
_ref_libs = {}


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class _Lenient:
    """Lets the binder set argtypes on symbols a library may not export (the
    reference driver exports a subset of the restatement's surface)."""

    def __init__(self, L):
        self.__dict__["_L"] = L

    def __getattr__(self, name):
        L = self.__dict__["_L"]
        return getattr(L, name) if hasattr(L, name) else type("_Missing", (), {})()


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def ref_available():
    """True when the reference itself (oracle/_ref/libref.so: the unmodified
    reference headers over the Eigen-API shim) is built; it only exists where
    /root/reference is present (the build container)."""
    return os.path.exists(REF_LIB_PATH)


def ref_lib(variant=""):
    """The reference build (variant "": oracle/_ref/libref.so; "fma": the same
    sources compiled with FMA contraction, oracle/_ref/libref_fma.so, used to
    measure the reference's own round-off floor)."""
    if variant not in _ref_libs:
        path = REF_LIB_PATH if not variant else os.path.join(ORACLE_DIR, "_ref", f"libref_{variant}.so")
        _ref_libs[variant] = _bind(C.CDLL(path))
        L = _ref_libs[variant]
        L.orc_mg_create_traced.restype = C.c_void_p
        L.orc_mg_create_traced.argtypes = [C.POINTER(Problem)]
        L.orc_mg_trace.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_double)]
        L.orc_tts.argtypes = [C.POINTER(Problem), C.c_int, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_double)]
    return _ref_libs[variant]


def _bind(L0):
    if True:
        L = _Lenient(L0)
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        lp = C.POINTER(C.c_longlong)
        L.orc_mg_create.restype = P
        L.orc_mg_create.argtypes = [C.POINTER(Problem)]
        L.orc_last_error.restype = C.c_char_p
        for name in ["orc_mg_n", "orc_mg_n_full", "orc_mg_nnz", "orc_mg_rows", "orc_mg_P_nnz", "orc_mg_patches"]:
            getattr(L, name).restype = C.c_longlong
        L.orc_mg_setup_seconds.restype = C.c_double
        L.orc_mg_time_apply.restype = C.c_double
        L.orc_check_picard_newton.restype = C.c_double
        L.orc_check_upwind_lifting.restype = C.c_double
        L.orc_seeded_load.argtypes = [C.c_int, C.c_uint, C.c_double, C.c_double, dp]
        L.orc_mg_krylov.argtypes = [P, C.c_int, dp, dp, C.c_double, C.c_double, C.c_int, C.POINTER(Stats)]
        L.orc_mg_uzawa.argtypes = [P, C.c_int, C.c_double, C.c_double, C.c_int, dp, dp,
                                   C.POINTER(C.c_int), dp, C.POINTER(C.c_int), dp, dp]
        L.orc_mg_rt_l2_norm.restype = C.c_double
        L.orc_mg_rt_l2_norm.argtypes = [P, dp, dp]
        L.orc_ns_solve.argtypes = [C.POINTER(Problem), C.POINTER(NSOpts), dp, dp, dp, C.POINTER(NSReport)]
        L.orc_mg_smooth.argtypes = [P, C.c_int, C.c_int, dp, dp, C.c_int, C.c_double]
        L.orc_check_cr_equivalence.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_double, C.c_int, dp]
        for name in ["orc_mg_destroy", "orc_mg_n", "orc_mg_n_full", "orc_mg_num_levels", "orc_mg_ne",
                     "orc_mg_setup_seconds"]:
            getattr(L, name).argtypes = [P]
        L.orc_mg_time_apply.argtypes = [P, C.c_int]
        L.orc_mg_set_restart.argtypes = [P, C.c_int]
        # every handle-taking entry point gets an explicit void* first argument
        # (an untyped Python int would be truncated to 32 bits)
        L.orc_mg_rows.argtypes = [P, C.c_int]
        L.orc_mg_nnz.argtypes = [P, C.c_int]
        L.orc_mg_P_nnz.argtypes = [P, C.c_int]
        L.orc_mg_csr.argtypes = [P, C.c_int, lp, lp, dp]
        L.orc_mg_P_csr.argtypes = [P, C.c_int, lp, lp, dp]
        L.orc_mg_rhs.argtypes = [P, dp]
        L.orc_mg_free_to_full.argtypes = [P, lp]
        L.orc_mg_g_full.argtypes = [P, dp]
        L.orc_mg_apply.argtypes = [P, dp, dp]
        L.orc_mg_spmv.argtypes = [P, dp, dp]
        L.orc_mg_num_patches.argtypes = [P, C.c_int]
        L.orc_mg_patches.argtypes = [P, C.c_int, lp, lp]
        L.orc_mg_recover.argtypes = [P, dp, dp, dp, dp]
        L.orc_mg_wind.argtypes = [P, dp, dp]
        L.orc_mg_postprocess.argtypes = [P, dp, dp, dp, dp]
        L.orc_mg_errors.argtypes = [P, dp, dp, dp, dp, C.c_int, dp]
        L.orc_mms_point.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, dp]
        L.orc_mg_centroids.argtypes = [P, dp]
        L.orc_set_max_order.argtypes = [C.c_int]
    return L0


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _lp(a):
    return a.ctypes.data_as(C.POINTER(C.c_longlong))


def random_vec(n, seed):
    """std::mt19937 + uniform(-1,1), the reference tests' random_vec."""
    out = np.empty(int(n))
    lib().orc_random_vec(C.c_longlong(int(n)), C.c_uint(seed), _dp(out))
    return out


def seeded_load(n, seed, lo=-1.0, hi=1.0):
    out = np.empty(4 * n * n)
    lib().orc_seeded_load(n, seed, lo, hi, _dp(out))
    return out


class OracleMG:
    """Oracle MGPreconditioner + solvers for one problem (reference inc/multigrid.hpp)."""

    def __init__(self, *, mesh_kind=0, base_n=2, levels=2, k=0, nu=1.0, beta=0.0, mass_coef=0.0,
                 inv_eps=1e6, bc=BC_NONE, load_kind=LOAD_NONE, load=None, wind=WIND_NONE,
                 cycle=CYCLE_W, smoother=SM_MULT, smooth_steps=1, jacobi_damping=1.0 / 3.0, newton=False,
                 mass_field=False, reference=False, traced=False):
        L = (ref_lib("" if reference is True else reference)) if reference else lib()
        self.L = L
        self._load = None if load is None else np.ascontiguousarray(load, dtype=np.float64)
        p = Problem(mesh_kind, base_n, levels, k, nu, beta, mass_coef, inv_eps, bc, load_kind,
                    _dp(self._load) if self._load is not None else None, wind, cycle, smoother,
                    smooth_steps, jacobi_damping, int(newton), int(mass_field))
        self.h = (L.orc_mg_create_traced if traced else L.orc_mg_create)(C.byref(p))
        if not self.h:
            raise RuntimeError(L.orc_last_error().decode())
        self.n = L.orc_mg_n(self.h)
        self.n_full = L.orc_mg_n_full(self.h)
        self.ne = L.orc_mg_ne(self.h)
        self.k = k

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_mg_destroy(self.h)
            self.h = None

    @property
    def setup_seconds(self):
        return self.L.orc_mg_setup_seconds(self.h)

    def csr(self, level=-1):
        import scipy.sparse as sp
        L = self.L
        rows = L.orc_mg_rows(self.h, level)
        nnz = L.orc_mg_nnz(self.h, level)
        ptr = np.empty(rows + 1, np.int64)
        idx = np.empty(nnz, np.int64)
        val = np.empty(nnz)
        L.orc_mg_csr(self.h, level, _lp(ptr), _lp(idx), _dp(val))
        return sp.csr_matrix((val, idx, ptr), shape=(rows, rows))

    def prolongation(self, level):
        import scipy.sparse as sp
        L = self.L
        rows = L.orc_mg_rows(self.h, level)
        cols = L.orc_mg_rows(self.h, level - 1)
        nnz = L.orc_mg_P_nnz(self.h, level)
        ptr = np.empty(rows + 1, np.int64)
        idx = np.empty(nnz, np.int64)
        val = np.empty(nnz)
        L.orc_mg_P_csr(self.h, level, _lp(ptr), _lp(idx), _dp(val))
        return sp.csr_matrix((val, idx, ptr), shape=(rows, cols))

    def rhs(self):
        out = np.empty(self.n)
        self.L.orc_mg_rhs(self.h, _dp(out))
        return out

    def free_to_full(self):
        out = np.empty(self.n, np.int64)
        self.L.orc_mg_free_to_full(self.h, _lp(out))
        return out

    def g_full(self):
        out = np.empty(self.n_full)
        self.L.orc_mg_g_full(self.h, _dp(out))
        return out

    def apply(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.n)
        self.L.orc_mg_apply(self.h, _dp(b), _dp(x))
        return x

    def spmv(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        self.L.orc_mg_spmv(self.h, _dp(x), _dp(y))
        return y

    def smooth(self, level, which, x, b, sweeps=1, damping=1.0 / 3.0):
        x = np.array(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        self.L.orc_mg_smooth(self.h, level, which, _dp(x), _dp(b), sweeps, damping)
        return x

    def patches(self, level=-1):
        L = self.L
        n = L.orc_mg_num_patches(self.h, level)
        tot = L.orc_mg_patches(self.h, level, None, None)
        offs = np.empty(n + 1, np.int64)
        dofs = np.empty(tot, np.int64)
        L.orc_mg_patches(self.h, level, _lp(offs), _lp(dofs))
        return [dofs[offs[j]:offs[j + 1]] for j in range(n)]

    def krylov(self, b, x0=None, method=0, rel_tol=1e-8, abs_tol=1e-10, max_it=500):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n) if x0 is None else np.array(x0, dtype=np.float64)
        st = Stats()
        self.L.orc_mg_krylov(self.h, method, _dp(b), _dp(x), rel_tol, abs_tol, max_it, C.byref(st))
        return x, dict(iterations=st.iterations, converged=bool(st.converged),
                       not_applicable=bool(st.not_applicable), residual=st.residual)

    def uzawa(self, outer=2, rel_tol=1e-8, abs_tol=1e-10, max_it=500, initial_velocity=None):
        init = None if initial_velocity is None else np.ascontiguousarray(initial_velocity, dtype=np.float64)
        vel = np.empty(self.n_full)
        p = np.empty(self.ne)
        inner = (C.c_int * outer)()
        hist = np.zeros(outer)
        flags = (C.c_int * 2)()
        secs = np.zeros(1)
        done = self.L.orc_mg_uzawa(self.h, outer, rel_tol, abs_tol, max_it, _dp(vel), _dp(p), inner,
                                  _dp(hist), flags, _dp(secs), None if init is None else _dp(init))
        return dict(velocity=vel, pressure=p, inner_iterations=list(inner)[:done],
                    divergence_history=list(hist[:done]), converged=bool(flags[0]),
                    not_applicable=bool(flags[1]), seconds=float(secs[0]))

    def recover(self, velocity_full):
        k = self.k
        ns = (k + 1) * (k + 2) // 2
        v = np.ascontiguousarray(velocity_full, dtype=np.float64)
        interior = np.zeros((self.ne, max(k * (k + 1), 1)))
        p = np.zeros((self.ne, max(ns - 1, 1)))
        g = np.zeros((self.ne, 4 * ns))
        self.L.orc_mg_recover(self.h, _dp(v), _dp(interior), _dp(p), _dp(g))
        return interior[:, : k * (k + 1)], p[:, : ns - 1], g

    def set_restart(self, m):
        """GMRES(m) for the following krylov/uzawa calls (restatement only:
        the reference's GMRES is unrestarted)."""
        self.L.orc_mg_set_restart(self.h, int(m))

    def trace(self, cap=4096):
        """The MG residual trace of the last apply (reference contexts made
        with traced=True): (levels, entering flags, residual norms)."""
        lv = (C.c_int * cap)()
        en = (C.c_int * cap)()
        res = np.zeros(cap)
        n = min(self.L.orc_mg_trace(self.h, cap, lv, en, _dp(res)), cap)
        return list(lv)[:n], list(en)[:n], res[:n]

    def time_apply(self, reps):
        return self.L.orc_mg_time_apply(self.h, reps)

    def wind(self):
        """The interpolated advection state (compound full, interior [ne][k(k+1)])."""
        c = np.empty(self.n_full)
        i = np.zeros(max(self.ne * self.k * (self.k + 1), 1))
        self.L.orc_mg_wind(self.h, _dp(c), _dp(i))
        return c, i[: self.ne * self.k * (self.k + 1)]

    def rt_l2_norm(self, compound_full, interior):
        c = np.ascontiguousarray(compound_full, dtype=np.float64)
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        if i.size == 0:
            i = np.zeros(1)
        return self.L.orc_mg_rt_l2_norm(self.h, _dp(c), _dp(i))


    def postprocess(self, compound_full, interior, grad):
        """postprocess_velocity: [ne][2 ns_hi] (x modes, then y modes)."""
        nh = (self.k + 2) * (self.k + 3) // 2
        out = np.zeros((self.ne, 2 * nh))
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        self.L.orc_mg_postprocess(self.h, _dp(np.ascontiguousarray(compound_full, dtype=np.float64)),
                                 _dp(i if i.size else np.zeros(1)), _dp(np.ascontiguousarray(grad, dtype=np.float64)),
                                 _dp(out))
        return out

    def centroids(self):
        out = np.zeros((self.ne, 2))
        self.L.orc_mg_centroids(self.h, _dp(out))
        return out

    def errors(self, compound_full, interior, grad, post, kind):
        """measure_errors against exact flow `kind`: dict e_u, e_L, e_ustar, div_u."""
        out = np.zeros(4)
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        self.L.orc_mg_errors(self.h, _dp(np.ascontiguousarray(compound_full, dtype=np.float64)),
                            _dp(i if i.size else np.zeros(1)), _dp(np.ascontiguousarray(grad, dtype=np.float64)),
                            _dp(np.ascontiguousarray(post, dtype=np.float64)), kind, _dp(out))
        return dict(zip(("e_u", "e_L", "e_ustar", "div_u"), out))


def set_max_order(k):
    """Highest accepted order (3 = the reference's cap); returns the previous one."""
    return lib().orc_set_max_order(k)


def mms_point(x, y, nu, beta):
    """Manufactured flow at (x, y): u(2), grad u(4, row-major), lap u(2), p,
    grad p(2), stokes_load(nu, beta)(2), ns_load(nu)(2)."""
    out = np.zeros(15)
    lib().orc_mms_point(x, y, nu, beta, _dp(out))
    return out


def ns_solve(*, mesh_kind=0, base_n=2, levels=2, k=0, nu=1.0, inv_eps=1e3, bc=BC_LID_UNIT, load_kind=LOAD_NONE,
             load=None, cycle=CYCLE_V, smoother=SM_MULT, smooth_steps=1, picard_tol=1e-4, newton_rel_tol=1e-8,
             newton_abs_tol=1e-10, max_picard=60, max_newton=25, pseudo_time_inv=0.0, outer=2, rel_tol=1e-8,
             abs_tol=1e-10, max_it=500, reference=False):
    """Oracle navier_stokes_solve (reference inc/ns.hpp:69-149); reference=True
    runs the reference's own driver (oracle/_ref/libref.so)."""
    L = ref_lib() if reference else lib()
    ld = None if load is None else np.ascontiguousarray(load, dtype=np.float64)
    p = Problem(mesh_kind, base_n, levels, k, nu, 0.0, 0.0, inv_eps, bc, load_kind,
                _dp(ld) if ld is not None else None, WIND_NONE, cycle, smoother, smooth_steps, 1.0 / 3.0, 0, 0)
    o = NSOpts(picard_tol, newton_rel_tol, newton_abs_tol, max_picard, max_newton, pseudo_time_inv, outer, rel_tol,
               abs_tol, max_it)
    # sizes from a throwaway problem of the same mesh and order
    probe = OracleMG(mesh_kind=mesh_kind, base_n=base_n, levels=levels, k=k, nu=nu, inv_eps=inv_eps, bc=bc,
                     reference=reference)
    vel = np.zeros(probe.n_full)
    interior = np.zeros(max(probe.ne * k * (k + 1), 1))
    pres = np.zeros(probe.ne)
    rep = NSReport()
    if L.orc_ns_solve(C.byref(p), C.byref(o), _dp(vel), _dp(interior), _dp(pres), C.byref(rep)):
        raise RuntimeError(L.orc_last_error().decode())
    return dict(velocity=vel, interior=interior[: probe.ne * k * (k + 1)], pressure=pres,
                picard_iterations=rep.picard_iterations, newton_iterations=rep.newton_iterations,
                picard_inner=list(rep.picard_inner[: rep.n_picard_inner]),
                newton_inner=list(rep.newton_inner[: rep.n_newton_inner]),
                picard_diffs=list(rep.picard_diffs[: rep.picard_iterations]),
                newton_diffs=list(rep.newton_diffs[: rep.newton_iterations]),
                converged=bool(rep.converged), not_applicable=bool(rep.not_applicable),
                final_divergence=rep.final_divergence, seconds=rep.seconds)


def check(name, *args, n_out):
    out = np.zeros(n_out)
    getattr(lib(), name)(*args, _dp(out))
    return out
