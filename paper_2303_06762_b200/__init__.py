"""hpmg: B200-native hp-multigrid preconditioned Krylov solver (Python mirror).

Mirrors the reference hdivmg operator interface (proj/include/hdivmg):
``MGPreconditioner`` (multigrid.hpp:43-146), ``pcg`` / ``gmres`` (krylov.hpp:30-144)
and ``uzawa_solve`` (uzawa.hpp:51-91), on top of the C ABI in
include/hpmg/capi.h implemented by the in-tree ``lib/libhpmg.so`` (CUDA,
sm_100a). There is no CPU fallback: loading fails loudly without the library,
and every call fails without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPMG_LIB") or os.path.join(_PKG, "lib", "libhpmg.so")  # HPMG_LIB: A/B builds

CYCLE_V, CYCLE_W, CYCLE_VARIABLE_V = 0, 1, 2
SMOOTH_MULTIPLICATIVE, SMOOTH_ADDITIVE = 0, 1
DEVICE_PTRS = 1

FIELD_FN = C.CFUNCTYPE(None, C.c_double, C.c_double, C.POINTER(C.c_double), C.c_void_p)
TENSOR_FN = FIELD_FN  # same signature, 4 outputs (row-major gradient)


class _Mesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int), ("xy", C.POINTER(C.c_double)), ("n_elements", C.c_int),
                ("elements", C.POINTER(C.c_int)), ("n_tag_overrides", C.c_int),
                ("tag_overrides", C.POINTER(C.c_int)), ("levels", C.c_int)]


# multiplicative sweep variants (hpmg_options.sweep_variant): patch records on
# every level (default), or the direct-gather correction form on advected
# (nonsymmetric) levels
SWEEP_VARIANTS = {"records": 0, "direct_nonsym": 1}


class _Options(C.Structure):
    _fields_ = [("k", C.c_int), ("nu", C.c_double), ("beta", C.c_double), ("mass_coef", C.c_double),
                ("inv_eps", C.c_double), ("cycle", C.c_int), ("smoother", C.c_int), ("smooth_steps", C.c_int),
                ("jacobi_damping", C.c_double), ("sweep_variant", C.c_int)]


class _Problem(C.Structure):
    _fields_ = [("bc", FIELD_FN), ("bc_user", C.c_void_p), ("load", FIELD_FN), ("load_user", C.c_void_p),
                ("load_per_element", C.POINTER(C.c_double)), ("wind_compound", C.POINTER(C.c_double)),
                ("wind_interior", C.POINTER(C.c_double)), ("newton", C.c_int),
                ("structured_load", C.POINTER(C.c_double)), ("structured_n", C.c_int),
                ("wind", FIELD_FN), ("wind_user", C.c_void_p),
                ("mass_compound", C.POINTER(C.c_double)), ("mass_interior", C.POINTER(C.c_double))]


class _KOpts(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("abs_tol", C.c_double), ("max_iterations", C.c_int), ("restart", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("not_applicable", C.c_int),
                ("residual", C.c_double)]


class _UOpts(C.Structure):
    _fields_ = [("outer_iterations", C.c_int), ("krylov", _KOpts), ("initial_velocity", C.POINTER(C.c_double))]


class _NSOpts(C.Structure):
    _fields_ = [("picard_tol", C.c_double), ("newton_rel_tol", C.c_double), ("newton_abs_tol", C.c_double),
                ("max_picard", C.c_int), ("max_newton", C.c_int), ("pseudo_time_inv", C.c_double),
                ("uzawa", _UOpts)]


class _NSReport(C.Structure):
    _fields_ = [("picard_iterations", C.c_int), ("newton_iterations", C.c_int), ("n_picard_inner", C.c_int),
                ("n_newton_inner", C.c_int), ("picard_inner", C.c_int * 512), ("newton_inner", C.c_int * 256),
                ("picard_diffs", C.c_double * 128), ("newton_diffs", C.c_double * 64), ("converged", C.c_int),
                ("not_applicable", C.c_int), ("final_divergence", C.c_double), ("seconds", C.c_double),
                ("setup_seconds", C.c_double)]


class _UReport(C.Structure):
    _fields_ = [("n_outer", C.c_int), ("inner_iterations", C.c_int * 64), ("divergence_history", C.c_double * 64),
                ("converged", C.c_int), ("not_applicable", C.c_int), ("final_divergence", C.c_double),
                ("seconds", C.c_double)]


_lib = None


def lib():
    """Loads lib/libhpmg.so (builds it with nvcc first if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = C.CDLL(LIB_PATH)
    vp, dp, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)
    L.hpmg_create.argtypes = [C.POINTER(vp), C.POINTER(_Mesh), C.POINTER(_Options), C.POINTER(_Problem)]
    L.hpmg_destroy.argtypes = [vp]
    L.hpmg_last_error.restype = C.c_char_p
    L.hpmg_ctx_error.restype = C.c_char_p
    L.hpmg_ctx_error.argtypes = [vp]
    for name in ("hpmg_n", "hpmg_n_full"):
        getattr(L, name).restype = C.c_int64
        getattr(L, name).argtypes = [vp]
    for name in ("hpmg_ne", "hpmg_num_levels", "hpmg_symmetric", "hpmg_kernel_launches_per_apply"):
        getattr(L, name).argtypes = [vp]
    L.hpmg_level_n.restype = C.c_int64
    L.hpmg_level_n.argtypes = [vp, C.c_int]
    L.hpmg_level_patches.restype = C.c_int
    L.hpmg_level_patches.argtypes = [vp, C.c_int]
    L.hpmg_penalty.restype = C.c_double
    L.hpmg_penalty.argtypes = [vp]
    L.hpmg_free_to_full.argtypes = [vp, lp]
    L.hpmg_g_full.argtypes = [vp, dp]
    L.hpmg_rhs.argtypes = [vp, vp, C.c_int]
    L.hpmg_matrix_csr.argtypes = [vp, C.c_int, lp, lp, lp, dp]
    L.hpmg_spmv.argtypes = [vp, vp, vp, C.c_int]
    L.hpmg_apply.argtypes = [vp, vp, vp, C.c_int]
    L.hpmg_smooth.argtypes = [vp, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int]
    L.hpmg_pcg.argtypes = [vp, vp, vp, C.POINTER(_KOpts), C.POINTER(_Stats), C.c_int]
    L.hpmg_gmres.argtypes = [vp, vp, vp, C.POINTER(_KOpts), C.POINTER(_Stats), C.c_int]
    L.hpmg_uzawa.argtypes = [vp, C.POINTER(_UOpts), dp, dp, C.POINTER(_UReport)]
    L.hpmg_recover.argtypes = [vp, vp, vp, vp, vp]
    L.hpmg_postprocess.argtypes = [vp, dp, dp, dp, dp]
    L.hpmg_apply_batch.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]
    L.hpmg_apply_trace.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.hpmg_time_spmv.restype = C.c_double
    L.hpmg_time_spmv.argtypes = [vp, C.c_int, dp]
    L.hpmg_write_matrix_market.argtypes = [vp, C.c_int, C.c_char_p]
    L.hpmg_measure_errors.argtypes = [vp, dp, dp, dp, dp, FIELD_FN, vp, TENSOR_FN, vp, dp]
    L.hpmg_mms_pressure.restype = C.c_double
    L.hpmg_mms_pressure.argtypes = [C.c_double, C.c_double]
    L.hpmg_interpolate_hdg.argtypes = [vp, FIELD_FN, vp, dp, dp]
    L.hpmg_update.argtypes = [vp, C.POINTER(_Options), C.POINTER(_Problem)]
    L.hpmg_rt_l2_norm.restype = C.c_double
    L.hpmg_rt_l2_norm.argtypes = [vp, dp, dp]
    L.hpmg_ns_solve.argtypes = [C.POINTER(_Mesh), C.POINTER(_Options), C.POINTER(_Problem), C.POINTER(_NSOpts),
                                dp, dp, dp, C.POINTER(_NSReport), dp, dp]
    L.hpmg_stream.restype = vp
    L.hpmg_stream.argtypes = [vp]
    L.hpmg_vcycle_bytes.restype = C.c_double
    L.hpmg_vcycle_bytes.argtypes = [vp, dp]
    L.hpmg_spmv_bytes.restype = C.c_double
    L.hpmg_spmv_bytes.argtypes = [vp]
    L.hpmg_time_apply.restype = C.c_double
    L.hpmg_time_apply.argtypes = [vp, C.c_int, dp]
    L.hpmg_setup_seconds.restype = C.c_double
    L.hpmg_setup_seconds.argtypes = [vp, dp]
    L.hpmg_seeded_load.argtypes = [C.c_int, C.c_uint, C.c_double, C.c_double, dp]
    L.hpmg_structured_to_elements.argtypes = [vp, C.c_int, dp, dp]
    L.hpmg_unit_square_mesh.argtypes = [C.c_int, C.c_int, C.POINTER(_Mesh)]
    L.hpmg_step_mesh.argtypes = [C.c_int, C.c_int, C.POINTER(_Mesh)]
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


NAMED_FIELDS = {"config5_wind": "hpmg_field_config5_wind", "rotation": "hpmg_field_rotation",
                "lid_unit": "hpmg_field_lid_unit",
                # reference manufactured.hpp / test_postprocess.cpp flows; the two
                # parametrised loads take ("mms_stokes_load", (nu, beta)) / ("mms_ns_load", (nu,))
                "mms_velocity": "hpmg_field_mms_velocity", "mms_stokes_load": "hpmg_field_mms_stokes_load",
                "mms_ns_load": "hpmg_field_mms_ns_load", "linear_flow": "hpmg_field_linear_flow",
                "linear_flow_load": "hpmg_field_linear_flow_load"}
NAMED_TENSORS = {"mms_gradient": "hpmg_tensor_mms_gradient", "linear_flow_gradient": "hpmg_tensor_linear_flow_gradient"}
# exact flows of measure_errors by name: (velocity, gradient)
EXACT_FLOWS = {"mms": ("mms_velocity", "mms_gradient"), "linear_flow": ("linear_flow", "linear_flow_gradient")}


def _field_user(spec):
    """(callback, user pointer, keep-alive) of a field spec: None, a callable,
    a NAMED_FIELDS name, or (name, params) for the parametrised named loads."""
    if isinstance(spec, tuple) and len(spec) == 2 and isinstance(spec[0], str):
        params = np.ascontiguousarray(spec[1], dtype=np.float64)
        return _field(spec[0]), C.c_void_p(params.ctypes.data), params
    return _field(spec), None, None


def _tensor(fn):
    """Wraps a callable (x, y) -> 2x2 (d u_i / d x_j) or a NAMED_TENSORS name."""
    if isinstance(fn, str):
        return C.cast(getattr(lib(), NAMED_TENSORS[fn]), TENSOR_FN)

    def cb(x, y, out, _user):
        g = np.asarray(fn(x, y), dtype=np.float64).reshape(4)
        for i in range(4):
            out[i] = float(g[i])

    return TENSOR_FN(cb)


@dataclass
class ErrorNorms:
    """reference postprocess.hpp:84-89"""
    e_u: float = 0.0
    e_L: float = 0.0
    e_ustar: float = 0.0
    div_u: float = 0.0


def estimated_order(coarse, fine):
    """EOC between two error levels under uniform refinement (postprocess.hpp:190-194)."""
    return float(np.log2(coarse / fine))


def mms_pressure(x, y):
    return lib().hpmg_mms_pressure(x, y)


def _field(fn):
    """Wraps a python callable (x, y) -> (fx, fy) as a C point callback; a
    name from NAMED_FIELDS selects the library's own C implementation."""
    if fn is None:
        return FIELD_FN()
    if isinstance(fn, str):
        return C.cast(getattr(lib(), NAMED_FIELDS[fn]), FIELD_FN)

    def cb(x, y, out, _user):
        v = fn(x, y)
        out[0] = float(v[0])
        out[1] = float(v[1])

    return FIELD_FN(cb)


def seeded_load(n, seed, lo=-1.0, hi=1.0):
    """BASELINE per-triangle force: mt19937(seed), uniform(lo, hi), structured order."""
    out = np.empty(4 * n * n)
    lib().hpmg_seeded_load(n, seed, lo, hi, _dp(out))
    return out


@dataclass
class KrylovOptions:
    """reference krylov.hpp:12-16"""
    rel_tol: float = 1e-8
    abs_tol: float = 1e-10
    max_iterations: int = 500
    restart: int = 0

    def c(self):
        return _KOpts(self.rel_tol, self.abs_tol, self.max_iterations, self.restart)


@dataclass
class SolveStats:
    """reference krylov.hpp:18-26"""
    iterations: int = 0
    converged: bool = False
    not_applicable: bool = False
    residual: float = 0.0


@dataclass
class UzawaReport:
    """reference uzawa.hpp:23-33"""
    inner_iterations: list = field(default_factory=list)
    divergence_history: list = field(default_factory=list)
    converged: bool = False
    not_applicable: bool = False
    final_divergence: float = 0.0
    seconds: float = 0.0


@dataclass
class StokesSolution:
    velocity: np.ndarray
    pressure: np.ndarray
    report: UzawaReport


class HpmgError(RuntimeError):
    pass


class MGPreconditioner:
    """hp-multigrid preconditioner on the device (reference multigrid.hpp:43-146).

    mesh: "unit_square" or "step" with base size ``base_n`` refined to ``levels``
    mesh levels (MeshHierarchy::build). ``load`` is a point callback, or
    ``load_per_element`` a per-finest-element constant force, or
    ``structured_load=(n, array)`` the seeded BASELINE force on an n x n grid.
    """

    def __init__(self, *, mesh="unit_square", base_n=2, levels=2, k=0, nu=1.0, beta=0.0, mass_coef=0.0,
                 inv_eps=1e6, cycle=CYCLE_W, smoother=SMOOTH_MULTIPLICATIVE, smooth_steps=1,
                 jacobi_damping=1.0 / 3.0, bc=None, load=None, load_per_element=None, structured_load=None,
                 wind=None, newton=False, mass_field=None, sweep="records"):
        L = lib()
        md = _Mesh()
        rc = (L.hpmg_unit_square_mesh if mesh == "unit_square" else L.hpmg_step_mesh)(base_n, levels, C.byref(md))
        if rc:
            raise HpmgError(L.hpmg_last_error().decode())
        if sweep not in SWEEP_VARIANTS:
            raise ValueError(f"sweep must be one of {sorted(SWEEP_VARIANTS)}")
        self._optargs = dict(k=k, nu=nu, beta=beta, mass_coef=mass_coef, inv_eps=inv_eps, cycle=cycle,
                             smoother=smoother, smooth_steps=smooth_steps, jacobi_damping=jacobi_damping,
                             sweep_variant=SWEEP_VARIANTS[sweep])
        opt = _Options(**self._optargs)
        self._bc, self._bc_user, self._bc_keep = _field_user(bc)
        self._load, self._load_user, self._load_keep = _field_user(load)
        self._static = dict(load_per_element=load_per_element, structured_load=structured_load)
        prob = self._problem(wind, newton, mass_field)
        h = C.c_void_p()
        rc = L.hpmg_create(C.byref(h), C.byref(md), C.byref(opt), C.byref(prob))
        if rc:
            raise HpmgError(L.hpmg_last_error().decode())
        self.h = h
        self.k = k
        self.n = L.hpmg_n(h)
        self.n_full = L.hpmg_n_full(h)
        self.ne = L.hpmg_ne(h)

    def _problem(self, wind, newton, mass_field):
        """_Problem for the stored bc / load and the given linearisation state."""
        self._keep = []
        # Oseen / Newton advection state: a wind field (callable or NAMED_FIELDS
        # name) interpolated by the library, or an HDG velocity (compound, interior)
        hdg_wind = isinstance(wind, tuple)
        self._wind = _field(None if hdg_wind else wind)
        prob = _Problem(self._bc, self._bc_user, self._load, self._load_user, None, None, None, int(bool(newton)),
                        None, 0, self._wind,
                        None, None, None)
        if hdg_wind:
            wc, wi = (np.ascontiguousarray(a, dtype=np.float64) for a in wind)
            self._keep += [wc, wi]
            prob.wind_compound = _dp(wc)
            prob.wind_interior = _dp(wi) if wi.size else None
        if mass_field is not None:  # pseudo-time load mass_coef (m, v): HDG velocity (compound, interior)
            mc, mi = (np.ascontiguousarray(a, dtype=np.float64) for a in mass_field)
            self._keep += [mc, mi]
            prob.mass_compound = _dp(mc)
            prob.mass_interior = _dp(mi) if mi.size else None
        if self._static["load_per_element"] is not None:
            a = np.ascontiguousarray(self._static["load_per_element"], dtype=np.float64)
            self._keep.append(a)
            prob.load_per_element = _dp(a)
        if self._static["structured_load"] is not None:
            n, arr = self._static["structured_load"]
            a = np.ascontiguousarray(arr, dtype=np.float64)
            self._keep.append(a)
            prob.structured_load = _dp(a)
            prob.structured_n = int(n)
        return prob

    def update(self, *, wind=None, newton=False, mass_field=None, **opt_changes):
        """Re-linearise in place (hpmg_update): new wind / Newton flag / mass
        field and nu, beta, mass_coef, inv_eps, jacobi_damping; the hierarchy,
        plans and wave schedules are kept."""
        bad = set(opt_changes) - {"nu", "beta", "mass_coef", "inv_eps", "jacobi_damping"}
        if bad:
            raise ValueError(f"update cannot change {sorted(bad)}")
        self._optargs.update(opt_changes)
        opt = _Options(**self._optargs)
        prob = self._problem(wind, newton, mass_field)
        self._check(lib().hpmg_update(self.h, C.byref(opt), C.byref(prob)))
        return self

    def close(self):
        if getattr(self, "h", None):
            lib().hpmg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise HpmgError(lib().hpmg_ctx_error(self.h).decode())

    # -- reference accessors
    def symmetric(self):
        return bool(lib().hpmg_symmetric(self.h))

    def penalty(self):
        return lib().hpmg_penalty(self.h)

    def num_levels(self):
        return lib().hpmg_num_levels(self.h)

    def free_to_full(self):
        out = np.empty(self.n, np.int64)
        lib().hpmg_free_to_full(self.h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def g_full(self):
        out = np.empty(self.n_full)
        lib().hpmg_g_full(self.h, _dp(out))
        return out

    def rhs(self):
        out = np.empty(self.n)
        self._check(lib().hpmg_rhs(self.h, out.ctypes.data, 0))
        return out

    def level_n(self, level=-1):
        return int(lib().hpmg_level_n(self.h, level))

    def interpolate(self, field):
        """interpolate_hdg of a field (callable or NAMED_FIELDS name) into the
        finest space: (compound full, interior [ne, k(k+1)])."""
        f = _field(field)
        c = np.zeros(self.n_full)
        i = np.zeros(max(self.ne * self.k * (self.k + 1), 1))
        self._check(lib().hpmg_interpolate_hdg(self.h, f, None, _dp(c), _dp(i)))
        return c, i[: self.ne * self.k * (self.k + 1)].reshape(self.ne, self.k * (self.k + 1))

    def rt_l2_norm(self, compound_full, interior):
        """L2 norm of the finest-space RT field (reference assembly.hpp:487-501)."""
        c = np.ascontiguousarray(compound_full, dtype=np.float64)
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        v = lib().hpmg_rt_l2_norm(self.h, _dp(c), _dp(i) if i.size else None)
        if v < 0:
            raise HpmgError(lib().hpmg_ctx_error(self.h).decode())
        return v

    def level_patches(self, level=-1):
        return int(lib().hpmg_level_patches(self.h, level))

    def matrix(self, level=-1):
        """Host CSR mirror in the reference free order (multigrid.hpp:133)."""
        import scipy.sparse as sp
        L = lib()
        nnz = C.c_int64()
        self._check(L.hpmg_matrix_csr(self.h, level, C.byref(nnz), None, None, None))
        rows = self.level_n(level)
        ptr = np.empty(rows + 1, np.int64)
        idx = np.empty(nnz.value, np.int64)
        val = np.empty(nnz.value)
        self._check(L.hpmg_matrix_csr(self.h, level, C.byref(nnz), ptr.ctypes.data_as(C.POINTER(C.c_int64)),
                                      idx.ctypes.data_as(C.POINTER(C.c_int64)), _dp(val)))
        return sp.csr_matrix((val, idx, ptr), shape=(rows, rows))

    def write_matrix_market(self, path, level=-1):
        """MatrixMarket dump of matrix(level) by the native writer (io.hpp:74-81)."""
        self._check(lib().hpmg_write_matrix_market(self.h, level, os.fsencode(path)))

    # -- operators (host numpy in, host numpy out)
    def _vec(self, v, name="vector"):
        """A C-contiguous float64 host copy/view of length n (the native side
        reads exactly n doubles through the raw pointer)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.ndim != 1 or v.shape[0] != self.n:
            raise ValueError(f"{name} must have shape ({self.n},), got {v.shape}")
        return v

    def apply(self, b):
        b = self._vec(b, "b")
        z = np.empty(self.n)
        self._check(lib().hpmg_apply(self.h, b.ctypes.data, z.ctypes.data, 0))
        return z

    def apply_trace(self, b, cap=4096):
        """apply(b) with the MG residual trace (reference MGOptions::trace):
        returns (z, levels, entering flags, residual norms)."""
        b = self._vec(b, "b")
        z = np.empty(self.n)
        lv = (C.c_int * cap)()
        en = (C.c_int * cap)()
        res = np.zeros(cap)
        cnt = C.c_int(0)
        self._check(lib().hpmg_apply_trace(self.h, b.ctypes.data, z.ctypes.data, 0, cap, lv, en, _dp(res),
                                            C.byref(cnt)))
        n = min(cnt.value, cap)
        return z, list(lv)[:n], list(en)[:n], res[:n]

    def apply_batch(self, rs, zs=None):
        """apply() over independent host vectors with the PCIe copies of
        neighbouring vectors overlapped with the V-cycles (hpmg_apply_batch).
        rs / zs: sequences of float64 host arrays (pinned for overlap)."""
        rs = [self._vec(r, "rs[i]") for r in rs]
        if zs is None:
            zs = [np.empty(self.n) for _ in rs]
        if len(zs) != len(rs):
            raise ValueError(f"apply_batch: {len(rs)} inputs but {len(zs)} outputs")
        for z in zs:  # written in place by the native side: no silent copies
            if not (isinstance(z, np.ndarray) and z.dtype == np.float64 and z.ndim == 1 and z.shape[0] == self.n
                    and z.flags.c_contiguous and z.flags.writeable):
                raise ValueError(f"apply_batch: every output must be a writable C-contiguous float64 array of "
                                 f"length {self.n}")
        rp = (C.c_void_p * len(rs))(*[r.ctypes.data for r in rs])
        zp = (C.c_void_p * len(zs))(*[z.ctypes.data for z in zs])
        self._check(lib().hpmg_apply_batch(self.h, len(rs), rp, zp))
        return zs

    def spmv(self, x):
        x = self._vec(x, "x")
        y = np.empty(self.n)
        self._check(lib().hpmg_spmv(self.h, x.ctypes.data, y.ctypes.data, 0))
        return y

    def smooth(self, level, which, x, b, sweeps=1):
        x = np.array(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        nl = self.level_n(level)
        if x.shape != (nl,) or b.shape != (nl,):
            raise ValueError(f"smooth: x and b must have shape ({nl},)")
        self._check(lib().hpmg_smooth(self.h, level, which, x.ctypes.data, b.ctypes.data, sweeps, 0))
        return x

    def as_operator(self):
        return self.apply

    def recover(self, velocity_full):
        """recover_locals on the finest system (reference assembly.hpp:513-549):
        returns (interior [ne, k(k+1)], p_ortho [ne, ns-1], grad [ne, 4 ns])."""
        k = self.k
        ns = (k + 1) * (k + 2) // 2
        v = np.ascontiguousarray(velocity_full, dtype=np.float64)
        interior = np.zeros((self.ne, max(k * (k + 1), 1)))
        p = np.zeros((self.ne, max(ns - 1, 1)))
        g = np.zeros((self.ne, 4 * ns))
        self._check(lib().hpmg_recover(self.h, v.ctypes.data, interior.ctypes.data, p.ctypes.data, g.ctypes.data))
        return interior[:, : k * (k + 1)], p[:, : ns - 1], g

    def postprocess(self, velocity_full, interior, grad):
        """postprocess_velocity (reference postprocess.hpp:24-80): u* in
        [P^{k+1}]^2 per element, [ne, 2 ns_hi] (x modes then y modes)."""
        nh = (self.k + 2) * (self.k + 3) // 2
        out = np.zeros((self.ne, 2 * nh))
        v = np.ascontiguousarray(velocity_full, dtype=np.float64)
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        g = np.ascontiguousarray(grad, dtype=np.float64)
        self._check(lib().hpmg_postprocess(self.h, _dp(v), _dp(i) if i.size else None, _dp(g), _dp(out)))
        return out

    def measure_errors(self, velocity_full, interior, grad, post, exact="mms"):
        """measure_errors (reference postprocess.hpp:140-188) against an exact
        flow: a name from EXACT_FLOWS (evaluated on the device) or a pair of
        callables (velocity (x, y) -> 2, gradient (x, y) -> 2x2)."""
        if isinstance(exact, str):
            fu, fg = _field(EXACT_FLOWS[exact][0]), _tensor(EXACT_FLOWS[exact][1])
        else:
            fu, fg = _field(exact[0]), _tensor(exact[1])
        out = np.zeros(4)
        v = np.ascontiguousarray(velocity_full, dtype=np.float64)
        i = np.ascontiguousarray(interior, dtype=np.float64).ravel()
        g = np.ascontiguousarray(grad, dtype=np.float64)
        p = np.ascontiguousarray(post, dtype=np.float64)
        self._check(lib().hpmg_measure_errors(self.h, _dp(v), _dp(i) if i.size else None, _dp(g), _dp(p), fu, None,
                                              fg, None, _dp(out)))
        return ErrorNorms(*out)

    # -- measurement hooks
    def stream(self):
        return lib().hpmg_stream(self.h)

    def vcycle_bytes(self):
        parts = np.zeros(8)
        tot = lib().hpmg_vcycle_bytes(self.h, _dp(parts))
        return tot, parts

    def spmv_bytes(self):
        return lib().hpmg_spmv_bytes(self.h)

    def time_apply(self, reps, phases=False):
        ph = np.zeros(8)
        ms = lib().hpmg_time_apply(self.h, reps, _dp(ph) if phases else None)
        return ms, ph

    def time_spmv(self, reps):
        """(ms per finest-operator spmv, bytes as stored, reference-accounting bytes)."""
        b = np.zeros(2)
        ms = lib().hpmg_time_spmv(self.h, reps, _dp(b))
        return ms, b[0], b[1]

    def launches_per_apply(self):
        return lib().hpmg_kernel_launches_per_apply(self.h)

    def setup_seconds(self):
        parts = np.zeros(8)
        tot = lib().hpmg_setup_seconds(self.h, _dp(parts))
        return tot, parts


def pcg(B: MGPreconditioner, b, x=None, opt: KrylovOptions | None = None):
    """Device PCG with B.matrix() and B.apply (reference krylov.hpp:30-73)."""
    opt = opt or KrylovOptions()
    b = B._vec(b, "b")
    x = np.zeros(B.n) if x is None else B._vec(np.array(x, dtype=np.float64), "x")
    st = _Stats()
    B._check(lib().hpmg_pcg(B.h, b.ctypes.data, x.ctypes.data, C.byref(opt.c()), C.byref(st), 0))
    return x, SolveStats(st.iterations, bool(st.converged), bool(st.not_applicable), st.residual)


def gmres(B: MGPreconditioner, b, x=None, opt: KrylovOptions | None = None):
    """Device right-preconditioned MGS GMRES (reference krylov.hpp:79-144)."""
    opt = opt or KrylovOptions()
    b = B._vec(b, "b")
    x = np.zeros(B.n) if x is None else B._vec(np.array(x, dtype=np.float64), "x")
    st = _Stats()
    B._check(lib().hpmg_gmres(B.h, b.ctypes.data, x.ctypes.data, C.byref(opt.c()), C.byref(st), 0))
    return x, SolveStats(st.iterations, bool(st.converged), bool(st.not_applicable), st.residual)


def uzawa_solve(B: MGPreconditioner, outer_iterations=2, krylov: KrylovOptions | None = None,
                initial_velocity=None):
    """Augmented-Lagrangian Uzawa loop on the device (reference uzawa.hpp:51-91);
    `initial_velocity` (full compound) warm-starts the first Krylov solve."""
    krylov = krylov or KrylovOptions()
    vel = np.empty(B.n_full)
    p = np.empty(B.ne)
    rep = _UReport()
    init = None if initial_velocity is None else np.ascontiguousarray(initial_velocity, dtype=np.float64)
    if init is not None and init.shape != (B.n_full,):
        raise ValueError(f"initial_velocity must have shape ({B.n_full},)")
    o = _UOpts(outer_iterations, krylov.c(), None if init is None else _dp(init))
    B._check(lib().hpmg_uzawa(B.h, C.byref(o), _dp(vel), _dp(p), C.byref(rep)))
    r = UzawaReport(list(rep.inner_iterations[: rep.n_outer]), list(rep.divergence_history[: rep.n_outer]),
                    bool(rep.converged), bool(rep.not_applicable), rep.final_divergence, rep.seconds)
    return StokesSolution(vel, p, r)


@dataclass
class NSReport:
    picard_iterations: int
    newton_iterations: int
    picard_inner: list
    newton_inner: list
    picard_diffs: list
    newton_diffs: list
    converged: bool
    not_applicable: bool
    final_divergence: float
    seconds: float
    setup_seconds: float


@dataclass
class NSSolution:
    velocity: np.ndarray   # full compound
    interior: np.ndarray   # [ne, k(k+1)] interior RT coefficients
    pressure: np.ndarray   # element means
    report: NSReport
    grad: np.ndarray = None  # [ne, 4 ns] gradient variable of the final state (LocalSolution::grad_coeffs)


def navier_stokes_solve(*, mesh="unit_square", base_n=2, levels=2, k=0, nu=1.0, inv_eps=1e6, bc=None, load=None,
                        load_per_element=None, structured_load=None, cycle=CYCLE_W, smoother=SMOOTH_MULTIPLICATIVE,
                        smooth_steps=1, jacobi_damping=1.0 / 3.0, sweep="records", picard_tol=1e-4,
                        newton_rel_tol=1e-8, newton_abs_tol=1e-10, max_picard=60, max_newton=25,
                        pseudo_time_inv=0.0, outer_iterations=2, krylov: KrylovOptions | None = None):
    """Stationary Navier-Stokes driver (reference ns.hpp:69-149): Stokes guess,
    Picard, then Newton, each linearised step on a device hp-MG hierarchy
    rebuilt around the current velocity, warm-started AL-Uzawa."""
    L = lib()
    md = _Mesh()
    rc = (L.hpmg_unit_square_mesh if mesh == "unit_square" else L.hpmg_step_mesh)(base_n, levels, C.byref(md))
    if rc:
        raise HpmgError(L.hpmg_last_error().decode())
    opt = _Options(k, nu, 0.0, 0.0, inv_eps, cycle, smoother, smooth_steps, jacobi_damping, SWEEP_VARIANTS[sweep])
    bcf, bcu, bck = _field_user(bc)
    ldf, ldu, ldk = _field_user(load)
    keep = [bcf, ldf, bck, ldk]
    prob = _Problem(bcf, bcu, ldf, ldu, None, None, None, 0, None, 0, FIELD_FN(), None, None, None)
    if load_per_element is not None:
        a = np.ascontiguousarray(load_per_element, dtype=np.float64)
        keep.append(a)
        prob.load_per_element = _dp(a)
    if structured_load is not None:
        n, arr = structured_load
        a = np.ascontiguousarray(arr, dtype=np.float64)
        keep.append(a)
        prob.structured_load = _dp(a)
        prob.structured_n = int(n)
    krylov = krylov or KrylovOptions()
    o = _NSOpts(picard_tol, newton_rel_tol, newton_abs_tol, max_picard, max_newton, pseudo_time_inv,
                _UOpts(outer_iterations, krylov.c(), None))
    ne = md.n_elements * 4 ** (levels - 1)
    # size of the compound space: 2 (k+1) per facet of the finest mesh (Euler: nf = nv + ne - 1)
    nv = md.n_vertices
    nf_base = nv + md.n_elements - 1
    nf = nf_base
    nv_l, ne_l = nv, md.n_elements
    for _ in range(levels - 1):
        nv_l, nf, ne_l = nv_l + nf, 2 * nf + 3 * ne_l, 4 * ne_l
    vel = np.zeros(2 * (k + 1) * nf)
    interior = np.zeros(max(ne * k * (k + 1), 1))
    pres = np.zeros(ne)
    grad = np.zeros((ne, 2 * (k + 1) * (k + 2)))
    rep = _NSReport()
    rc = L.hpmg_ns_solve(C.byref(md), C.byref(opt), C.byref(prob), C.byref(o), _dp(vel), _dp(interior), _dp(pres),
                         C.byref(rep), None, _dp(grad))
    if rc:
        raise HpmgError(L.hpmg_last_error().decode())
    r = NSReport(rep.picard_iterations, rep.newton_iterations, list(rep.picard_inner[: rep.n_picard_inner]),
                 list(rep.newton_inner[: rep.n_newton_inner]), list(rep.picard_diffs[: rep.picard_iterations]),
                 list(rep.newton_diffs[: rep.newton_iterations]), bool(rep.converged), bool(rep.not_applicable),
                 rep.final_divergence, rep.seconds, rep.setup_seconds)
    return NSSolution(vel, interior[: ne * k * (k + 1)].reshape(ne, k * (k + 1)), pres, r, grad)
