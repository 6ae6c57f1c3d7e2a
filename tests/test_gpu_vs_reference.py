"""Device against the reference ITSELF (oracle/_ref/libref.so: the unmodified
reference headers over the Eigen-API shim) across the features the
BASELINE configs do not exercise: the backward-facing-step domain with an
inhomogeneous inlet profile and an outflow (do-nothing) boundary, W and
variable-V cycles with two smoothing steps, the additive smoother, the
rotation wind with the Newton linearisation, and the stationary
Navier-Stokes driver (reference ns.hpp:69-149). Tolerances as in
test_gpu_parity.py; counts +-1; Uzawa velocities <= 1e-9; single Krylov
solves and the Picard/Newton driver 1e-8."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="reference library not built")]

H = pytest.importorskip("paper_2303_06762_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def inlet(x, y):  # reference tests' step inflow (BC_INLET): parabolic on x = 0
    return (16.0 * (1.0 - y) * (y - 0.5), 0.0) if x < 1e-12 else (0.0, 0.0)


def lid_top(x, y):
    return (4 * x * (1 - x), 0.0) if y > 1.0 - 1e-12 else (0.0, 0.0)


@pytest.mark.parametrize("k,cycle,m", [(0, O.CYCLE_W, 2), (1, O.CYCLE_VARV, 1), (2, O.CYCLE_W, 2),
                                       (3, O.CYCLE_V, 1)])
def test_step_domain_inlet_outflow(k, cycle, m):
    kw = dict(base_n=2, levels=3, k=k, beta=0.0, inv_eps=1e3, cycle=cycle, smooth_steps=m)
    ref = O.OracleMG(reference=True, mesh_kind=1, bc=O.BC_INLET, **kw)
    gpu = H.MGPreconditioner(mesh="step", bc=inlet, **kw)
    assert gpu.n == ref.n and np.array_equal(gpu.free_to_full(), ref.free_to_full())
    A_g, A_r = gpu.matrix(), ref.csr()
    assert abs(A_g - A_r).max() <= 1e-13 * abs(A_r).max()
    assert rel(gpu.rhs(), ref.rhs()) < 1e-13
    b = O.random_vec(ref.n, 3)
    assert rel(gpu.apply(b), ref.apply(b)) < 2e-12
    ur, ug = ref.uzawa(), H.uzawa_solve(gpu)
    assert ug.report.converged and ur["converged"]
    for a, c in zip(ug.report.inner_iterations, ur["inner_iterations"]):
        assert abs(a - c) <= 1
    assert rel(ug.velocity, ur["velocity"]) < 1e-9
    assert rel(ug.pressure, ur["pressure"]) < 1e-7


@pytest.mark.parametrize("k", [1, 2])
def test_additive_smoother(k):
    kw = dict(base_n=2, levels=3, k=k, beta=1.0, inv_eps=1e3, cycle=O.CYCLE_V, smoother=O.SM_ADD, smooth_steps=2)
    ref = O.OracleMG(reference=True, bc=O.BC_LID_TOP, **kw)
    gpu = H.MGPreconditioner(bc=lid_top, **kw)
    b = O.random_vec(ref.n, 5)
    assert rel(gpu.apply(b), ref.apply(b)) < 2e-12
    xr, sr = ref.krylov(ref.rhs())
    xg, sg = H.pcg(gpu, ref.rhs())
    assert abs(sg.iterations - sr["iterations"]) <= 1
    assert rel(xg, xr) < 1e-8  # one PCG solve to 1e-8 (test_gpu_parity.py: same bound)


@pytest.mark.parametrize("newton", [False, True])
def test_rotation_wind_picard_and_newton(newton):
    kw = dict(base_n=2, levels=3, k=1, nu=2e-2, beta=0.0, inv_eps=1e3, cycle=O.CYCLE_V)
    ref = O.OracleMG(reference=True, bc=O.BC_LID_UNIT, wind=O.WIND_ROT, newton=newton, **kw)
    gpu = H.MGPreconditioner(bc="lid_unit", wind="rotation", newton=newton, **kw)
    assert not gpu.symmetric()
    A_g, A_r = gpu.matrix(), ref.csr()
    assert abs(A_g - A_r).max() <= 1e-12 * abs(A_r).max()
    assert rel(gpu.rhs(), ref.rhs()) < 1e-12
    xr, sr = ref.krylov(ref.rhs(), method=1)
    xg, sg = H.gmres(gpu, ref.rhs())
    assert abs(sg.iterations - sr["iterations"]) <= 1
    assert rel(xg, xr) < 1e-8


@pytest.mark.parametrize("k", [0, 1, 2])
def test_navier_stokes_driver(k):
    kw = dict(base_n=2, levels=3, k=k, nu=1e-2, inv_eps=1e3)
    ref = O.ns_solve(reference=True, bc=O.BC_LID_UNIT, cycle=O.CYCLE_V, **kw)
    gpu = H.navier_stokes_solve(bc="lid_unit", cycle=H.CYCLE_V, **kw)
    assert gpu.report.converged and ref["converged"]
    assert gpu.report.picard_iterations == ref["picard_iterations"]
    assert gpu.report.newton_iterations == ref["newton_iterations"]
    for a, c in zip(gpu.report.picard_inner + gpu.report.newton_inner, ref["picard_inner"] + ref["newton_inner"]):
        assert abs(a - c) <= 1
    assert rel(gpu.velocity, ref["velocity"]) < 1e-8
    assert rel(gpu.pressure, ref["pressure"]) < 1e-6
