"""GPU-vs-oracle parity of the stationary Navier-Stokes path (SURVEY.md 8(f)
rank 1, reference inc/ns.hpp:69-149): Newton linearisation and pseudo-time
mass-field load in the device condensation, recovery under the same
linearisation, warm-started Uzawa, the RT L2 norm, and the whole
Stokes -> Picard -> Newton driver. Tolerances as in test_gpu_parity.py;
the driver's per-step Krylov counts +-1 and identical Picard/Newton counts."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_2303_06762_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def pair(k, newton=False, mass_coef=0.0, mass_field=False, base_n=2, levels=3, nu=1e-2, inv_eps=1e3, seed=3):
    n_f = base_n << (levels - 1)
    F = O.seeded_load(n_f, seed, -0.1, 0.1)
    orc = O.OracleMG(base_n=base_n, levels=levels, k=k, nu=nu, beta=0.0, mass_coef=mass_coef, inv_eps=inv_eps,
                     bc=O.BC_LID_UNIT, load_kind=O.LOAD_ARRAY, load=F, wind=O.WIND_CURL, cycle=O.CYCLE_V,
                     newton=newton, mass_field=mass_field)
    mf = None
    if mass_field:
        # each side interpolates the field in its own interior basis (basis-dependent coefficients)
        probe = H.MGPreconditioner(base_n=base_n, levels=levels, k=k, nu=nu, inv_eps=inv_eps, bc="lid_unit")
        mf = probe.interpolate("config5_wind")
    gpu = H.MGPreconditioner(base_n=base_n, levels=levels, k=k, nu=nu, beta=0.0, mass_coef=mass_coef,
                             inv_eps=inv_eps, bc="lid_unit", structured_load=(n_f, F), wind="config5_wind",
                             newton=newton, mass_field=mf, cycle=H.CYCLE_V)
    return orc, gpu


def compare_interior(ig, io, k, scale, tol=1e-10):
    """Interior RT coefficients: the divergence-reproducing functions match;
    the k(k-1)/2 divergence-free bubbles are fixed only up to sign (k=2) or
    rotation (k=3) by the basis construction (test_gpu_parity.py)."""
    nb = k * (k - 1) // 2
    ig, io = ig.reshape(len(ig), -1), io.reshape(len(io), -1)
    assert np.abs(ig[:, nb:] - io[:, nb:]).max(initial=0.0) <= tol * scale
    if nb == 1:
        assert np.abs(np.abs(ig[:, 0]) - np.abs(io[:, 0])).max() <= tol * scale


@pytest.mark.parametrize("k", [0, 1, 2])
def test_newton_operator_and_rhs(k):
    orc, gpu = pair(k, newton=True)
    assert not gpu.symmetric()
    x = O.random_vec(orc.n, 5)
    assert rel(gpu.spmv(x), orc.spmv(x)) < 1e-13
    assert rel(gpu.rhs(), orc.rhs()) < 1e-13
    for l in range(3):
        A_g, A_o = gpu.matrix(l), orc.csr(l)
        assert abs(A_g - A_o).max() <= 1e-12 * abs(A_o).max()


@pytest.mark.parametrize("k", [0, 2])
def test_pseudo_time_mass_field_load(k):
    orc, gpu = pair(k, mass_coef=4.0, mass_field=True)
    x = O.random_vec(orc.n, 6)
    assert rel(gpu.spmv(x), orc.spmv(x)) < 1e-13
    assert rel(gpu.rhs(), orc.rhs()) < 1e-13


@pytest.mark.parametrize("k", [1, 2])
def test_newton_gmres_and_recovery(k):
    orc, gpu = pair(k, newton=True, levels=4)
    b = orc.rhs()
    xo, so = orc.krylov(b, method=1)
    xg, sg = H.gmres(gpu, b)
    assert so["converged"] and sg.converged and abs(sg.iterations - so["iterations"]) <= 1
    assert rel(xg, xo) < 1e-8
    # recovery re-eliminates the interior unknowns under the same linearisation
    u = O.random_vec(orc.n_full, 31)  # non-solenoidal: every interior coefficient O(1)
    io, po, go = orc.recover(u)
    ig, pg, gg = gpu.recover(u)
    assert rel(gg.ravel(), go.ravel()) < 1e-10
    assert rel(pg.ravel(), po.ravel()) < 1e-10
    compare_interior(ig, io, k, np.abs(u).max())


def test_warm_started_uzawa():
    orc, gpu = pair(1, levels=4)
    u0 = orc.uzawa(outer=1)["velocity"]  # a nearby state
    ro = orc.uzawa(initial_velocity=u0)
    rg = H.uzawa_solve(gpu, initial_velocity=u0)
    assert ro["converged"] and rg.report.converged
    for a, b in zip(rg.report.inner_iterations, ro["inner_iterations"]):
        assert abs(a - b) <= 1
    assert rel(rg.velocity, ro["velocity"]) < 1e-8
    cold = H.uzawa_solve(gpu)
    assert rg.report.inner_iterations[0] < cold.report.inner_iterations[0]


@pytest.mark.parametrize("k", [0, 1, 3])
def test_rt_l2_norm(k):
    orc, gpu = pair(k)
    # facet (flux) functions are canonical: any compound vector, zero interior
    c = O.random_vec(orc.n_full, 8)
    z = np.zeros(orc.ne * k * (k + 1))
    assert abs(gpu.rt_l2_norm(c, z) - orc.rt_l2_norm(c, z)) <= 1e-13 * orc.rt_l2_norm(c, z)
    # a field interpolated by each side in its own interior basis has one norm
    cg, ig = gpu.interpolate("config5_wind")
    co, io = orc.wind()
    assert rel(cg, co) < 1e-14
    ng, no = gpu.rt_l2_norm(cg, ig), orc.rt_l2_norm(co, io)
    exact = np.pi * np.sqrt(3.0 / 8.0)  # ||curl(sin^2 pi x sin^2 pi y)||_L2 on the unit square
    assert abs(ng - no) <= 1e-13 * no and abs(no - exact) < 0.25 * exact


@pytest.mark.parametrize("k,nu,pseudo,max_picard", [(1, 1e-2, 0.0, 60), (2, 1e-2, 0.0, 60), (1, 4e-3, 20.0, 10)])
def test_navier_stokes_driver(k, nu, pseudo, max_picard):
    # lid-driven cavity, Re = 1/nu, Stokes -> Picard -> Newton on an 8x8 mesh;
    # the Re = 250 case runs pseudo-time Picard steps (mass field load)
    kw = dict(base_n=2, levels=3, k=k, nu=nu, inv_eps=1e3, picard_tol=1e-4, pseudo_time_inv=pseudo,
              max_picard=max_picard)
    ro = O.ns_solve(bc=O.BC_LID_UNIT, cycle=O.CYCLE_V, **kw)
    rg = H.navier_stokes_solve(bc="lid_unit", cycle=H.CYCLE_V, **kw)
    g = rg.report
    assert ro["converged"] and g.converged
    assert g.picard_iterations == ro["picard_iterations"]
    assert g.newton_iterations == ro["newton_iterations"]
    for a, b in zip(g.picard_inner + g.newton_inner, ro["picard_inner"] + ro["newton_inner"]):
        assert abs(a - b) <= 1
    for a, b in zip(g.picard_diffs, ro["picard_diffs"]):
        assert abs(a - b) <= 1e-6 * b
    assert g.newton_diffs[-1] < 1e-8 * max(1.0, np.linalg.norm(rg.velocity))  # quadratic convergence reached
    assert rel(rg.velocity, ro["velocity"]) < 1e-8
    assert rel(rg.pressure, ro["pressure"]) < 1e-7
    compare_interior(rg.interior, ro["interior"].reshape(rg.interior.shape), k, np.abs(ro["velocity"]).max(), 1e-7)


def lid_top(x, y):
    return (4 * x * (1 - x), 0.0) if y > 1.0 - 1e-12 else (0.0, 0.0)


def test_navier_stokes_newton_quadratic_on_device():
    # reference tests/test_ns.cpp:58-73 on the device driver: early hand-over,
    # variable V-cycle, Newton updates shrink quadratically
    r = H.navier_stokes_solve(base_n=2, levels=3, k=0, nu=1e-2, inv_eps=1e4, bc=lid_top, cycle=H.CYCLE_VARIABLE_V,
                              picard_tol=1e-1).report
    assert r.converged and len(r.newton_diffs) >= 3
    d = r.newton_diffs
    assert d[1] < 5.0 * d[0] ** 2 and d[2] < 5.0 * d[1] ** 2
    assert d[1] < 0.1 * d[0] and d[2] < 0.1 * d[1]
    ro = O.ns_solve(base_n=2, levels=3, k=0, nu=1e-2, inv_eps=1e4, bc=O.BC_LID_TOP, cycle=O.CYCLE_VARV,
                    picard_tol=1e-1)
    assert r.picard_iterations == ro["picard_iterations"] and r.newton_iterations == ro["newton_iterations"]


@pytest.mark.parametrize("k", [0, 2])
def test_update_in_place_equals_fresh_context(k):
    # hpmg_update re-linearises the hierarchy in place: Picard wind -> Newton
    # about a second wind with a pseudo-time mass field and a new nu; the result
    # must be bit-identical to a context created for the final state
    n_f = 8
    F = O.seeded_load(n_f, 3, -0.1, 0.1)
    base = dict(base_n=2, levels=3, k=k, inv_eps=1e3, bc="lid_unit", structured_load=(n_f, F), cycle=H.CYCLE_V)
    gpu = H.MGPreconditioner(nu=1e-2, wind="rotation", **base)
    probe = H.MGPreconditioner(nu=1e-2, **base)
    w2 = probe.interpolate("config5_wind")
    gpu.update(wind=w2, newton=True, mass_field=w2, nu=5e-3, mass_coef=3.0)
    fresh = H.MGPreconditioner(nu=5e-3, mass_coef=3.0, wind=w2, newton=True, mass_field=w2, **base)
    b = O.random_vec(gpu.n, 4)
    assert np.array_equal(gpu.rhs(), fresh.rhs())
    assert np.array_equal(gpu.spmv(b), fresh.spmv(b))
    assert np.array_equal(gpu.apply(b), fresh.apply(b))
    u = O.random_vec(gpu.n_full, 5)
    for a, c in zip(gpu.recover(u), fresh.recover(u)):
        assert np.array_equal(a, c)
    with pytest.raises(H.HpmgError):
        gpu.update()  # advected -> Stokes is a structural change
