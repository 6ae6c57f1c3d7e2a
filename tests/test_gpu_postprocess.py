"""Device post-processing and error measurement (SURVEY.md 8(f) rank 3,
reference inc/postprocess.hpp) against the oracle, and the known answers of
the reference's tests/test_postprocess.cpp reproduced through the device
pipeline (uzawa -> recover -> postprocess -> measure_errors).

Parity is on the velocity each side recovers from the SAME compound vector:
the gradient variable and u* are basis-independent (orthonormal scalar
bases), the interior RT coefficients are not (test_gpu_navier_stokes.py), so
every comparison goes through quantities both sides define identically.
Tolerances: 1e-11 relative for u* (a 14x14 SPD solve per element at k = 3, in
a different summation order: reference-tensor contraction on the device,
quadrature loop in the oracle), 1e-10 relative for the error norms."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_2303_06762_b200")

POST_TOL = 1e-11
ERR_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def pair(k, levels, nu=1.0, beta=1.0, manufactured=True):
    if manufactured:
        orc = O.OracleMG(base_n=2, levels=levels, k=k, nu=nu, beta=beta, inv_eps=1e6 * nu, bc=O.BC_ZERO,
                         load_kind=O.LOAD_MMS_STOKES)
        gpu = H.MGPreconditioner(base_n=2, levels=levels, k=k, nu=nu, beta=beta, inv_eps=1e6 * nu,
                                 load=("mms_stokes_load", (nu, beta)))
    else:
        orc = O.OracleMG(base_n=2, levels=levels, k=k, nu=nu, beta=beta, inv_eps=1e6 * nu, bc=O.BC_LINEAR_FLOW,
                         load_kind=O.LOAD_LINEAR_FLOW)
        gpu = H.MGPreconditioner(base_n=2, levels=levels, k=k, nu=nu, beta=beta, inv_eps=1e6 * nu,
                                 bc="linear_flow", load="linear_flow_load")
    return orc, gpu


def device_pipeline(gpu, exact, krylov=None):
    sol = H.uzawa_solve(gpu, krylov=krylov)
    interior, _, grad = gpu.recover(sol.velocity)
    post = gpu.postprocess(sol.velocity, interior, grad)
    return sol, gpu.measure_errors(sol.velocity, interior, grad, post, exact)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_postprocess_and_errors_match_oracle(k):
    orc, gpu = pair(k, 3)
    assert rel(gpu.rhs(), orc.rhs()) < 1e-13  # the named device-side load is the oracle's
    u = orc.uzawa()["velocity"]
    io, _, go = orc.recover(u)
    ig, _, gg = gpu.recover(u)
    assert rel(gg.ravel(), go.ravel()) < 1e-10
    po = orc.postprocess(u, io, go)
    pg = gpu.postprocess(u, ig, gg)
    assert pg.shape == po.shape == (orc.ne, (k + 2) * (k + 3))
    assert rel(pg, po) < POST_TOL
    eo = orc.errors(u, io, go, po, O.EXACT_MMS)
    eg = gpu.measure_errors(u, ig, gg, pg, "mms")
    for key in ("e_u", "e_L", "e_ustar"):
        assert abs(getattr(eg, key) - eo[key]) <= ERR_TOL * eo[key], key
    assert abs(eg.div_u - eo["div_u"]) <= 1e-12 + ERR_TOL * eo["div_u"]


@pytest.mark.parametrize("k", [2, 3])
def test_postprocess_random_data_matches_oracle(k):
    # arbitrary (non-solution) data: random compound, random non-bubble interior
    # coefficients (the k(k-1)/2 divergence-free bubbles are basis-specific, so
    # they are zero), random gradient coefficients
    orc, gpu = pair(k, 2)
    rng = np.random.default_rng(11)
    c = rng.normal(size=orc.n_full)
    nb, no = k * (k - 1) // 2, k * (k + 1)
    i = rng.normal(size=(orc.ne, no))
    i[:, :nb] = 0.0
    ns = (k + 1) * (k + 2) // 2
    g = rng.normal(size=(orc.ne, 4 * ns))
    po = orc.postprocess(c, i, g)
    pg = gpu.postprocess(c, i, g)
    assert rel(pg, po) < POST_TOL
    eo = orc.errors(c, i, g, po, O.EXACT_MMS)
    eg = gpu.measure_errors(c, i, g, pg, "mms")
    assert np.allclose([eg.e_u, eg.e_L, eg.e_ustar, eg.div_u], [eo["e_u"], eo["e_L"], eo["e_ustar"], eo["div_u"]],
                       rtol=ERR_TOL, atol=0)


def test_host_callback_exact_flow_equals_device_flow():
    _, gpu = pair(1, 2)
    sol = H.uzawa_solve(gpu)
    interior, _, grad = gpu.recover(sol.velocity)
    post = gpu.postprocess(sol.velocity, interior, grad)
    dev = gpu.measure_errors(sol.velocity, interior, grad, post, "mms")

    def G(s):
        return s * s * (s - 1) ** 2

    def G1(s):
        return 2 * s * (s - 1) * (2 * s - 1)

    def G2(s):
        return 12 * s * s - 12 * s + 2

    u = lambda x, y: (-G(x) * G1(y), G1(x) * G(y))
    du = lambda x, y: ((-G1(x) * G1(y), -G(x) * G2(y)), (G2(x) * G(y), G1(x) * G1(y)))
    host = gpu.measure_errors(sol.velocity, interior, grad, post, (u, du))
    for key in ("e_u", "e_L", "e_ustar", "div_u"):
        assert abs(getattr(host, key) - getattr(dev, key)) <= 1e-13 * max(getattr(dev, key), 1e-300) + 1e-300


def test_linear_flow_reproduced_exactly():
    # test_postprocess.cpp:120-157 through the device pipeline
    orc, gpu = pair(1, 2, nu=0.5, beta=2.0, manufactured=False)
    sol, err = device_pipeline(gpu, "linear_flow", H.KrylovOptions(rel_tol=1e-12, abs_tol=1e-13))
    assert sol.report.converged
    assert err.e_u < 1e-7 and err.e_L < 1e-7 and err.e_ustar < 1e-7 and err.div_u < 1e-9
    c = orc.centroids()
    assert np.abs(sol.pressure - (c[:, 0] + c[:, 1] - 1.0)).max() < 1e-4


@pytest.mark.parametrize("k", [0, 1, 2])
def test_reconstruction_gains_one_order(k):
    # test_postprocess.cpp:227-260 through the device pipeline
    _, gc = pair(k, 2)
    _, gf = pair(k, 3)
    sc, c = device_pipeline(gc, "mms")
    sf, f = device_pipeline(gf, "mms")
    assert sc.report.converged and sf.report.converged and c.div_u < 1e-10 and f.div_u < 1e-10
    eoc = lambda key: H.estimated_order(getattr(c, key), getattr(f, key))
    if k == 0:
        assert eoc("e_u") > 0.9 and eoc("e_L") > 0.7
    elif k == 1:
        assert eoc("e_u") > 1.75 and eoc("e_L") > 1.7 and eoc("e_ustar") > 2.7 and f.e_ustar < 0.25 * f.e_u
    else:
        assert eoc("e_u") > 2.6 and eoc("e_L") > 2.5 and eoc("e_ustar") > 3.4


def test_order_three_and_navier_stokes_manufactured():
    # beyond the reference's orders: k = 3 gains one order after reconstruction;
    # the manufactured NS load drives the device NS driver to the exact flow
    _, gc = pair(3, 2)
    _, gf = pair(3, 3)
    (_, c), (_, f) = device_pipeline(gc, "mms"), device_pipeline(gf, "mms")
    assert H.estimated_order(c.e_u, f.e_u) > 3.5 and H.estimated_order(c.e_ustar, f.e_ustar) > 4.4
    errs = []
    for levels in (2, 3):
        r = H.navier_stokes_solve(base_n=2, levels=levels, k=1, nu=0.1, inv_eps=1e5, load=("mms_ns_load", (0.1,)))
        assert r.report.converged
        gpu = H.MGPreconditioner(base_n=2, levels=levels, k=1, nu=0.1, inv_eps=1e5)
        post = gpu.postprocess(r.velocity, r.interior, r.grad)
        errs.append(gpu.measure_errors(r.velocity, r.interior, r.grad, post, "mms"))
    for key in ("e_u", "e_L"):
        assert H.estimated_order(getattr(errs[0], key), getattr(errs[1], key)) > 1.7, key
    assert errs[1].e_ustar < 0.5 * errs[1].e_u
