"""Pins of the oracle's post-processing and error measurement against the
known answers of the reference's own tests (tests/test_postprocess.cpp):
manufactured source terms vs finite differences, exact reproduction of a
linear flow through the whole pipeline, element means and the weak gradient
equation of u*, and the convergence orders on the manufactured flow."""
import numpy as np
import pytest

import oracle_lib as O


def pipeline(k, levels, *, nu, beta, bc, load_kind, exact, rel_tol=1e-8, abs_tol=1e-10):
    """run_pipeline (test_postprocess.cpp:21-41): unit_square_mesh(2) refined,
    inv_eps = 1e6 nu, default MG options, uzawa, recover, postprocess, measure."""
    orc = O.OracleMG(base_n=2, levels=levels, k=k, nu=nu, beta=beta, inv_eps=1e6 * nu, bc=bc, load_kind=load_kind)
    sol = orc.uzawa(rel_tol=rel_tol, abs_tol=abs_tol)
    interior, _, grad = orc.recover(sol["velocity"])
    post = orc.postprocess(sol["velocity"], interior, grad)
    return orc, sol, orc.errors(sol["velocity"], interior, grad, post, exact)


def test_manufactured_sources_match_finite_differences():
    rng = np.random.default_rng(7)
    h, nu, beta = 1e-4, 0.7, 3.2
    u = lambda x, y: O.mms_point(x, y, nu, beta)[0:2]
    p = lambda x, y: O.mms_point(x, y, nu, beta)[8]
    for _ in range(20):
        x, y = rng.uniform(0.05, 0.95, 2)
        v = O.mms_point(x, y, nu, beta)
        lap = (u(x + h, y) + u(x - h, y) + u(x, y + h) + u(x, y - h) - 4 * u(x, y)) / h**2
        gp = np.array([p(x + h, y) - p(x - h, y), p(x, y + h) - p(x, y - h)]) / (2 * h)
        g = np.column_stack([(u(x + h, y) - u(x - h, y)) / (2 * h), (u(x, y + h) - u(x, y - h)) / (2 * h)])
        assert np.linalg.norm(v[11:13] - (-nu * lap + beta * v[0:2] + gp)) < 1e-5
        v_ns = O.mms_point(x, y, 0.05, 0.0)
        assert np.linalg.norm(v_ns[13:15] - (-0.05 * lap + g @ v[0:2] + gp)) < 1e-5
        assert abs(v[2] + v[5]) < 1e-15 and abs(np.trace(g)) < 1e-7
        assert np.allclose(v[2:6].reshape(2, 2), g, atol=1e-6)
    for s in np.linspace(0, 1, 11):
        for x, y in ((0, s), (1, s), (s, 0), (s, 1)):
            assert np.linalg.norm(O.mms_point(x, y, nu, beta)[0:2]) == 0.0
    t, w = np.polynomial.legendre.leggauss(8)
    X, Y = np.meshgrid(0.5 * (t + 1), 0.5 * (t + 1))
    P = np.vectorize(lambda a, b: O.mms_point(a, b, nu, beta)[8])(X, Y)
    assert abs(0.25 * w @ P @ w) < 1e-14


def test_linear_flow_reproduced_exactly():
    orc, sol, err = pipeline(1, 2, nu=0.5, beta=2.0, bc=O.BC_LINEAR_FLOW, load_kind=O.LOAD_LINEAR_FLOW,
                             exact=O.EXACT_LINEAR, rel_tol=1e-12, abs_tol=1e-13)
    assert sol["converged"]
    assert err["e_u"] < 1e-7 and err["e_L"] < 1e-7 and err["e_ustar"] < 1e-7 and err["div_u"] < 1e-9
    c = orc.centroids()
    assert np.abs(sol["pressure"] - (c[:, 0] + c[:, 1] - 1.0)).max() < 1e-4


def test_postprocess_means_and_weak_gradient():
    mean_err, residual = O.check("orc_check_postprocess_weak", n_out=2)
    assert mean_err < 1e-11 and residual < 1e-10


def eoc(c, f, key):
    return np.log2(c[key] / f[key])


@pytest.mark.parametrize("k", [0, 1, 2])
def test_reconstruction_gains_one_order(k):
    kw = dict(nu=1.0, beta=1.0, bc=O.BC_ZERO, load_kind=O.LOAD_MMS_STOKES, exact=O.EXACT_MMS)
    _, sc, c = pipeline(k, 2, **kw)
    _, sf, f = pipeline(k, 3, **kw)
    assert sc["converged"] and sf["converged"] and c["div_u"] < 1e-10 and f["div_u"] < 1e-10
    if k == 0:
        assert eoc(c, f, "e_u") > 0.9 and eoc(c, f, "e_L") > 0.7
    elif k == 1:
        assert eoc(c, f, "e_u") > 1.75 and eoc(c, f, "e_L") > 1.7 and eoc(c, f, "e_ustar") > 2.7
        assert f["e_ustar"] < 0.25 * f["e_u"]
    else:
        assert eoc(c, f, "e_u") > 2.6 and eoc(c, f, "e_L") > 2.5 and eoc(c, f, "e_ustar") > 3.4
