"""Pins the CPU restatement (oracle/) against the reference ITSELF.

oracle/_ref/libref.so is the unmodified reference headers
(/root/reference/proj/include/hdivmg/*.hpp) compiled against the Eigen-API
shim in oracle/eigen_shim and driven by oracle/ref_capi.cpp (the
reference's own MGPreconditioner, pcg, gmres, uzawa_solve, recover_locals,
velocity_patches). On identical seeded inputs the restatement must equal it
to round-off: operator and right-hand side entrywise, one preconditioner
application, Krylov iteration counts exactly and solutions to the solver
tolerance, the Uzawa report and the recovered locals. The shim evaluates in
plain sequential order, so agreement with an Eigen build is to round-off,
not bitwise.
"""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref/libref.so not built (needs /root/reference)")


def pair(**kw):
    return O.OracleMG(**kw), O.OracleMG(reference=True, **kw)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def stokes(k, base_n=4, levels=3, beta=1.0, inv_eps=1e3, seed=1, **extra):
    n = base_n << (levels - 1)
    kw = dict(base_n=base_n, levels=levels, k=k, beta=beta, inv_eps=inv_eps, load_kind=O.LOAD_ARRAY,
              load=O.seeded_load(n, seed), cycle=O.CYCLE_V)
    kw.update(extra)
    return kw


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_operator_rhs_and_patches_equal_reference(k):
    o, r = pair(**stokes(k))
    assert o.n == r.n and o.n_full == r.n_full
    assert np.array_equal(o.free_to_full(), r.free_to_full())
    A, B = o.csr(), r.csr()
    assert abs(A - B).max() <= 1e-14 * abs(B).max()
    assert rel(o.rhs(), r.rhs()) < 1e-14
    po, pr = o.patches(-1 if k > 0 else 2), r.patches()
    assert len(po) == len(pr) and all(np.array_equal(a, b) for a, b in zip(po, pr))


@pytest.mark.parametrize("k,cycle,smoother", [(0, O.CYCLE_V, O.SM_MULT), (1, O.CYCLE_W, O.SM_MULT),
                                              (2, O.CYCLE_VARV, O.SM_MULT), (3, O.CYCLE_V, O.SM_MULT),
                                              (2, O.CYCLE_V, O.SM_ADD)])
def test_apply_equals_reference(k, cycle, smoother):
    o, r = pair(**stokes(k, cycle=cycle, smoother=smoother))
    b = O.random_vec(o.n, 3)
    assert rel(o.apply(b), r.apply(b)) < 1e-11


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_pcg_and_uzawa_equal_reference(k):
    o, r = pair(**stokes(k))
    xo, so = o.krylov(o.rhs())
    xr, sr = r.krylov(r.rhs())
    assert so["iterations"] == sr["iterations"] and so["converged"] and sr["converged"]
    assert rel(xo, xr) < 1e-10
    uo, ur = o.uzawa(), r.uzawa()
    assert uo["inner_iterations"] == ur["inner_iterations"]
    assert rel(uo["velocity"], ur["velocity"]) < 1e-10
    assert rel(uo["pressure"], ur["pressure"]) < 1e-8


@pytest.mark.parametrize("k,nu", [(1, 1.0), (2, 1e-2)])
def test_oseen_gmres_equals_reference(k, nu):
    # config-5 family at reduced size: lid-driven Oseen with the curl wind
    n = 16
    kw = dict(base_n=4, levels=3, k=k, nu=nu, inv_eps=1e3, bc=O.BC_LID_UNIT, load_kind=O.LOAD_ARRAY,
              load=O.seeded_load(n, 1, -0.1, 0.1), wind=O.WIND_CURL, cycle=O.CYCLE_V)
    o, r = pair(**kw)
    A, B = o.csr(), r.csr()
    assert abs(A - B).max() <= 1e-13 * abs(B).max()
    b = O.random_vec(o.n, 5)
    assert rel(o.apply(b), r.apply(b)) < 1e-11
    xo, so = o.krylov(o.rhs(), method=1)
    xr, sr = r.krylov(r.rhs(), method=1)
    assert so["iterations"] == sr["iterations"]
    assert rel(xo, xr) < 1e-9
    uo, ur = o.uzawa(), r.uzawa()
    assert uo["inner_iterations"] == ur["inner_iterations"]
    assert rel(uo["velocity"], ur["velocity"]) < 1e-9


@pytest.mark.parametrize("k", [1, 2, 3])
def test_recover_locals_equal_reference(k):
    # Pressure modes and the gradient variable live in the unique orthonormal
    # P^k basis and compare entrywise. The interior RT coefficients are
    # coordinates in a basis the reference picks by SVD (fespace.hpp:148-168;
    # any basis of the same space is admissible), so they are
    # compared as the field they describe: the RT L2 norm of the recovered
    # velocity, each side in its own basis.
    o, r = pair(**stokes(k))
    u = r.uzawa()["velocity"]
    (io, po, go), (ir, pr, gr) = o.recover(u), r.recover(u)
    assert np.linalg.norm(po - pr) <= 1e-11 * np.linalg.norm(pr)
    assert np.linalg.norm(go - gr) <= 1e-11 * np.linalg.norm(gr)
    no, nr = o.rt_l2_norm(u, io), r.rt_l2_norm(u, ir)
    assert abs(no - nr) <= 1e-12 * nr


def test_penalised_and_mass_free_sweep_cases():
    # config-3 corners at reduced size: AL 1e4 without mass, AL 1 with mass 1e2
    for inv_eps, beta in ((1e4, 0.0), (1.0, 1e2)):
        o, r = pair(**stokes(2, beta=beta, inv_eps=inv_eps))
        uo, ur = o.uzawa(), r.uzawa()
        assert uo["inner_iterations"] == ur["inner_iterations"]
        assert rel(uo["velocity"], ur["velocity"]) < 1e-9


def test_reference_trace_levels():
    # MGOptions::trace (multigrid.hpp:18-33): entering/leaving residuals of
    # every level, head one index above the finest mesh level
    r = O.OracleMG(reference=True, traced=True, **stokes(2))
    b = O.random_vec(r.n, 3)
    r.apply(b)
    lv, ent, res = r.trace()
    assert lv[0] == 3 and ent[0] == 1 and abs(res[0] - np.linalg.norm(b)) < 1e-12 * np.linalg.norm(b)
    assert lv[-1] == 3 and ent[-1] == 0 and res[-1] < res[0]
    assert sorted(set(lv)) == [0, 1, 2, 3]
