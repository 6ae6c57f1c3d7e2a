"""The device path, through the C ABI, against committed outputs of the
reference itself (tests/golden, from oracle/_ref/libref.so = the unmodified
reference headers; tools/make_golden.py). Needs neither /root/reference nor
libref.so on the GPU box. Bounds as in test_gpu_parity.py: rhs to
round-off, operator entrywise <= 1e-13 max|A|, one V-cycle <= 2e-12 at
inv_eps 1e3 (scaled with the penalty), Krylov / Uzawa counts +-1, Krylov
solution <= 1e-8 and Uzawa velocity <= 1e-9 relative L2 (north star). The
advected (Oseen) case takes test_gpu_oseen.py's bounds: one V-cycle <= 1e-10
(explicit nonsymmetric patch inverses against the reference's LU solves),
Uzawa velocity <= 1e-8."""
import numpy as np
import pytest

from golden_cases import NAMES, gpu_kwargs, load, rel

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_2303_06762_b200")


@pytest.mark.parametrize("name", NAMES)
def test_device_matches_reference_golden(name):
    meta, g = load(name)
    gpu = H.MGPreconditioner(**gpu_kwargs(meta, g))
    assert gpu.n == meta["n"]
    assert np.array_equal(gpu.free_to_full(), g["free_to_full"])
    assert rel(gpu.rhs(), g["rhs"]) < 1e-13
    if "A_data" in g:
        import scipy.sparse as sp
        R = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=tuple(g["A_shape"]))
        assert abs(gpu.matrix() - R).max() <= 1e-13 * abs(R).max()
    inv_eps = meta["kwargs"]["inv_eps"]
    advected = meta["krylov"] == "gmres"
    apply_tol = 1e-10 if advected else 2e-12 * max(1.0, inv_eps / 1e3)
    assert rel(gpu.apply(g["apply_in"]), g["apply_out"]) < apply_tol
    solve = H.gmres if advected else H.pcg
    x, st = solve(gpu, gpu.rhs())
    assert st.converged and abs(st.iterations - int(g["krylov_iterations"])) <= 1
    assert rel(x, g["krylov_x"]) < 1e-8
    sol = H.uzawa_solve(gpu)
    assert sol.report.converged
    for a, c in zip(sol.report.inner_iterations, g["uzawa_inner"]):
        assert abs(a - int(c)) <= 1
    assert rel(sol.velocity, g["uzawa_velocity"]) < (1e-8 if advected else 1e-9)
