"""The CPU restatement (oracle/) against committed outputs of the reference
itself (tests/golden, written by tools/make_golden.py from oracle/_ref/
libref.so: the unmodified reference headers over the Eigen-API shim). Runs
without /root/reference or libref.so: the pins of test_reference_pins.py,
frozen. Same bounds as there: operator and rhs to round-off, one
preconditioner application <= 1e-11, Krylov and Uzawa iteration counts
exactly equal, solutions to the solver tolerance."""
import numpy as np
import pytest

import oracle_lib as O
from golden_cases import NAMES, load, oracle_kwargs, rel


@pytest.mark.parametrize("name", NAMES)
def test_restatement_matches_reference_golden(name):
    meta, g = load(name)
    orc = O.OracleMG(**oracle_kwargs(meta, g))
    assert orc.n == meta["n"]
    assert np.array_equal(orc.free_to_full(), g["free_to_full"])
    assert rel(orc.rhs(), g["rhs"]) < 1e-13
    if "A_data" in g:
        A = orc.csr().tocsr()
        import scipy.sparse as sp
        R = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=tuple(g["A_shape"]))
        assert abs(A - R).max() <= 1e-13 * abs(R).max()
    assert rel(orc.apply(g["apply_in"]), g["apply_out"]) < 1e-11 * max(1.0, meta["kwargs"]["inv_eps"] / 1e3)
    x, st = orc.krylov(orc.rhs(), method=1 if meta["krylov"] == "gmres" else 0)
    assert st["iterations"] == int(g["krylov_iterations"])
    assert rel(x, g["krylov_x"]) < 1e-8
    uz = orc.uzawa()
    assert uz["inner_iterations"] == [int(i) for i in g["uzawa_inner"]]
    assert rel(uz["velocity"], g["uzawa_velocity"]) < 1e-9


def test_golden_index_is_the_reference():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "index.json")) as f:
        src = json.load(f)["_source"]
    assert "oracle/_ref/libref.so" in src and "unmodified reference headers" in src
