"""The reference's result formats (tests/test_io.cpp): CSV schema, row
formatting with empty gaps, MatrixMarket round trip; plus the native
MatrixMarket writer of the C ABI and the device EOC study (GPU)."""
import io

import numpy as np
import pytest
import scipy.sparse as sp

import oracle_lib as O
from paper_2303_06762_b200 import io as hio


def test_csv_schema_is_stable():
    os_ = io.StringIO()
    hio.write_csv_header(os_)
    assert os_.getvalue() == ("run_id,subcommand,k,level,nu,beta,m,cycle,outer,inner_iters,"
                              "avg_picard,avg_newton,e_u,e_L,e_ustar,div_u,eoc_u,eoc_L,eoc_ustar,status\n")


def test_csv_row_prints_populated_cells_and_leaves_gaps():
    row = hio.CsvRow(run_id=3, subcommand="cavity", k=1, level=5, nu=1e-2, beta=1000.0, m=2, cycle="v", outer=2,
                     inner_iters=[12, 4], div_u=2.5e-9)
    os_ = io.StringIO()
    hio.write_csv_row(os_, row)
    assert os_.getvalue() == "3,cavity,1,5,0.01,1000,2,v,2,12;4,,,,,,2.5e-09,,,,ok\n"
    row.status = "NA"
    row.inner_iters = []
    row.div_u = None
    na = io.StringIO()
    hio.write_csv_row(na, row)
    assert na.getvalue() == "3,cavity,1,5,0.01,1000,2,v,2,,,,,,,,,,,NA\n"


def test_matrix_market_round_trip():
    # the reference test's 7 x 5 pattern, values from mt19937(11) uniform(-1, 1)
    cells = [(i, j) for i in range(7) for j in range(5) if (i + 2 * j) % 3 == 0]
    vals = O.random_vec(len(cells), 11)
    A = sp.coo_matrix((vals, ([c[0] for c in cells], [c[1] for c in cells])), shape=(7, 5)).tocsr()
    os_ = io.StringIO()
    hio.write_matrix_market(os_, A)
    text = os_.getvalue()
    assert text.splitlines()[0] == "%%MatrixMarket matrix coordinate real general"
    assert text.splitlines()[1] == f"7 5 {A.nnz}"
    B = hio.read_matrix_market(io.StringIO(text))
    assert B.shape == (7, 5) and abs(A - B).max() == 0.0


@pytest.mark.gpu
def test_native_matrix_market_writer(tmp_path):
    H = pytest.importorskip("paper_2303_06762_b200")
    B = H.MGPreconditioner(base_n=2, levels=3, k=2, nu=1e-2, inv_eps=1e3, bc="lid_unit", wind="rotation")
    for level in (-1, 0, 2):
        path = tmp_path / f"A{level}.mtx"
        B.write_matrix_market(str(path), level)
        with open(path) as fh:
            M = hio.read_matrix_market(fh)
        A = B.matrix(level)
        assert M.shape == A.shape and abs(M - A).max() == 0.0
        lines = path.read_text().splitlines()
        cols = [int(t.split()[1]) for t in lines[2:]]
        assert cols == sorted(cols)  # column by column (io.hpp:78-80)


@pytest.mark.gpu
@pytest.mark.parametrize("ns", [False, True])
def test_eoc_study_on_device(ns):
    # tools/hdivmg.cpp eoc subcommand: k = 1, three levels
    rows = hio.eoc_study(k=1, levels=3, nu=1.0 if not ns else 0.1, beta=1.0 if not ns else 0.0, ns=ns)
    assert [r.status for r in rows] == ["ok"] * 3
    assert rows[0].eoc_u is None and rows[1].eoc_u is not None
    assert rows[2].eoc_u > 1.75 and rows[2].eoc_L > 1.7 and rows[2].eoc_ustar > 2.5
    out = io.StringIO()
    hio.write_csv_header(out)
    for r in rows:
        hio.write_csv_row(out, r)
    lines = out.getvalue().splitlines()
    assert len(lines) == 4 and all(len(l.split(",")) == 20 for l in lines)
    if not ns:
        # the oracle's pipeline on the same configuration: same errors to solver tolerance
        for r in rows:
            orc = O.OracleMG(base_n=2, levels=r.level, k=1, nu=1.0, beta=1.0, inv_eps=1e6, bc=O.BC_ZERO,
                             load_kind=O.LOAD_MMS_STOKES, cycle=O.CYCLE_VARV)
            sol = orc.uzawa()
            i, _, g = orc.recover(sol["velocity"])
            e = orc.errors(sol["velocity"], i, g, orc.postprocess(sol["velocity"], i, g), O.EXACT_MMS)
            assert abs(r.e_u - e["e_u"]) < 1e-6 * e["e_u"] and abs(r.e_ustar - e["e_ustar"]) < 1e-5 * e["e_ustar"]
            assert all(abs(a - b) <= 1 for a, b in zip(r.inner_iters, sol["inner_iterations"]))
