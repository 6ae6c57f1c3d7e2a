"""Result formats of the reference (inc/io.hpp): the benchmark CSV schema and
the MatrixMarket dump, plus the convergence study that fills the CSV's error
columns (tools/hdivmg.cpp:255-330, `eoc` subcommand) run through the device
pipeline (uzawa / NS driver -> recover -> postprocess -> measure_errors)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# io.hpp:16-18
CSV_HEADER = ("run_id,subcommand,k,level,nu,beta,m,cycle,outer,inner_iters,"
              "avg_picard,avg_newton,e_u,e_L,e_ustar,div_u,eoc_u,eoc_L,eoc_ustar,status")


@dataclass
class CsvRow:
    """io.hpp:20-35"""
    run_id: int = 0
    subcommand: str = ""
    k: int = 0
    level: int = 0
    nu: float = 1.0
    beta: float = 0.0
    m: int = 1
    cycle: str = ""
    outer: int = 0
    inner_iters: list = field(default_factory=list)
    avg_picard: Optional[float] = None
    avg_newton: Optional[float] = None
    e_u: Optional[float] = None
    e_L: Optional[float] = None
    e_ustar: Optional[float] = None
    div_u: Optional[float] = None
    eoc_u: Optional[float] = None
    eoc_L: Optional[float] = None
    eoc_ustar: Optional[float] = None
    status: str = "ok"


def _num(v):
    # std::ostream with precision 12 and the default float field (io.hpp:39-44)
    return "%.12g" % v


def _opt(v):
    return "" if v is None else _num(v)


def write_csv_header(os):
    os.write(CSV_HEADER + "\n")


def write_csv_row(os, row: CsvRow):
    """io.hpp:54-70: empty cells for absent values, inner counts joined by ';'."""
    cells = [str(row.run_id), row.subcommand, str(row.k), str(row.level), _num(row.nu), _num(row.beta), str(row.m),
             row.cycle, str(row.outer), ";".join(str(i) for i in row.inner_iters), _opt(row.avg_picard),
             _opt(row.avg_newton), _opt(row.e_u), _opt(row.e_L), _opt(row.e_ustar), _opt(row.div_u), _opt(row.eoc_u),
             _opt(row.eoc_L), _opt(row.eoc_ustar), row.status]
    os.write(",".join(cells) + "\n")


def write_matrix_market(os, A):
    """io.hpp:72-81 for a scipy sparse matrix: coordinate real general,
    1-based, 17 significant digits, column by column (column-major order)."""
    A = A.tocsc()
    A.sort_indices()
    os.write("%%MatrixMarket matrix coordinate real general\n")
    os.write(f"{A.shape[0]} {A.shape[1]} {A.nnz}\n")
    for c in range(A.shape[1]):
        for q in range(A.indptr[c], A.indptr[c + 1]):
            os.write("%d %d %.17g\n" % (A.indices[q] + 1, c + 1, A.data[q]))


def read_matrix_market(fh):
    """Inverse of write_matrix_market (the reference test's round trip)."""
    import scipy.sparse as sp
    banner = fh.readline().rstrip("\n")
    if banner != "%%MatrixMarket matrix coordinate real general":
        raise ValueError(f"unexpected banner {banner!r}")
    rows, cols, nnz = (int(t) for t in fh.readline().split())
    r = np.empty(nnz, np.int64)
    c = np.empty(nnz, np.int64)
    v = np.empty(nnz)
    for e in range(nnz):
        a, b, x = fh.readline().split()
        r[e], c[e], v[e] = int(a) - 1, int(b) - 1, float(x)
    return sp.coo_matrix((v, (r, c)), shape=(rows, cols)).tocsr()


def eoc_study(*, k=0, levels=4, nu=1.0, beta=0.0, m=1, cycle="v", penalty_exponent=6, ns=False,
              pseudo_time_inv=0.0, first_run_id=1):
    """Error and EOC table on the manufactured flow (tools/hdivmg.cpp:255-330,
    option meanings of its RunConfig :27-40 and mg_options :75-81: cycle "w"
    is the W-cycle, anything else the variable V-cycle; inv_eps = nu 10^p).
    For l = 1..levels: unit_square_mesh(2) refined to l levels, homogeneous
    Dirichlet data; Stokes (load stokes_load(nu, beta)) by AL-Uzawa or, with
    ns, stationary Navier-Stokes (load navier_stokes_load(nu)) by the Picard ->
    Newton driver; errors of u_h, L_h, u* and div u_h, EOC against the
    previous converged level. Returns one CsvRow per level."""
    from . import (CYCLE_VARIABLE_V, CYCLE_W, MGPreconditioner, estimated_order, navier_stokes_solve,
                   uzawa_solve)
    cyc = CYCLE_W if cycle == "w" else CYCLE_VARIABLE_V
    inv_eps = nu * 10.0 ** penalty_exponent
    rows, prev = [], None
    for l in range(1, levels + 1):
        row = CsvRow(run_id=first_run_id + l - 1, subcommand="eoc", k=k, level=l, nu=nu, beta=beta, m=m,
                     cycle=cycle)
        err = None
        if ns:
            sol = navier_stokes_solve(base_n=2, levels=l, k=k, nu=nu, inv_eps=inv_eps, cycle=cyc, smooth_steps=m,
                                      load=("mms_ns_load", (nu,)), pseudo_time_inv=pseudo_time_inv)
            r = sol.report
            row.outer = r.picard_iterations + r.newton_iterations
            row.inner_iters = list(r.picard_inner) + list(r.newton_inner)
            if r.picard_inner:
                row.avg_picard = float(np.mean(r.picard_inner))
            if r.newton_inner:
                row.avg_newton = float(np.mean(r.newton_inner))
            status = "NA" if r.not_applicable else ("fail" if not r.converged else "ok")
            if status == "ok":
                row.div_u = r.final_divergence
                B = MGPreconditioner(base_n=2, levels=l, k=k, nu=nu, inv_eps=inv_eps, cycle=cyc, smooth_steps=m)
                post = B.postprocess(sol.velocity, sol.interior, sol.grad)
                err = B.measure_errors(sol.velocity, sol.interior, sol.grad, post, "mms")
        else:
            B = MGPreconditioner(base_n=2, levels=l, k=k, nu=nu, beta=beta, inv_eps=inv_eps, cycle=cyc,
                                 smooth_steps=m, load=("mms_stokes_load", (nu, beta)))
            sol = uzawa_solve(B)
            rep = sol.report
            row.outer, row.inner_iters = len(rep.inner_iterations), list(rep.inner_iterations)
            status = "NA" if rep.not_applicable else ("fail" if not rep.converged else "ok")
            if status == "ok":
                row.div_u = rep.final_divergence
                interior, _, grad = B.recover(sol.velocity)
                post = B.postprocess(sol.velocity, interior, grad)
                err = B.measure_errors(sol.velocity, interior, grad, post, "mms")
        row.status = status
        if err is not None:
            row.e_u, row.e_L, row.e_ustar, row.div_u = err.e_u, err.e_L, err.e_ustar, err.div_u
            if prev is not None:
                row.eoc_u = estimated_order(prev.e_u, err.e_u)
                row.eoc_L = estimated_order(prev.e_L, err.e_L)
                row.eoc_ustar = estimated_order(prev.e_ustar, err.e_ustar)
        prev = err
        rows.append(row)
    return rows
