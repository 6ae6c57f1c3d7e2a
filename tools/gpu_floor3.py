"""Operator part of a device-vs-reference solve difference: numpy PCG with
the device operator (and the reference preconditioner), and with the
reference operator perturbed entrywise at the measured device-vs-reference
operator difference (what any re-assembly in another rounding order does).

usage: python tools/gpu_floor3.py [k] [inv_eps] [beta] [levels] [base_n]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
import paper_2303_06762_b200 as H  # noqa: E402
from gpu_floor2 import np_pcg, rel  # noqa: E402


def main():
    a = sys.argv[1:]
    k = int(a[0]) if a else 2
    inv_eps = float(a[1]) if len(a) > 1 else 1e4
    beta = float(a[2]) if len(a) > 2 else 0.0
    levels = int(a[3]) if len(a) > 3 else 5
    base_n = int(a[4]) if len(a) > 4 else 8
    n = base_n << (levels - 1)
    F = O.seeded_load(n, 1)
    kw = dict(base_n=base_n, levels=levels, k=k, beta=beta, inv_eps=inv_eps, load_kind=O.LOAD_ARRAY, load=F,
              cycle=O.CYCLE_V)
    ref = O.OracleMG(reference=O.ref_available(), **kw)
    gpu = H.MGPreconditioner(base_n=base_n, levels=levels, k=k, beta=beta, inv_eps=inv_eps, structured_load=(n, F),
                             cycle=H.CYCLE_V) if len(a) < 6 else None
    rhs = ref.rhs()
    xr, _ = ref.krylov(rhs)
    Ar = ref.csr()
    out = {}
    if gpu is not None:
        Ag = gpu.matrix()
        D = (Ag - Ar).tocoo()
        out["A_maxdiff_rel_max"] = float(abs(D).max() / abs(Ar).max())
        out["A_entry_rel_median"] = float(np.median(np.abs(D.data) / np.maximum(np.abs(Ar.tocsr()[D.row, D.col]).A1, 1e-300)))
        x, its = np_pcg(lambda v: Ag @ v, ref.apply, rhs)
        out["numpy_pcg_A_gpu_M_ref"] = {"its": its, "vs_ref_pcg": rel(x, xr)}
        xg, _ = H.pcg(gpu, rhs)
        out["numpy_pcg_A_gpu_vs_gpu_pcg"] = rel(x, xg)
    rng = np.random.default_rng(7)
    for eps in (1e-16, 1e-15):
        P = Ar.tocoo()
        noise = eps * rng.standard_normal(P.nnz)
        Pn = P.copy()
        Pn.data = P.data * (1.0 + noise)
        Pn = Pn.tocsr()
        Pn = 0.5 * (Pn + Pn.T)  # keep it symmetric (the reference's A is)
        x, its = np_pcg(lambda v: Pn @ v, ref.apply, rhs)
        out[f"numpy_pcg_A_ref_noise{eps:g}"] = {"its": its, "vs_ref_pcg": rel(x, xr)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
