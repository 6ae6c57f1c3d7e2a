"""Device-vs-reference distance at one config, stage by stage (apply, first
PCG solve, full Uzawa), next to the restatement-vs-reference distance.

usage: python tools/gpu_floor.py [k] [inv_eps] [beta] [levels] [base_n]
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


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


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
    orc = O.OracleMG(**kw)
    gpu = H.MGPreconditioner(base_n=base_n, levels=levels, k=k, beta=beta, inv_eps=inv_eps, structured_load=(n, F),
                             cycle=H.CYCLE_V)
    out = {"ref_is_reference": O.ref_available()}
    b = O.random_vec(ref.n, 3)
    zr = ref.apply(b)
    out["apply_gpu"], out["apply_orc"] = rel(gpu.apply(b), zr), rel(orc.apply(b), zr)
    out["rhs_gpu"] = rel(gpu.rhs(), ref.rhs())
    rhs = ref.rhs()
    xr, sr = ref.krylov(rhs)
    xo, so = orc.krylov(rhs)
    xg, sg = H.pcg(gpu, rhs)
    out["pcg_its"] = [sr["iterations"], so["iterations"], sg.iterations]
    out["pcg_gpu"], out["pcg_orc"] = rel(xg, xr), rel(xo, xr)
    ur, uo, ug = ref.uzawa(), orc.uzawa(), H.uzawa_solve(gpu)
    out["uzawa_its"] = [ur["inner_iterations"], uo["inner_iterations"], ug.report.inner_iterations]
    out["uzawa_gpu"], out["uzawa_orc"] = rel(ug.velocity, ur["velocity"]), rel(uo["velocity"], ur["velocity"])
    out["pressure_gpu"], out["pressure_orc"] = rel(ug.pressure, ur["pressure"]), rel(uo["pressure"], ur["pressure"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
