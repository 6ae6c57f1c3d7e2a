"""Splits a device-vs-reference PCG difference into its preconditioner and
Krylov-arithmetic parts: one numpy PCG (reference krylov.hpp:30-73) run with
the reference's, the restatement's and the device's preconditioner apply,
against the reference's own pcg and the device's.

usage: python tools/gpu_floor2.py [k] [inv_eps] [beta] [levels] [base_n]
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


def np_pcg(A, M, b, tol=1e-8, abs_tol=1e-10, max_it=500):
    x = np.zeros_like(b)
    target = max(tol * np.linalg.norm(b), abs_tol)
    r = b - A(x)
    z = M(r)
    rz = r @ z
    p = z.copy()
    for it in range(max_it):
        Ap = A(p)
        alpha = rz / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        if np.linalg.norm(r) <= target:
            return x, it + 1
        z = M(r)
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return x, max_it


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
    rhs = ref.rhs()
    xr, sr = ref.krylov(rhs)
    xg, sg = H.pcg(gpu, rhs)
    out = {}
    for name, M in (("ref", ref.apply), ("orc", orc.apply), ("gpu", gpu.apply)):
        x, its = np_pcg(ref.spmv, M, rhs)
        out[f"numpy_pcg_M_{name}"] = {"its": its, "vs_ref_pcg": rel(x, xr), "vs_gpu_pcg": rel(x, xg)}
    out["gpu_pcg_vs_ref_pcg"] = rel(xg, xr)
    # a tiny symmetric perturbation of the reference preconditioner at the
    # device's apply-difference level: how sensitive is the solve itself?
    rng = np.random.default_rng(5)
    for eps in (1e-12, 4e-12):
        def Mp(v, eps=eps):
            z = ref.apply(v)
            return z * (1.0 + eps * rng.standard_normal(z.shape))
        x, its = np_pcg(ref.spmv, Mp, rhs)
        out[f"numpy_pcg_M_ref_noise{eps:g}"] = {"its": its, "vs_ref_pcg": rel(x, xr)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
