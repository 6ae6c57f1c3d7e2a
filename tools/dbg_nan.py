"""Development: locate the first divergence from the oracle in the advected
path, optionally after running other GPU tests in the same process."""
import sys, numpy as np
import pytest
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
if len(sys.argv) > 1:
    pytest.main(["-q", "-m", "gpu", "-p", "no:cacheprovider"] + sys.argv[1:])
import oracle_lib as O
import paper_2303_06762_b200 as H
from test_gpu_oseen import pair, rel


def dense(A):
    return np.asarray(A.toarray() if hasattr(A, "toarray") else A)


for k, nu in [(1, 1e-2), (0, 1.0), (2, 1e-2)]:
    orc, gpu = pair(k, nu=nu, levels=4)
    for l in range(4):
        d, o = dense(gpu.matrix(l)), dense(orc.csr(l))
        print(k, "level", l, "nonfinite", int((~np.isfinite(d)).sum()), "maxdiff", float(np.nanmax(abs(d - o))))
    b = O.random_vec(orc.n, 11)
    print(k, "spmv", rel(gpu.spmv(b), orc.spmv(b)), "apply", rel(gpu.apply(b), orc.apply(b)))
    for lv in range(1, 4):
        nl = gpu.level_n(lv)
        bl, xl = O.random_vec(nl, 7), O.random_vec(nl, 9)
        for which in (0, 1):
            print(k, "smooth level", lv, which, rel(gpu.smooth(lv, which, xl, bl, 1), orc.smooth(lv, which, xl, bl, 1)))
    b = orc.rhs()
    xo, so = orc.krylov(b, method=1)
    xg, sg = H.gmres(gpu, b)
    print(k, "gmres", so["iterations"], sg, rel(xg, xo))
