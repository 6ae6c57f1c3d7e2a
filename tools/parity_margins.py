"""Development: measured GPU-vs-oracle discrepancies behind the parity tolerances."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
from test_gpu_parity import pair, rel, lid_top  # noqa: E402

for k in range(4):
    orc, gpu = pair(k, bc=lid_top)
    x = O.random_vec(orc.n, 5)
    print("k", k, "spmv %.2e rhs %.2e" % (rel(gpu.spmv(x), orc.spmv(x)), rel(gpu.rhs(), orc.rhs())))
for k, cyc, inv_eps in [(0, O.CYCLE_V, 1e3), (1, O.CYCLE_V, 1e3), (2, O.CYCLE_W, 1e3), (3, O.CYCLE_V, 1e3),
                        (1, O.CYCLE_VARV, 1e3), (2, O.CYCLE_V, 1e4), (3, O.CYCLE_V, 1e6)]:
    orc, gpu = pair(k, levels=4, cycle=cyc, inv_eps=inv_eps)
    b = O.random_vec(orc.n, 11)
    print("k", k, "cycle", cyc, "inv_eps %.0e" % inv_eps, "apply %.2e" % rel(gpu.apply(b), orc.apply(b)))
