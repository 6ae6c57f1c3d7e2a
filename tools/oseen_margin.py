"""Development: V-cycle and GMRES parity margins of the advected (Oseen) path
vs the oracle, for both sweep variants (records, direct_nonsym)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import oracle_lib as O  # noqa: E402
from test_gpu_oseen import pair  # noqa: E402

for nu, sweep in ((1e-2, "records"), (1e-3, "records"), (1e-2, "direct_nonsym"), (1e-3, "direct_nonsym")):
    orc, gpu = pair(2, nu=nu, levels=4, sweep=sweep)
    b = O.random_vec(orc.n, 11)
    xo = orc.apply(b)
    e = np.linalg.norm(gpu.apply(b) - xo) / np.linalg.norm(xo)
    rhs = orc.rhs()
    _, so = orc.krylov(rhs, method=1)
    _, sg = H.gmres(gpu, rhs)
    print(f"{sweep} nu {nu:g}: vcycle rel {e:.2e}  gmres oracle {so['iterations']} gpu {sg.iterations}")
