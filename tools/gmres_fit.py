"""Per-MGS-step and per-iteration cost of the device GMRES: unrestarted solves
capped at k iterations (k = 4..40), least-squares fit of
T(k) = a + b k + s k(k+1)/2 (s = one Gram-Schmidt step). usage: gmres_fit.py [config]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5_re1"
B = H.MGPreconditioner(**R.device_kwargs(name))
rhs = B.rhs()
ks = [4, 8, 12, 16, 20, 24, 28, 32, 36, 40]
ts = []
for k in ks:
    opt = H.KrylovOptions(max_iterations=k, rel_tol=1e-30, abs_tol=0.0, restart=64)
    H.gmres(B, rhs, opt=opt)
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        H.gmres(B, rhs, opt=opt)
        best = min(best, time.perf_counter() - t0)
    ts.append(best * 1e3)
k = np.array(ks, float)
M = np.c_[np.ones_like(k), k, k * (k + 1) / 2]
a, b, s = np.linalg.lstsq(M, np.array(ts), rcond=None)[0]
print(json.dumps({"config": name, "fixed_ms": round(a, 3), "per_iteration_ms": round(b, 4), "per_mgs_step_us": round(s * 1e3, 2),
                  "vcycle_ms": round(B.time_apply(20)[0], 4), "spmv_ms": round(B.time_spmv(20)[0], 4),
                  "times_ms": [round(t, 3) for t in ts]}))
