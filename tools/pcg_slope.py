"""Per-iteration cost of the device PCG: slope of solve time vs iteration cap
(same rhs, capped runs), next to the V-cycle and spmv times.
usage: python tools/pcg_slope.py [config]"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
B = H.MGPreconditioner(**R.device_kwargs(name))
rhs = B.rhs()
solver = H.pcg if B.symmetric() else H.gmres


def t(k, reps=5):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        solver(B, rhs, opt=H.KrylovOptions(max_iterations=k, rel_tol=1e-30, abs_tol=0.0))
        best = min(best, time.perf_counter() - t0)
    return best


t(3)
a, b = 5, 25
ta, tb = t(a), t(b)
print(json.dumps({"config": name, "per_iteration_ms": round((tb - ta) / (b - a) * 1e3, 4),
                  "fixed_ms": round((ta - a * (tb - ta) / (b - a)) * 1e3, 3),
                  "vcycle_ms": round(B.time_apply(20)[0], 4), "spmv_ms": round(B.time_spmv(20)[0], 4),
                  "host_loop": os.environ.get("HPMG_KRYLOV_HOST", "0")}))
