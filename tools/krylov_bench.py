"""Krylov overhead per iteration: device PCG/GMRES solve time vs the V-cycle
time (graph-launched), per config. Run with HPMG_KRYLOV_HOST=1 for the
host-driven loops. usage: python tools/krylov_bench.py [config2 config1 config5 ...]"""
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

for name in sys.argv[1:] or ["config2", "config1", "config5_re1"]:
    if name == "config5":
        name = "config5_re1"
    B = H.MGPreconditioner(**R.device_kwargs(name))
    rhs = B.rhs()
    solver = H.pcg if B.symmetric() else H.gmres
    opt = H.KrylovOptions(restart=50) if not B.symmetric() else None
    solver(B, rhs, opt=opt)  # warm (graph build)
    t0 = time.perf_counter()
    x, st = solver(B, rhs, opt=opt)
    wall = time.perf_counter() - t0
    ms_v, _ = B.time_apply(20)
    per_it = wall * 1e3 / max(st.iterations, 1)
    print(json.dumps({"config": name, "solver": solver.__name__, "iterations": st.iterations,
                      "solve_ms": round(wall * 1e3, 3), "ms_per_iteration": round(per_it, 4),
                      "vcycle_ms": round(ms_v, 4), "spmv_ms": round(B.time_spmv(20)[0], 4),
                      "host_loop": os.environ.get("HPMG_KRYLOV_HOST", "0")}))
