"""Development A/B: device GMRES / PCG solve time with an alternative build of
libhpmg.so (path in argv[1], or 'cur'), same config and caps; prints ms per
iteration over repeated fixed-length solves. usage: ab_krylov.py LIB [config] [iters] [restart]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402

if sys.argv[1] != "cur":
    H.LIB_PATH = os.path.abspath(sys.argv[1])
import ref_runs as R  # noqa: E402

name = sys.argv[2] if len(sys.argv) > 2 else "config5_re1"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 30
restart = int(sys.argv[4]) if len(sys.argv) > 4 else 50
B = H.MGPreconditioner(**R.device_kwargs(name))
rhs = B.rhs()
solver = H.pcg if B.symmetric() else H.gmres
opt = H.KrylovOptions(max_iterations=iters, rel_tol=1e-30, abs_tol=0.0, restart=restart)
solver(B, rhs, opt=opt)
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    solver(B, rhs, opt=opt)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(json.dumps({"lib": sys.argv[1], "config": name, "iters": iters, "ms_per_iteration_best": round(ts[0] * 1e3 / iters, 4),
                  "ms_per_iteration_median": round(ts[4] * 1e3 / iters, 4), "vcycle_ms": round(B.time_apply(20)[0], 4)}))
