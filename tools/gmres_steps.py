"""Cost of one MGS step in the device GMRES: 24-iteration solves with
GMRES(m) for several m (mean Arnoldi index ~ m/2) on config 5 (Re = 1)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

B = H.MGPreconditioner(**R.device_kwargs("config5_re1"))
rhs = B.rhs()
out = {}
for m in (2, 6, 12, 24):
    opt = H.KrylovOptions(max_iterations=24, rel_tol=1e-30, abs_tol=0.0, restart=m)
    H.gmres(B, rhs, opt=opt)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        H.gmres(B, rhs, opt=opt)
        best = min(best, time.perf_counter() - t0)
    # MGS steps in 24 iterations of GMRES(m): (24/m) cycles x m(m+1)/2 steps
    steps = (24 // m) * m * (m + 1) // 2
    out[m] = {"ms": round(best * 1e3, 3), "mgs_steps": steps}
print(json.dumps(out))
ms = [out[m]["ms"] for m in (2, 24)]
st = [out[m]["mgs_steps"] for m in (2, 24)]
print("per MGS step (us, incl. the extra restart work difference):", round((ms[1] - ms[0]) / (st[1] - st[0]) * 1e3, 2))
