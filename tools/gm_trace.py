"""Development: in-situ timeline of the device GMRES loop kernels (CTA-0 start
stamps): per-MGS-step spacing, no-op step cost, tail/new-vector/V-cycle gaps."""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

B = H.MGPreconditioner(**R.device_kwargs(sys.argv[1] if len(sys.argv) > 1 else "config5_re1"))
L = H.lib()
L.hpmg_debug_gm_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
rhs = B.rhs()
opt = H.KrylovOptions(max_iterations=30, rel_tol=1e-30, abs_tol=0.0, restart=50)
H.gmres(B, rhs, opt=opt)
L.hpmg_debug_gm_trace(1, None)
H.gmres(B, rhs, opt=opt)
out = np.zeros(1 + 4 * 8192, np.int64)
L.hpmg_debug_gm_trace(0, out.ctypes.data)
k = int(out[0])
ev = out[1:1 + 3 * k].reshape(-1, 3)
end = out[1 + 3 * 8192:1 + 3 * 8192 + k].astype(np.float64)
o = np.argsort(ev[:, 2], kind="stable")
ev, end = ev[o], end[o]
body = (end - ev[:, 2]) * 1e-3
real = (ev[:, 0] == 1) & (end > 0)
ids, steps, t = ev[:, 0], ev[:, 1], ev[:, 2].astype(np.float64) * 1e-3  # us
d = np.diff(t)
nxt = ids[1:]
cur = ids[:-1]
res = {"events": k}
for a, b, name in [(1, 1, "mgs->mgs"), (1, 2, "mgs->noop"), (2, 2, "noop->noop"), (2, 1, "noop->mgs(next body)"),
                   (1, 3, "mgs->tail"), (2, 3, "noop->tail"), (3, 4, "tail->newv"), (4, 1, "newv->first mgs (V-cycle+spmv)")]:
    m = (cur == a) & (nxt == b)
    if m.any():
        res[name] = {"n": int(m.sum()), "median_us": round(float(np.median(d[m])), 2), "mean_us": round(float(d[m].mean()), 2)}
res["mgs CTA-0 body us (median)"] = round(float(np.median(body[real])), 2)
print(json.dumps(res, indent=1))
