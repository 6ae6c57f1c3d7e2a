"""Development tool: per-pass clock64 timeline of the one-CTA small-level sweep."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_06762_b200 as H  # noqa: E402

B = H.MGPreconditioner(base_n=16, levels=5, k=3, beta=1e-2, inv_eps=1e3, cycle=H.CYCLE_V,
                       structured_load=(256, H.seeded_load(256, 1)))
L = H.lib()
L.hpmg_debug_small_trace.argtypes = [C.c_int, C.c_void_p]
B.apply(np.ones(B.n))
L.hpmg_debug_small_trace(1, None)
B.apply(np.ones(B.n))
out = np.zeros(4096, np.int64)
L.hpmg_debug_small_trace(0, out.ctypes.data)
t = out.reshape(-1, 4)
n = int((t[:, 3] > 0).sum())
t = t[:n]
wait = t[:, 1] - t[:, 0]
res = t[:, 2] - t[:, 1]
gemv = t[:, 3] - t[:, 2]
gap = np.r_[0, t[1:, 0] - t[:-1, 3]]
print("passes", n, "cycles/pass total %.0f" % ((t[-1, 3] - t[0, 0]) / n))
print("wait  median %.0f mean %.0f" % (np.median(wait), wait.mean()))
print("resid median %.0f mean %.0f" % (np.median(res), res.mean()))
print("gemv  median %.0f mean %.0f" % (np.median(gemv), gemv.mean()))
print("gap   median %.0f mean %.0f" % (np.median(gap), gap.mean()))
g = out[4088:4096].astype(np.float64)
print("pre  (ns): load %.0f sweeps %.0f resid+restrict %.0f" % (g[1] - g[0], g[2] - g[1], g[3] - g[2]))
print("post (ns): prolong %.0f sweeps %.0f store %.0f" % (g[5] - g[4], g[6] - g[5], g[7] - g[6]))
print("pre->post gap (ns) %.0f" % (g[4] - g[3]))
