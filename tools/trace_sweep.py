"""Development: per-CTA phase timeline of the head wave sweep (HPMG_DBG=4 HPMG_SWEEP=waves).
Slots >= 11439 are written only by the first (16639-CTA) wave of a config-2 forward sweep."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_06762_b200 as H  # noqa: E402

B = H.MGPreconditioner(base_n=16, levels=5, k=3, beta=1e-2, inv_eps=1e3, cycle=H.CYCLE_V,
                       structured_load=(256, H.seeded_load(256, 1)))
L = H.lib()
L.hpmg_debug_sweep_trace.argtypes = [C.c_void_p]
n = B.n
x, b = np.zeros(n), np.random.default_rng(1).standard_normal(n)
for _ in range(3):
    B.smooth(-1, 0, x, b, 1)
out = np.zeros(5 * 32768, np.int64)
L.hpmg_debug_sweep_trace(out.ctypes.data)
lo, hi = (11439, 16639) if os.environ.get("HPMG_SWEEP") == "waves" else (0, 32768)
t = out.reshape(-1, 5)[lo:hi].astype(np.float64)
t = t[t[:, 4] > 0]
t0 = t[:, 0].min()
print("CTAs", len(t), "span us %.1f" % ((t[:, 4].max() - t0) / 1e3))
for name, a, c in [("tma A+deps", 0, 1), ("gather", 1, 2), ("resid+S wait", 2, 3), ("gemv", 3, 4), ("total", 0, 4)]:
    d = (t[:, c] - t[:, a]) / 1e3
    print("%-13s median %.2f us  p10 %.2f  p90 %.2f" % (name, np.median(d), np.percentile(d, 10), np.percentile(d, 90)))
