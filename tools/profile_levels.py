"""Per-level V-cycle time split on the GPU (development tool)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_06762_b200 as H  # noqa: E402

CFG = {"config2": dict(base_n=16, levels=5, k=3, beta=1e-2, inv_eps=1e3),
       "config1": dict(base_n=8, levels=5, k=1, beta=1.0, inv_eps=1e3),
       "config3": dict(base_n=8, levels=5, k=2, beta=0.0, inv_eps=1e4)}

for name in (sys.argv[1:] or ["config2", "config1"]) if __name__ == "__main__" else []:
    c = CFG[name]
    nf = c["base_n"] << (c["levels"] - 1)
    B = H.MGPreconditioner(base_n=c["base_n"], levels=c["levels"], k=c["k"], beta=c["beta"], inv_eps=c["inv_eps"],
                           cycle=H.CYCLE_V, structured_load=(nf, H.seeded_load(nf, 1)))
    L = H.lib()
    L.hpmg_profile_levels.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
    out = np.zeros(64)
    B.apply(np.ones(B.n))
    n = L.hpmg_profile_levels(B.h, 10, out.ctypes.data_as(C.POINTER(C.c_double)))
    lv = c["levels"] - 1
    rep = {"coarse": out[0]}
    for l in range(1, lv + 1):
        rep[f"L{l}_pre"] = out[2 * l]
        rep[f"L{l}_post"] = out[2 * l + 1]
    rep["head_pre"], rep["head_res"], rep["head_post"] = out[2 * (lv + 1):2 * (lv + 1) + 3]
    ms, _ = B.time_apply(20)
    rep["graph_ms_per_vcycle"] = ms
    rep["sum_parts"] = float(sum(v for k, v in rep.items() if k != "graph_ms_per_vcycle"))
    print(name, json.dumps({k: round(float(v), 4) for k, v in rep.items()}))
