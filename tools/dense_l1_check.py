"""A/B of the dense level-1 sub-cycle (HPMG_DENSE_L1) on one GPU.

For each config: V-cycle output with the one-CTA level-1 sweeps vs the dense
map (relative difference), PCG / Uzawa iteration counts and velocity with
both, warm setup wall time of each, and the V-cycle graph time (CUDA events
through hpmg_apply on device buffers is what bench.py measures; here the
drop-in apply on host buffers, best of 20, for a relative figure only).
Prints one JSON line per config.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_06762_b200 as H  # noqa: E402

CONFIGS = {
    "config2": dict(base_n=16, levels=5, k=3, nu=1.0, beta=1e-2, inv_eps=1e3),
    "config1": dict(base_n=8, levels=5, k=1, nu=1.0, beta=1.0, inv_eps=1e3),
    "config3": dict(base_n=8, levels=5, k=2, nu=1.0, beta=0.0, inv_eps=1e4),
}


def make(cfg, dense):
    os.environ["HPMG_DENSE_L1"] = "1" if dense else "0"
    n_f = cfg["base_n"] << (cfg["levels"] - 1)
    F = H.seeded_load(n_f, 1)
    t0 = time.perf_counter()
    B = H.MGPreconditioner(mesh="unit_square", base_n=cfg["base_n"], levels=cfg["levels"], k=cfg["k"],
                           nu=cfg["nu"], beta=cfg["beta"], inv_eps=cfg["inv_eps"], cycle=H.CYCLE_V,
                           smoother=H.SMOOTH_MULTIPLICATIVE, smooth_steps=1, structured_load=(n_f, F))
    return B, time.perf_counter() - t0


def main():
    names = sys.argv[1:] or list(CONFIGS)
    for name in names:
        cfg = CONFIGS[name]
        out = {"config": name}
        res = {}
        for dense in (False, True, False, True):
            B, setup = make(cfg, dense)
            rng = np.random.default_rng(3)
            b = rng.standard_normal(B.n)
            z = B.apply(b)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                B.apply(b)
                ts.append(time.perf_counter() - t0)
            x, st = H.pcg(B, B.rhs())
            u = H.uzawa_solve(B)
            res[dense] = dict(z=z, x=x, its=st.iterations, setup=setup, apply_ms=1e3 * min(ts), u=u)
            B.close()
        a, d = res[False], res[True]
        out["vcycle_rel_diff"] = float(np.linalg.norm(a["z"] - d["z"]) / np.linalg.norm(a["z"]))
        out["pcg_its"] = [a["its"], d["its"]]
        out["pcg_x_rel_diff"] = float(np.linalg.norm(a["x"] - d["x"]) / np.linalg.norm(a["x"]))
        ua, ud = a["u"], d["u"]
        out["uzawa_inner"] = [ua.report.inner_iterations, ud.report.inner_iterations]
        out["uzawa_u_rel_diff"] = float(np.linalg.norm(ua.velocity - ud.velocity) / np.linalg.norm(ua.velocity))
        out["setup_s"] = [a["setup"], d["setup"]]
        out["apply_host_ms"] = [a["apply_ms"], d["apply_ms"]]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
