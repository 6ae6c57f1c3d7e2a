"""Runs every BASELINE.json configuration the reference can express on the GPU
and (optionally) the CPU oracle, and prints one JSON line per run: DOFs,
setup time, per-Uzawa-step inner iteration counts, device solve time,
V-cycle time. Used to fill BASELINE.md's measurement table."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402


def runs():
    # config 1: 8x8 base + 4 refinements, k=1, AL 1e3, mass 1, nu 1, homogeneous Dirichlet
    yield dict(name="config1", base_n=8, levels=5, k=1, nu=1.0, beta=1.0, inv_eps=1e3)
    # config 2: 16x16 base, 5 GMG levels, k=3, AL 1e3, mass 1e-2
    yield dict(name="config2", base_n=16, levels=5, k=3, nu=1.0, beta=1e-2, inv_eps=1e3)
    # config 3: 128^2, k=2, AL in {1,1e2,1e4}, mass in {0,1e2} (k=4,6: no reference, k<=3)
    for al in (1.0, 1e2, 1e4):
        for beta in (0.0, 1e2):
            yield dict(name=f"config3_al{al:g}_m{beta:g}", base_n=8, levels=5, k=2, nu=1.0, beta=beta, inv_eps=al)
    # config 5: 8x8 base + 5 refinements (256^2), k=2, AL 1e3, nu = 1/Re, lid (1,0), curl wind, GMRES(50)
    for re in (1.0, 100.0, 1000.0):
        yield dict(name=f"config5_re{re:g}", base_n=8, levels=6, k=2, nu=1.0 / re, beta=0.0, inv_eps=1e3,
                   oseen=True, lo=-0.1, hi=0.1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--oracle", action="store_true", help="also run the CPU oracle (slow for config 2/5)")
    args = ap.parse_args()
    for r in runs():
        if args.only and not r["name"].startswith(args.only):
            continue
        n_f = r["base_n"] << (r["levels"] - 1)
        F = H.seeded_load(n_f, 1, r.get("lo", -1.0), r.get("hi", 1.0))
        oseen = r.get("oseen", False)
        t0 = time.perf_counter()
        B = H.MGPreconditioner(base_n=r["base_n"], levels=r["levels"], k=r["k"], nu=r["nu"], beta=r["beta"],
                               inv_eps=r["inv_eps"], cycle=H.CYCLE_V, structured_load=(n_f, F),
                               bc="lid_unit" if oseen else None, wind="config5_wind" if oseen else None)
        setup = time.perf_counter() - t0
        ms, _ = B.time_apply(10)
        kopt = H.KrylovOptions(restart=50) if oseen else H.KrylovOptions()
        t1 = time.perf_counter()
        sol = H.uzawa_solve(B, krylov=kopt)
        wall = time.perf_counter() - t1
        out = dict(config=r["name"], n=int(B.n), k=r["k"], setup_s=round(setup, 3), vcycle_ms=round(ms, 4),
                   inner_iterations=sol.report.inner_iterations, solve_device_s=round(sol.report.seconds, 4),
                   solve_wall_s=round(wall, 4), tts_s=round(setup + wall, 3), converged=sol.report.converged,
                   final_divergence=sol.report.final_divergence,
                   krylov="GMRES(50)" if oseen else "PCG")
        if args.oracle:
            import oracle_lib as O
            t2 = time.perf_counter()
            orc = O.OracleMG(base_n=r["base_n"], levels=r["levels"], k=r["k"], nu=r["nu"], beta=r["beta"],
                             inv_eps=r["inv_eps"], bc=O.BC_LID_UNIT if oseen else O.BC_NONE,
                             load_kind=O.LOAD_ARRAY, load=F, wind=O.WIND_CURL if oseen else O.WIND_NONE,
                             cycle=O.CYCLE_V)
            osetup = time.perf_counter() - t2
            ro = orc.uzawa()
            out.update(oracle_inner_iterations=ro["inner_iterations"], oracle_setup_s=round(osetup, 2),
                       oracle_solve_s=round(ro["seconds"], 2),
                       velocity_rel_diff=float(np.linalg.norm(sol.velocity - ro["velocity"]) /
                                               np.linalg.norm(ro["velocity"])))
        print(json.dumps(out), flush=True)
        B.close()


if __name__ == "__main__":
    main()
