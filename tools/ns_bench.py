"""Navier-Stokes driver time-to-solution (lid cavity, config-5 mesh family):
device driver vs the CPU oracle on a smaller mesh. Usage: ns_bench.py [levels] [k] [Re] [oracle_levels]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
re = float(sys.argv[3]) if len(sys.argv) > 3 else 100.0
olev = int(sys.argv[4]) if len(sys.argv) > 4 else 0
kw = dict(base_n=8, k=k, nu=1.0 / re, inv_eps=1e3)
t0 = time.perf_counter()
s = H.navier_stokes_solve(levels=levels, bc="lid_unit", cycle=H.CYCLE_V, **kw)
wall = time.perf_counter() - t0
r = s.report
out = {"device": {"mesh": f"{8 << (levels - 1)}^2 x 2", "k": k, "Re": re, "wall_s": wall, "driver_s": r.seconds,
                  "setup_s": r.setup_seconds, "picard": r.picard_iterations, "newton": r.newton_iterations,
                  "inner": r.picard_inner + r.newton_inner, "converged": r.converged}}
if olev:
    import oracle_lib as O
    t0 = time.perf_counter()
    ro = O.ns_solve(levels=olev, bc=O.BC_LID_UNIT, cycle=O.CYCLE_V, **kw)
    out["oracle"] = {"mesh": f"{8 << (olev - 1)}^2 x 2", "wall_s": time.perf_counter() - t0,
                     "picard": ro["picard_iterations"], "newton": ro["newton_iterations"],
                     "inner": ro["picard_inner"] + ro["newton_inner"], "converged": ro["converged"]}
print(json.dumps(out))
