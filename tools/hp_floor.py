"""Reference vs restatement vs the extended-precision restatement
(oracle/_build/hp_solve, long double) on one configuration: Uzawa counts and
velocity distances. Shows how far the reference's own double-precision
result sits from the exact-arithmetic result of the same algorithm.

usage: python tools/hp_floor.py NAME [levels_override] [restart]
  NAME as in tests/ref_runs.py (config1, config2, config3_k2_al10000_b0,
  config5_re100, ...)
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
import ref_runs as R  # noqa: E402


def main():
    name = sys.argv[1]
    kw, n, (lo, hi), wind = R.config_problem(name)
    okw = R.oracle_kwargs(name)
    if len(sys.argv) > 2 and sys.argv[2] != "-":
        lv = int(sys.argv[2])
        kw["levels"] = okw["levels"] = lv
        n = kw["base_n"] << (lv - 1)
        okw["load"] = O.seeded_load(n, 1, lo, hi)
    restart = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = {"name": name, "levels": kw["levels"], "restart": restart}
    vel = {}
    for tag, which in (("reference", True), ("restatement", False)):
        if restart and which is True:
            continue
        m = O.OracleMG(reference=which, **okw)
        if restart:
            m.set_restart(restart)
        u = m.uzawa()
        vel[tag] = u["velocity"]
        out[tag + "_inner"] = u["inner_iterations"]
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        args = [R.HP_SOLVE, str(kw["base_n"]), str(kw["levels"]), str(kw["k"]), repr(kw["beta"]), repr(kw["inv_eps"]),
                "1", f.name, repr(kw["nu"]), repr(lo), repr(hi), "2" if wind else "0", "4" if wind else "0",
                str(restart)]
        r = subprocess.run(args, capture_output=True, text=True, check=True)
        vel["hp"] = np.fromfile(f.name)
        out["hp_inner"] = [int(v) for v in r.stdout.split()]
    for tag in vel:
        if tag != "hp":
            out[tag + "_vs_hp"] = R.rel(vel[tag], vel["hp"])
    if "reference" in vel:
        out["restatement_vs_reference"] = R.rel(vel["restatement"], vel["reference"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
