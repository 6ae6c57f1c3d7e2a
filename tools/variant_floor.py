"""Attributes device-vs-reference solution differences to arithmetic
formulations: runs the restatement with each ORC_VARIANT (explicit patch
inverses, explicit coarse inverse, pull sweeps; oracle/orc_mg.hpp) and the
FMA-free reference build, and reports Uzawa counts and the velocity distance
to the reference build (oracle/_ref/libref.so) on one config.

usage: python tools/variant_floor.py [k] [inv_eps] [beta] [levels] [base_n]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
import oracle_lib as O
k, inv_eps, beta, levels, base_n, which = %s
n = base_n << (levels - 1)
kw = dict(base_n=base_n, levels=levels, k=k, beta=beta, inv_eps=inv_eps, load_kind=O.LOAD_ARRAY,
          load=O.seeded_load(n, 1), cycle=O.CYCLE_V)
m = O.OracleMG(reference=(which if which else False), **kw)
u = m.uzawa()
np.save(sys.argv[1], u["velocity"])
print(json.dumps(u["inner_iterations"]))
'''


def run(args, which, variant, out):
    env = dict(os.environ, ORC_VARIANT=str(variant))
    code = CHILD % (os.path.join(ROOT, "tests"), repr(tuple(args) + (which,)))
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True, check=True)
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    import numpy as np
    a = sys.argv[1:]
    args = (int(a[0]) if a else 2, float(a[1]) if len(a) > 1 else 1e4, float(a[2]) if len(a) > 2 else 0.0,
            int(a[3]) if len(a) > 3 else 5, int(a[4]) if len(a) > 4 else 8)
    cases = [("reference", True, 0), ("reference_nofma", "nofma", 0), ("restatement", "", 0),
             ("patch_inverse", "", 1), ("coarse_inverse", "", 2), ("pull_sweeps", "", 4), ("all_three", "", 7)]
    vel = {}
    for name, which, var in cases:
        out = f"/tmp/vf_{name}.npy"
        its = run(args, which, var, out)
        vel[name] = np.load(out)
        d = np.linalg.norm(vel[name] - vel["reference"]) / np.linalg.norm(vel["reference"])
        print(json.dumps({"case": name, "inner": its, "vel_rel_vs_reference": d}), flush=True)


if __name__ == "__main__":
    main()
