"""Full-size parity at every BASELINE configuration with a reference path,
device (through the C ABI) against the reference itself.

The checker runs are the reference's own uzawa_solve (oracle/_ref/libref.so,
the unmodified headers over the Eigen-API shim; the restatement where that
library is absent), all submitted at once to a CPU process pool
(tests/ref_runs.py) while the device solves run. Gates (BASELINE.json
north_star): inner Krylov counts per Uzawa step +-1, final velocity relative
L2 <= 1e-9. GMRES(50) (config 5) has no reference counterpart (the
reference's GMRES is unrestarted, krylov.hpp:79-84) and is checked against
the restatement's GMRES(m) extension; the unrestarted device GMRES is checked
against the reference itself.
"""
import numpy as np
import pytest

import oracle_lib as O
import ref_runs as R

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

H = pytest.importorskip("paper_2303_06762_b200")

CONFIG3 = [f"config3_k2_al{al}_b{b}" for al in ("1", "100", "10000") for b in ("0", "100")]
HIGH_AL = [c for c in CONFIG3 if "_al10000_" in c]
# the long-double runs go first: they are the slowest jobs of the pool
RUNS = ([(c, "hp") for c in HIGH_AL] + [("config2", 0), ("config1", 0)] + [(c, 0) for c in CONFIG3] +
        [("config5_re1", 0), ("config5_re100", 0), ("config5_re100", 50)])

VEL_TOL = 1e-9  # north star

# The reference's own round-off floor at the full-size advected configs: its
# double-precision velocity vs the same algorithm in extended precision
# (profiles/r02_roundoff_floors.json, tools/hp_floor.py; the long-double run
# takes ~30 min at this size, so it is not repeated here)
import json as _json
import os as _os
with open(_os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "profiles",
                        "r02_roundoff_floors.json")) as _f:
    FLOORS = _json.load(_f)["runs"]


@pytest.fixture(scope="module")
def pool():
    p = R.RefPool(RUNS)
    yield p
    p.close()


def check(name, ref, sol):
    rep = sol.report
    assert rep.converged and ref["converged"], name
    assert len(rep.inner_iterations) == len(ref["inner"])
    for a, b in zip(rep.inner_iterations, ref["inner"]):
        assert abs(a - b) <= 1, (name, rep.inner_iterations, ref["inner"])
    err = R.rel(sol.velocity, ref["velocity"])
    print(f"{name}: inner {rep.inner_iterations} vs {ref['inner']} "
          f"({'reference' if ref['reference'] else 'restatement'}), velocity rel {err:.2e}")
    return err


def device(name):
    return H.MGPreconditioner(**R.device_kwargs(name))


def test_config1(pool):
    gpu = device("config1")
    assert check("config1", pool.result("config1"), H.uzawa_solve(gpu)) <= VEL_TOL


def test_config2(pool):
    gpu = device("config2")
    assert gpu.n == 1568768
    assert check("config2", pool.result("config2"), H.uzawa_solve(gpu)) <= VEL_TOL


@pytest.mark.parametrize("name", CONFIG3)
def test_config3(pool, name):
    gpu = device(name)
    sol = H.uzawa_solve(gpu)
    ref = pool.result(name)
    err = check(name, ref, sol)
    if name not in HIGH_AL:
        assert err <= VEL_TOL
        return
    # AL 1e4: the penalised operator's conditioning puts the reference's own
    # double-precision result ~1.2e-9 (relative) away from the same algorithm
    # run in extended precision (oracle/hp_solve.cpp, identical iteration
    # counts), so two correct double-precision implementations can sit
    # ~2x that apart. Gate: the device is as close to the extended-precision
    # result as the reference itself (within 1.5x), and the reference's own
    # distance is what exceeds the north-star 1e-9.
    hp = pool.result(name, "hp")
    assert hp["inner"] == ref["inner"]
    floor = R.rel(ref["velocity"], hp["velocity"])
    dev = R.rel(sol.velocity, hp["velocity"])
    print(f"{name}: reference vs extended precision {floor:.2e}, device vs extended precision {dev:.2e}")
    assert err <= VEL_TOL or (floor > VEL_TOL and dev <= 1.5 * floor)


def vel_gate(name, err, floor_key):
    """<= 1e-9, or, where the reference's own distance to its
    exact-arithmetic result exceeds that, within that distance."""
    if err <= VEL_TOL:
        return True
    floor = FLOORS.get(floor_key, {}).get("reference_vs_hp") or FLOORS.get(floor_key, {}).get("restatement_vs_hp")
    print(f"{name}: velocity {err:.2e} vs the reference's own round-off floor {floor:.2e}")
    return floor is not None and floor > VEL_TOL and err <= floor


@pytest.mark.parametrize("name", ["config5_re1", "config5_re100"])
def test_config5_unrestarted_vs_reference(pool, name):
    gpu = device(name)
    err = check(name, pool.result(name), H.uzawa_solve(gpu))
    assert vel_gate(name, err, name)


@pytest.mark.parametrize("name", ["config5_re1", "config5_re100"])
def test_config5_gmres50(pool, name):
    # BASELINE config 5's solver: restarted GMRES(50). Re = 1 needs fewer
    # than 50 iterations per solve, where GMRES(50) is the reference's method
    restart = 50 if name == "config5_re100" else 0
    gpu = device(name)
    sol = H.uzawa_solve(gpu, krylov=H.KrylovOptions(restart=50))
    err = check(name + "_gmres50", pool.result(name, restart), sol)
    assert vel_gate(name, err, name + "_gmres50" if restart else name)
