"""Full-size CPU reference runs for the parity tests (TEST INFRASTRUCTURE).

Each BASELINE configuration's reference solve takes 10 s to a few minutes on
one core, so the full-size tests submit all of them at once to a process
pool and compare against the device as each finishes. The checker is the
reference itself (oracle/_ref/libref.so) where it is built, else the
restatement (oracle/_build/liborc.so); GMRES(m) runs always use the
restatement (the reference's GMRES is unrestarted, krylov.hpp:79-84).
"""
from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os
import time

import numpy as np

import oracle_lib as O


def config_problem(name):
    """(problem kwargs for OracleMG / MGPreconditioner, seeded load grid n) of a
    named BASELINE configuration (BASELINE.json configs)."""
    if name == "config1":
        n = 128
        return dict(base_n=8, levels=5, k=1, nu=1.0, beta=1.0, inv_eps=1e3), n, (-1.0, 1.0), None
    if name == "config2":
        n = 256
        return dict(base_n=16, levels=5, k=3, nu=1.0, beta=1e-2, inv_eps=1e3), n, (-1.0, 1.0), None
    if name.startswith("config3"):  # config3_k{k}_al{inv_eps}_b{beta}
        _, kk, al, b = name.split("_")
        return (dict(base_n=8, levels=5, k=int(kk[1:]), nu=1.0, beta=float(b[1:]), inv_eps=float(al[2:])), 128,
                (-1.0, 1.0), None)
    if name.startswith("config5"):  # config5_re{Re}
        re = float(name.split("_")[1][2:])
        return (dict(base_n=8, levels=6, k=2, nu=1.0 / re, beta=0.0, inv_eps=1e3), 256, (-0.1, 0.1), "config5_wind")
    raise ValueError(name)


def oracle_kwargs(name, seed=1):
    kw, n, (lo, hi), wind = config_problem(name)
    kw = dict(kw, load_kind=O.LOAD_ARRAY, load=O.seeded_load(n, seed, lo, hi), cycle=O.CYCLE_V)
    if wind:
        kw.update(wind=O.WIND_CURL, bc=O.BC_LID_UNIT)
    return kw


def device_kwargs(name, seed=1):
    kw, n, (lo, hi), wind = config_problem(name)
    kw = dict(kw, structured_load=(n, O.seeded_load(n, seed, lo, hi)), cycle=0)
    if wind:
        kw.update(wind=wind, bc="lid_unit")
    return kw


def _run(name, use_reference, restart, seed):
    t0 = time.time()
    m = O.OracleMG(reference=use_reference, **oracle_kwargs(name, seed))
    t1 = time.time()
    if restart:
        m.set_restart(restart)
    u = m.uzawa()
    return dict(name=name, reference=bool(use_reference), restart=restart, inner=u["inner_iterations"],
                velocity=u["velocity"], pressure=u["pressure"], converged=u["converged"],
                setup_s=t1 - t0, solve_s=time.time() - t1)


HP_SOLVE = os.path.join(O.ORACLE_DIR, "_build", "hp_solve")


def _run_hp(name, seed):
    """The restatement in extended precision (oracle/hp_solve.cpp, Real =
    long double) on a homogeneous-Dirichlet Stokes config: the yardstick for
    how far a double-precision run of the algorithm lands from its
    exact-arithmetic result."""
    import subprocess
    import tempfile

    kw, n, _, wind = config_problem(name)
    assert wind is None
    t0 = time.time()
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        out = subprocess.run([HP_SOLVE, str(kw["base_n"]), str(kw["levels"]), str(kw["k"]), repr(kw["beta"]),
                              repr(kw["inv_eps"]), str(seed), f.name], capture_output=True, text=True, check=True)
        vel = np.fromfile(f.name)
    return dict(name=name, reference=False, restart="hp", inner=[int(v) for v in out.stdout.split()],
                velocity=vel, converged=True, setup_s=0.0, solve_s=time.time() - t0)


class RefPool:
    """Submits named runs at construction; result(name, ...) blocks on one."""

    def __init__(self, runs, workers=None):
        workers = workers or max(1, min(len(runs), (os.cpu_count() or 2) - 1))
        self.ex = cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"))
        self.fut = {}
        for name, restart in runs:  # restart: 0 unrestarted, m > 0 GMRES(m), "hp" extended precision
            if restart == "hp":
                self.fut[(name, restart)] = self.ex.submit(_run_hp, name, 1)
                continue
            use_ref = O.ref_available() and not restart
            self.fut[(name, restart)] = self.ex.submit(_run, name, use_ref, restart, 1)

    def result(self, name, restart=0, timeout=3600):
        return self.fut[(name, restart)].result(timeout=timeout)

    def close(self):
        self.ex.shutdown(wait=False, cancel_futures=True)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))
