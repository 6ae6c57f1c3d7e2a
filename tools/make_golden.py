"""Writes tests/golden/*.npz: outputs of THE REFERENCE ITSELF (oracle/_ref/
libref.so = the unmodified /root/reference/proj/include/hdivmg headers over
the Eigen-API shim, oracle/Makefile target `ref`) on small seeded cases, so
that parity against the reference can be checked where the reference cannot
be built (the GPU box has no /root/reference). Run here, in the build
container: `python tools/make_golden.py` (needs `make -C oracle ref`).

Per case: the condensed operator (CSR, lowest and second-lowest orders
only: the k = 3 matrix is large), rhs, free_to_full, one preconditioner
application on a seeded vector, one Krylov solve of A x = rhs (PCG for
symmetric, GMRES for advected cases: iterations, solution) and a 2-step
AL-Uzawa solve (inner iterations, velocity, pressure).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# name -> (OracleMG kwargs without the load, load seed, load range, keep the CSR)
CASES = {
    "stokes_k0_v": (dict(base_n=4, levels=3, k=0, beta=1.0, inv_eps=1e3, cycle=O.CYCLE_V), 1, (-1, 1), True),
    "stokes_k1_v": (dict(base_n=4, levels=3, k=1, beta=1.0, inv_eps=1e3, cycle=O.CYCLE_V), 2, (-1, 1), True),
    "stokes_k2_w": (dict(base_n=4, levels=3, k=2, beta=1e-2, inv_eps=1e3, cycle=O.CYCLE_W), 3, (-1, 1), False),
    "stokes_k3_v": (dict(base_n=4, levels=3, k=3, beta=1e-2, inv_eps=1e3, cycle=O.CYCLE_V), 4, (-1, 1), False),
    "stokes_k1_additive": (dict(base_n=4, levels=3, k=1, beta=1.0, inv_eps=1e3, cycle=O.CYCLE_V,
                                smoother=O.SM_ADD, smooth_steps=2), 5, (-1, 1), False),
    "stokes_k2_al1e4_b0": (dict(base_n=4, levels=3, k=2, beta=0.0, inv_eps=1e4, cycle=O.CYCLE_V), 6, (-1, 1), False),
    "oseen_k2_nu1e-2": (dict(base_n=4, levels=3, k=2, nu=1e-2, beta=0.0, inv_eps=1e3, cycle=O.CYCLE_V,
                             bc=O.BC_LID_UNIT, wind=O.WIND_CURL), 7, (-0.1, 0.1), False),
}


def run(name, kw, seed, lohi, keep_csr):
    n_f = kw["base_n"] << (kw["levels"] - 1)
    F = O.seeded_load(n_f, seed, *lohi)
    ref = O.OracleMG(reference=True, load_kind=O.LOAD_ARRAY, load=F, **kw)
    out = dict(load=F, free_to_full=ref.free_to_full(), rhs=ref.rhs())
    b = O.random_vec(ref.n, seed + 100)
    out["apply_in"] = b
    out["apply_out"] = ref.apply(b)
    advected = kw.get("wind", O.WIND_NONE) != O.WIND_NONE
    x, st = ref.krylov(ref.rhs(), method=1 if advected else 0)
    out["krylov_x"] = x
    out["krylov_iterations"] = np.array(st["iterations"])
    uz = ref.uzawa()
    out["uzawa_velocity"] = uz["velocity"]
    out["uzawa_pressure"] = uz["pressure"]
    out["uzawa_inner"] = np.array(uz["inner_iterations"])
    if keep_csr:
        A = ref.csr().tocsr()
        out.update(A_data=A.data, A_indices=A.indices, A_indptr=A.indptr, A_shape=np.array(A.shape))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    meta = {k: (float(v) if isinstance(v, float) else v) for k, v in kw.items()}
    return dict(kwargs=meta, seed=seed, load_range=list(lohi), n=int(ref.n), krylov="gmres" if advected else "pcg",
                krylov_iterations=int(st["iterations"]), uzawa_inner=[int(i) for i in uz["inner_iterations"]])


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libref.so is not built: make -C oracle ref (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for name, (kw, seed, lohi, keep) in CASES.items():
        index[name] = run(name, kw, seed, lohi, keep)
        print(name, index[name]["n"], index[name]["krylov_iterations"], index[name]["uzawa_inner"], flush=True)
    index["_source"] = ("oracle/_ref/libref.so: the unmodified reference headers (proj/include/hdivmg) over "
                        "oracle/eigen_shim, driven by oracle/ref_capi.cpp; written by tools/make_golden.py")
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
