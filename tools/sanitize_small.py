"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): setup, V-cycles (k = 0..3; the wave sweeps, the one-CTA
small-level kernel, transfers, coarse solve), device PCG and GMRES graph
loops, Uzawa, recovery, on 4x4-base meshes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_06762_b200 as H  # noqa: E402

for k in (0, 1, 2, 3):
    n_f = 4 << 2
    B = H.MGPreconditioner(base_n=4, levels=3, k=k, beta=1.0, inv_eps=1e3, cycle=H.CYCLE_V,
                           structured_load=(n_f, H.seeded_load(n_f, 1)))
    b = np.random.default_rng(k).uniform(-1, 1, B.n)
    z = B.apply(b)
    x, st = H.pcg(B, B.rhs())
    sol = H.uzawa_solve(B)
    B.recover(sol.velocity)
    print("k", k, "pcg", st.iterations, "uzawa", sol.report.inner_iterations, flush=True)
# level 1 on 26 waves: the one-CTA small-level kernel (8x8 base)
B = H.MGPreconditioner(base_n=8, levels=3, k=1, beta=1.0, inv_eps=1e3, cycle=H.CYCLE_V,
                       structured_load=(32, H.seeded_load(32, 1)))
B.apply(np.ones(B.n))
# advected: record sweeps for A and A^T, GMRES graph loop
B = H.MGPreconditioner(base_n=4, levels=3, k=2, nu=1e-2, inv_eps=1e3, cycle=H.CYCLE_V, bc="lid_unit",
                       wind="config5_wind", structured_load=(16, H.seeded_load(16, 1, -0.1, 0.1)))
x, st = H.gmres(B, B.rhs(), opt=H.KrylovOptions(restart=10))
print("gmres(10)", st.iterations, st.converged, flush=True)
print("sanitize_small: done")
