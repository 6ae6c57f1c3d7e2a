"""Development: setup-time split (mesh+tables, condensation+assembly, patch inverses,
transfers, coarse inverse, workspace+graph, total), twice per process."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--torch" in sys.argv:
    import torch
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
import paper_2303_06762_b200 as H  # noqa: E402

keep = []
for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    B = H.MGPreconditioner(base_n=16, levels=5, k=3, beta=1e-2, inv_eps=1e3, cycle=H.CYCLE_V,
                           structured_load=(256, H.seeded_load(256, 1)))
    wall = time.perf_counter() - t0
    tot, parts = B.setup_seconds()
    print("rep", rep, "wall %.3f" % wall, " ".join("%.3f" % p for p in parts[:7]))
    if "--keep" in sys.argv:
        keep.append(B)  # as bench.py: the next context is built while this one lives
    else:
        del B
