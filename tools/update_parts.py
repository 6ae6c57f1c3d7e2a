"""Development: time split of hpmg_update (re-linearisation) at config-5 size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_06762_b200 as H  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = H.MGPreconditioner(base_n=8, levels=levels, k=k, nu=1e-2, inv_eps=1e3, bc="lid_unit", wind="config5_wind",
                       cycle=H.CYCLE_V)
w = B.interpolate("rotation")
names = ["-", "condense+assemble", "patch inverses", "transfers", "coarse", "-", "total"]
for rep in range(3):
    t0 = time.perf_counter()
    B.update(wind=w, newton=True)
    wall = time.perf_counter() - t0
    tot, parts = B.setup_seconds()
    print("update wall %.3f |" % wall, " ".join("%s %.3f" % (n, p) for n, p in zip(names, parts[:7]) if n != "-"))
