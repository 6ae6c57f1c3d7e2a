import os, sys
sys.path.insert(0, os.getcwd())
import paper_2303_06762_b200 as H
B = H.MGPreconditioner(base_n=16, levels=5, k=3, beta=1e-2, inv_eps=1e3, cycle=H.CYCLE_V, structured_load=(256, H.seeded_load(256, 1)))
print("ok", B.n)
