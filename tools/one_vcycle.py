"""Development: one graph-launched V-cycle inside a profiler range (for
`ncu --profile-from-start off`). Usage: one_vcycle.py config2"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_06762_b200 as H  # noqa: E402
from profile_levels import CFG  # noqa: E402

c = CFG[sys.argv[1] if len(sys.argv) > 1 else "config2"]
nf = c["base_n"] << (c["levels"] - 1)
B = H.MGPreconditioner(base_n=c["base_n"], levels=c["levels"], k=c["k"], beta=c["beta"], inv_eps=c["inv_eps"],
                       cycle=H.CYCLE_V, structured_load=(nf, H.seeded_load(nf, 1)))
b = np.ones(B.n)
B.apply(b)
B.apply(b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
B.time_apply(1)
torch.cuda.profiler.stop()
