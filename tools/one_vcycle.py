"""Development: graph-launched V-cycles inside a profiler range (for
`ncu --profile-from-start off`): four drop-in hpmg_apply calls on device
buffers, i.e. the bench step (permutations + cycle). Usage: one_vcycle.py config2"""
import ctypes
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
r = torch.from_numpy(b).cuda()
z = torch.empty_like(r)
L = H.lib()


def step():
    L.hpmg_apply(B.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(z.data_ptr()), H.DEVICE_PTRS)


step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(4):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
