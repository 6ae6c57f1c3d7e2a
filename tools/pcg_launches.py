"""Development: one short device PCG solve (3 iterations) inside a profiler
range, for `ncu --profile-from-start off` launch lists. usage: pcg_launches.py [config]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

B = H.MGPreconditioner(**R.device_kwargs(sys.argv[1] if len(sys.argv) > 1 else "config2"))
rhs = B.rhs()
H.pcg(B, rhs, opt=H.KrylovOptions(max_iterations=3))
torch.cuda.synchronize()
torch.cuda.profiler.start()
H.pcg(B, rhs, opt=H.KrylovOptions(max_iterations=3))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
