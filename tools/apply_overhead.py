"""Development tool: hpmg_apply (device pointers) vs the bare V-cycle graph."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

B = H.MGPreconditioner(**R.device_kwargs(sys.argv[1] if len(sys.argv) > 1 else "config2"))
lib = H.lib()
s = torch.cuda.ExternalStream(B.stream())
r = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, B.n)).cuda()
z = torch.empty_like(r)


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"apply_dev_ms": t(lambda: lib.hpmg_apply(B.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                                                    H.DEVICE_PTRS)),
       "graph_ms": B.time_apply(50)[0]}
out["apply_dev_ms_2"] = t(lambda: lib.hpmg_apply(B.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                                                 H.DEVICE_PTRS))
out["graph_ms_2"] = B.time_apply(50)[0]
print(json.dumps(out))
