"""V-cycle time back to back vs with an L2 flush (256 MB write) before each
one (events around the V-cycle only). usage: python tools/vcycle_flush.py [config]"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
B = H.MGPreconditioner(**R.device_kwargs(name))
L = H.lib()
st = torch.cuda.ExternalStream(B.stream())
r = torch.rand(B.n, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def vc():
    L.hpmg_apply(B.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(z.data_ptr()), H.DEVICE_PTRS)


out = {}
for mode in ("back_to_back", "flushed"):
    ts = []
    for i in range(25):
        with torch.cuda.stream(st):
            if mode == "flushed":
                flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            vc()
            e1.record(st)
        e1.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    out[mode] = round(float(np.median(ts)), 4)
print(json.dumps({"config": name, **out}))
