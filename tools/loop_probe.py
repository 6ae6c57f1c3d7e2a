"""Development: cost of the device-loop structure (graph while / if nodes)
around the V-cycle, against the plain apply graph. usage: loop_probe.py [config]"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_06762_b200 as H  # noqa: E402
import ref_runs as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
B = H.MGPreconditioner(**R.device_kwargs(name))
L = H.lib()
L.hpmg_debug_loop_probe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
L.hpmg_debug_loop_probe.restype = ctypes.c_double
out = {"config": name, "graph_vcycle_ms": B.time_apply(30)[0]}
for mode, label in [(0, "empty_while_ms"), (1, "while_vcycle_ms"), (2, "while_if_vcycle_ms"),
                    (3, "while_child_vcycle_ms")]:
    out[label] = L.hpmg_debug_loop_probe(B.h, mode, 200 if mode == 0 else 30)
out["graph_vcycle_ms_2"] = B.time_apply(30)[0]
print(json.dumps({k: (round(v, 5) if isinstance(v, float) else v) for k, v in out.items()}))
if out["empty_while_ms"] < 0:
    L.hpmg_last_error.restype = ctypes.c_char_p
    print(L.hpmg_last_error())
