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
if B.symmetric():
    H.pcg(B, B.rhs(), opt=H.KrylovOptions(max_iterations=1))  # b into the solver's workspace
out = {"config": name, "graph_vcycle_ms": B.time_apply(30)[0]}
for mode, label in [(0, "empty_while_ms"), (1, "while_vcycle_ms"), (2, "while_if_vcycle_ms"),
                    (3, "while_child_vcycle_ms")]:
    out[label] = L.hpmg_debug_loop_probe(B.h, mode, 200 if mode == 0 else 30)
if B.symmetric():
    # PCG-shaped bodies (32 + bits: 1 spmv+pAp, 2 update, 4 if{V-cycle}, 8 rz, 16 direction)
    for mode, label in [(63, "pcg_full"), (62, "pcg_no_spmv"), (61, "pcg_no_update"), (59, "pcg_no_vcycle_if"),
                        (55, "pcg_no_rz"), (47, "pcg_no_direction"), (36, "pcg_if_vcycle_only")]:
        out[label] = L.hpmg_debug_loop_probe(B.h, mode, 25)
    # round-2 loop body (64: V-cycle directly in the body, then 8 r.z, 1 A p', 2 update)
    for mode, label in [(96 + 11, "pcg2_full"), (96, "pcg2_vcycle_only"), (96 + 8, "pcg2_v_rz"),
                        (96 + 9, "pcg2_v_rz_spmv"), (32 + 1, "spmv_dir_only"), (32 + 2, "update_only"),
                        (32 + 8, "rz_only")]:
        out[label] = L.hpmg_debug_loop_probe(B.h, mode, 25)
out["graph_vcycle_ms_2"] = B.time_apply(30)[0]
print(json.dumps({k: (round(v, 5) if isinstance(v, float) else v) for k, v in out.items()}))
if out["empty_while_ms"] < 0:
    L.hpmg_last_error.restype = ctypes.c_char_p
    print(L.hpmg_last_error())
