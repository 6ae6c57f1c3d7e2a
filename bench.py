#!/usr/bin/env python
"""hp-MG V-cycle benchmark on B200 (BASELINE.json metric, config 2 by default).

Workload (BASELINE configs[1]): 2-D generalized Stokes, unit square, 16x16
base mesh + 4 red refinements (256^2 x 2 = 131,072 triangles, 5 GMG levels),
order k = 3 (n = 1,568,768 free DOFs), AL parameter 1e3, mass 1e-2, nu 1,
homogeneous Dirichlet, seeded per-triangle force U[-1,1] (mt19937 seed 1),
V(1,1) multiplicative vertex-patch smoothing, PCG to 1e-8.

One step = one hp-MG V-cycle (MGPreconditioner::apply) on an HBM-resident
residual. `value` = V-cycles/s over all ranks (replicas, one per GPU);
`e2e` = the same through the drop-in C-ABI call hpmg_apply (the
MGPreconditioner::apply equivalent) with pinned host buffers: H2D residual +
V-cycle + D2H correction inside the timed region, one call per step
(`e2e.batch_value`: the pipelined hpmg_apply_batch over independent
vectors). The V-cycle streams ~3 GB per call, far above the 126 MB L2, so no
explicit flush is needed.

--impl reference times the reference's own CPU implementation: its
unmodified headers compiled against the Eigen-API shim
(oracle/_ref/libref.so, built in the build container where the reference
tree exists; single-threaded like the reference), the restatement
(oracle/_build/liborc.so) where that library is absent. Rank 0 also times the
reference's time-to-solution (MGPreconditioner construction + uzawa_solve +
recover_locals) at the bench config in a pinned child process while the
device is measured (`tts.cpu_reference`).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CONFIGS = {
    # name: (base_n, levels, k, nu, beta, inv_eps)
    "config2": dict(base_n=16, levels=5, k=3, nu=1.0, beta=1e-2, inv_eps=1e3),
    "config1": dict(base_n=8, levels=5, k=1, nu=1.0, beta=1.0, inv_eps=1e3),
    "config3": dict(base_n=8, levels=5, k=2, nu=1.0, beta=0.0, inv_eps=1e4),
    # the robustness sweep's orders beyond the reference's k <= 3 (parity unpinned)
    "config3_k4": dict(base_n=8, levels=5, k=4, nu=1.0, beta=0.0, inv_eps=1e4),
    "config3_k6": dict(base_n=8, levels=5, k=6, nu=1.0, beta=0.0, inv_eps=1e4),
}
METRIC = "hp-MG V-cycles/sec (k=3, 256^2x2 tri, 1.57M DOFs)"
# both arms print the same config dict; an L2 flush between V-cycles measures
# the same as back-to-back (tools/vcycle_flush.py)
L2_NOTE = "no flush needed: one V-cycle moves ~3 GB (config 2) through the 126 MB L2"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_init():
    """One process per GPU under torchrun: NCCL when CUDA is visible (the
    plumbing for the barrier and the max-over-ranks), gloo otherwise (CPU
    tests). Replicas only: no collective touches the data path."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        return rank, world, local, dist
    return 0, 1, 0, None


def max_over_ranks(ms, dist, device="cpu"):
    """Device-timed milliseconds of this rank -> the max over all ranks."""
    if dist is None:
        return ms
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank, ms_max, world):
    """Weak scaling: every rank processes the same units; the job rate is the
    total over ranks divided by the slowest rank's time."""
    return units_per_rank * world / (ms_max * 1e-3)


def run_hpmg(args, rank, world, local, dist):
    import torch  # device selection / external-stream events (plumbing only)
    import paper_2303_06762_b200 as H

    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    n_f = cfg["base_n"] << (cfg["levels"] - 1)
    F = H.seeded_load(n_f, args.seed)
    t0 = time.perf_counter()
    B = H.MGPreconditioner(mesh="unit_square", base_n=cfg["base_n"], levels=cfg["levels"], k=cfg["k"],
                           nu=cfg["nu"], beta=cfg["beta"], inv_eps=cfg["inv_eps"], cycle=H.CYCLE_V,
                           smoother=H.SMOOTH_MULTIPLICATIVE, smooth_steps=1, structured_load=(n_f, F))
    setup_wall = time.perf_counter() - t0
    setup_dev, setup_parts = B.setup_seconds()
    # time-to-solution first, on further contexts (the first one in a process
    # also pays the one-time CUDA module loading), before the CPU reference's
    # TTS child starts loading the host; three runs (build, solve, recover,
    # close), the median reported: a context built while another lives maps
    # fresh pool memory, which now and then stalls for 0.1-0.4 s
    tts_runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        B2 = H.MGPreconditioner(mesh="unit_square", base_n=cfg["base_n"], levels=cfg["levels"], k=cfg["k"],
                                nu=cfg["nu"], beta=cfg["beta"], inv_eps=cfg["inv_eps"], cycle=H.CYCLE_V,
                                smoother=H.SMOOTH_MULTIPLICATIVE, smooth_steps=1, structured_load=(n_f, F))
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        sol2 = H.uzawa_solve(B2)
        t_solve = time.perf_counter() - t0
        t0 = time.perf_counter()
        B2.recover(sol2.velocity)  # recover_locals, as the CPU reference TTS includes it
        t_recover = time.perf_counter() - t0
        _, parts2 = B2.setup_seconds()
        B2.close()
        tts_runs.append((t_setup + t_solve + t_recover, t_setup, t_solve, t_recover, parts2))
    tts_runs_sorted = sorted(tts_runs, key=lambda r: r[0])
    _, setup_warm, solve_wall, recover_wall, setup_parts_warm = tts_runs_sorted[1]
    # Krylov loop cost per iteration (wall-clock slopes: measured before the
    # CPU reference child loads the host)
    krylov = None
    if args.krylov and args.config == "config2":
        # PCG on this context; GMRES(50) on BASELINE config 5 (Re = 1)
        krylov = {"pcg_config2": krylov_overhead(H, B)}
        B5 = H.MGPreconditioner(base_n=8, levels=6, k=2, nu=1.0, beta=0.0, inv_eps=1e3, cycle=H.CYCLE_V,
                                bc="lid_unit", wind="config5_wind",
                                structured_load=(256, H.seeded_load(256, args.seed, -0.1, 0.1)))
        krylov["gmres50_config5_re1"] = krylov_overhead(H, B5, restart=50)
        krylov["note"] = ("whole solve = one CUDA-graph launch (device conditional nodes); overhead = per-iteration "
                          "cost minus the V-cycle and the operator apply it contains (vector updates, reductions, "
                          "for GMRES the fused MGS step kernels, at j from 5 to 25); slope of capped solves, "
                          "PCG 5..45 and GMRES 5..25 iterations, best of 5 runs each, CUDA events on the "
                          "library stream")
        B5.close()
    tts_proc = start_cpu_tts(args) if (args.cpu_tts and rank == 0 and world == 1) else None

    n = B.n
    lib = H.lib()
    stream = torch.cuda.ExternalStream(B.stream())
    rng = np.random.default_rng(1234 + rank)
    r_host = torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory()
    z_host = torch.empty(n, dtype=torch.float64).pin_memory()
    r_dev = r_host.to(f"cuda:{local}")
    z_dev = torch.empty_like(r_dev)

    def step_dev():
        lib.hpmg_apply(B.h, ctypes.c_void_p(r_dev.data_ptr()), ctypes.c_void_p(z_dev.data_ptr()), H.DEVICE_PTRS)

    def step_e2e():
        lib.hpmg_apply(B.h, ctypes.c_void_p(r_host.data_ptr()), ctypes.c_void_p(z_host.data_ptr()), 0)

    # pipelined e2e: the same K applies of host vectors through hpmg_apply_batch
    # (H2D of vector i+1 and D2H of result i-1 overlap V-cycle i); two pinned
    # input/output pairs rotate
    r_host2 = torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory()
    z_host2 = torch.empty(n, dtype=torch.float64).pin_memory()
    L_batch = lib.hpmg_apply_batch
    L_batch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                        ctypes.POINTER(ctypes.c_void_p)]

    def batch_call(m):
        rp = (ctypes.c_void_p * m)(*[(r_host if i % 2 == 0 else r_host2).data_ptr() for i in range(m)])
        zp = (ctypes.c_void_p * m)(*[(z_host if i % 2 == 0 else z_host2).data_ptr() for i in range(m)])
        return lambda: L_batch(B.h, m, rp, zp)

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        return max_over_ranks(ms, dist, f"cuda:{local}" if dist and dist.get_backend() == "nccl" else "cpu")

    def timed_once(fn):
        # fn runs K steps itself; warm-up = the same call, W times
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1), dist,
                              f"cuda:{local}" if dist and dist.get_backend() == "nccl" else "cpu")

    with ClockSampler(local) as clk:
        ms_dev = timed(step_dev, args.steps)
    ms_e2e_serial = timed(step_e2e, max(3, args.steps // 2))
    k_e2e = max(3, args.steps // 2)
    batch = batch_call(k_e2e)
    ms_e2e = timed_once(batch)
    # per-phase split, each phase its own graph: head pre-sweep, head residual, h-cycle + embedding, head post-sweep
    _, phases = B.time_apply(max(3, args.steps // 4), phases=True)
    vbytes, vparts = B.vcycle_bytes()
    # physical bytes: streamed sweep records (head p6, levels p7), head mode-0
    # residual p1, level residuals p3, transfers p4, coarse inverse p5, plus the
    # head's x/b/ z vectors at the cycle boundary (b read twice, x written)
    phys_bytes = float(vparts[6] + vparts[7] + vparts[1] + vparts[3] + vparts[4] + vparts[5] + 3 * 8.0 * n)
    hbm, src = peaks()
    head_sweep_ms = phases[0] + phases[3]
    head_bytes = vparts[6]  # bytes the head sweeps stream (records + vector rows)
    achieved = head_bytes / (head_sweep_ms * 1e-3) / 1e9 if head_sweep_ms > 0 else None
    ref_equiv = vparts[0] / (head_sweep_ms * 1e-3) / 1e9 if head_sweep_ms > 0 else None
    # DRAM traffic of the head sweeps from the committed ncu --set full capture
    # (bytes per patch, cold cache) scaled to this V-cycle's patch visits
    traffic = None
    try:
        prof = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                           "r02_final_head_sweep_ncu.json")))
        if args.config == "config2":
            traffic = prof["dram_bytes_per_patch"] * 2 * B.level_patches(-1)
    except (OSError, KeyError, ValueError):
        pass
    # operator apply (finest condensed operator, k_spmv) against the same peak
    ms_spmv, spmv_bytes, spmv_ref_bytes = B.time_spmv(max(10, args.steps))
    # time-to-solution: device Uzawa (2 outer PCG solves to 1e-8); the setup is
    # timed again on a second context (the first one in a process also pays
    # the one-time CUDA module loading)
    sol = H.uzawa_solve(B)
    launches = B.launches_per_apply()
    out = None
    if rank == 0:
        out = {
            "metric": METRIC if args.config == "config2" else f"hp-MG V-cycles/sec ({args.config})",
            "value": whole_job_rate(args.steps, ms_dev, world),
            "unit": "V-cycles/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_dev / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: seeded per-triangle U[-1,1] force (mt19937 seed %d), random-init residual" % args.seed,
            "config": {**workload_config(args, cfg, n), "parallelism": f"replicas x{world}",
                       "l2": L2_NOTE},
            "e2e": {"value": whole_job_rate(k_e2e, ms_e2e_serial, world), "unit": "V-cycles/s",
                    "h2d_bytes_per_step": int(8 * n), "d2h_bytes_per_step": int(8 * n),
                    "api": "hpmg_apply (drop-in MGPreconditioner::apply): H2D of the residual, V-cycle, "
                           "D2H of the correction, one call per step",
                    "batch_value": whole_job_rate(k_e2e, ms_e2e, world),
                    "batch_api": "hpmg_apply_batch over %d independent pinned host vectors (copies of "
                                 "neighbouring vectors overlap the V-cycles)" % k_e2e},
            "roofline": {"bound": "hbm",
                         "kernel": "k_sweep<8,128,1,waves> (order-k head patch sweeps, TMA patch records)",
                         "bytes_note": "achieved = bytes the head sweeps must stream in this formulation "
                                       "(per patch: packed symmetric inverse, the <=2 external A blocks per facet, "
                                       "meta; b/x rows and x_e gathers) / measured head-sweep time. "
                                       "reference_storage_equiv_gbs uses SURVEY 8(d)'s reference bytes "
                                       "(full np^2 factors, A rows read twice) over the same time.",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                         "traffic_note": "bytes per V-cycle over the head sweeps: ncu dram read+write per "
                                         "patch (profiles/r02_final_head_sweep_ncu.json) x 2 sweeps x patches",
                         "peak_source": src, "algorithmic_bytes_per_vcycle": vbytes,
                         "head_sweep_bytes_per_vcycle": head_bytes, "head_sweep_ms": head_sweep_ms,
                         "reference_storage_head_bytes_per_vcycle": vparts[0],
                         "reference_storage_equiv_gbs": ref_equiv,
                         "vcycle_reference_storage_effective_gbs": vbytes / (ms_dev / args.steps * 1e-3) / 1e9,
                         "vcycle_physical_bytes": phys_bytes,
                         "vcycle_physical_gbs": phys_bytes / (ms_dev / args.steps * 1e-3) / 1e9,
                         "vcycle_physical_frac": phys_bytes / (ms_dev / args.steps * 1e-3) / 1e9 / hbm,
                         "vcycle_physical_note": "(level 1 counted as its sweeps, transfers and coarse solve; with the default dense level-1 map the device instead reads the ~146 MB symmetric map per cycle, so the bytes moved are ~0.14 GB higher and this fraction is a lower bound) bytes this implementation moves per V-cycle: head and level "
                                                 "sweep records + vector rows as streamed, head mode-0 residual, "
                                                 "level residuals, P / P^T, coarse inverse, E/E^T and the "
                                                 "boundary vectors; the reference-storage figure above uses "
                                                 "SURVEY 8(d)'s accounting (full LU factors, A rows twice)"},
            "phases_ms": {"head_pre": phases[0], "head_residual": phases[1], "h_cycle": phases[2],
                          "head_post": phases[3]},
            "gpu_launches": int(launches * args.steps),
            "kernels_per_vcycle": int(launches),
            "krylov": krylov,
            "operator_apply": {"kernel": "k_spmv<bs> (ELL-BSR, 5 slots per facet block row)",
                               "ms": ms_spmv, "bytes": spmv_bytes,
                               "achieved": spmv_bytes / (ms_spmv * 1e-3) / 1e9 if ms_spmv > 0 else None,
                               "peak": hbm, "unit": "GB/s",
                               "frac": spmv_bytes / (ms_spmv * 1e-3) / 1e9 / hbm if ms_spmv > 0 else None,
                               "reference_storage_bytes": spmv_ref_bytes},
            "tts": {"uzawa_device_s": sol.report.seconds, "setup_wall_s": setup_wall,
                    "setup_wall_warm_s": setup_warm, "uzawa_wall_s": solve_wall,
                    "recover_wall_s": recover_wall,
                    "tts_warm_s": setup_warm + solve_wall + recover_wall,
                    "tts_warm_runs_s": [r[0] for r in tts_runs],
                    "tts_note": "tts_warm_s = median of three runs (tts_warm_runs_s) of setup (a further "
                                "context in the process) + AL-Uzawa wall time "
                                "(2 outer PCG solves to 1e-8, velocity and pressure back on the host) + "
                                "recover_locals (interior, pressure modes, gradient back on the host); "
                                "cpu_reference times the same three phases of the reference itself",
                    "setup_parts_s": [float(x) for x in setup_parts[:7]],
                    "setup_parts_warm_s": [float(x) for x in setup_parts_warm[:7]],
                    "setup_parts_note": "mesh+tables, plans+condensation, patch inverses, transfers, coarse "
                                        "inverse, workspace+graph, total (first context / second context)",
                    "inner_iterations": sol.report.inner_iterations,
                    "final_divergence": sol.report.final_divergence, "converged": sol.report.converged},
            "clocks": clk.summary(),
        }
        if args.cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_baseline(args, cfg, n_f, F, sample_vcycles=args.cpu_vcycles)
        if tts_proc is not None:
            cpu = finish_cpu_tts(tts_proc, timeout=900)
            out["tts"]["cpu_reference"] = cpu
            if "tts_s" in cpu:
                out["tts"]["gpu_vs_cpu_reference_speedup"] = cpu["tts_s"] / (setup_warm + solve_wall + recover_wall)
    return out


def host_info():
    """Host CPU model and usable core count (the CPU baseline's hardware)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": len(os.sched_getaffinity(0))}


def cpu_lib():
    """(OracleMG constructor kwargs flag, kind): the reference itself where
    oracle/_ref/libref.so was built, else the restatement."""
    import oracle_lib as O
    if O.ref_available():
        return True, "reference"
    return False, "port"


def cpu_problem(cfg, F):
    import oracle_lib as O
    return dict(base_n=cfg["base_n"], levels=cfg["levels"], k=cfg["k"], nu=cfg["nu"], beta=cfg["beta"],
                inv_eps=cfg["inv_eps"], bc=O.BC_NONE, load_kind=O.LOAD_ARRAY, load=F, cycle=O.CYCLE_V,
                smooth_steps=1)


def cpu_baseline(args, cfg, n_f, F, sample_vcycles=3):
    """The reference (or its restatement), 1 thread, on the same config."""
    import oracle_lib as O
    use_ref, kind = cpu_lib()
    t0 = time.perf_counter()
    B = O.OracleMG(reference=use_ref, **cpu_problem(cfg, F))
    setup = time.perf_counter() - t0
    secs = B.time_apply(sample_vcycles)
    lib = "oracle/_ref/libref.so (unmodified reference headers + Eigen-API shim)" if use_ref else "oracle/ restatement"
    return {"value": sample_vcycles / secs, "unit": "V-cycles/s", "cores": 1, "kind": kind,
            "sample": f"{sample_vcycles} V-cycles of {args.config} after a {setup:.1f} s setup ({lib}, 1 thread)",
            "setup_s": setup, **host_info()}


def cpu_tts_child(config, seed):
    """Reference time-to-solution at `config` (runs in a child pinned to one
    core): MGPreconditioner construction, uzawa_solve (2 outer PCG solves to
    1e-8), recover_locals; prints one JSON line."""
    import ctypes as C
    import oracle_lib as O
    cfg = CONFIGS[config]
    n_f = cfg["base_n"] << (cfg["levels"] - 1)
    F = O.seeded_load(n_f, seed)
    use_ref, kind = cpu_lib()
    kw = cpu_problem(cfg, F)
    if use_ref:
        L = O.ref_lib()
        load = np.ascontiguousarray(kw["load"])
        p = O.Problem(0, kw["base_n"], kw["levels"], kw["k"], kw["nu"], kw["beta"], 0.0, kw["inv_eps"], kw["bc"],
                      kw["load_kind"], load.ctypes.data_as(C.POINTER(C.c_double)), 0, kw["cycle"], 0, 1, 1.0 / 3.0,
                      0, 0)
        inner = (C.c_int * 8)()
        secs = np.zeros(3)
        t0 = time.perf_counter()
        done = L.orc_tts(C.byref(p), 2, 1e-8, inner, secs.ctypes.data_as(C.POINTER(C.c_double)))
        wall = time.perf_counter() - t0
        out = {"kind": kind, "setup_s": float(secs[0]), "uzawa_s": float(secs[1]), "recover_s": float(secs[2]),
               "tts_s": float(secs.sum()), "wall_s": wall, "inner_iterations": list(inner)[:max(done, 0)]}
    else:
        t0 = time.perf_counter()
        B = O.OracleMG(**kw)
        t1 = time.perf_counter()
        u = B.uzawa()
        t2 = time.perf_counter()
        B.recover(u["velocity"])
        t3 = time.perf_counter()
        out = {"kind": kind, "setup_s": t1 - t0, "uzawa_s": t2 - t1, "recover_s": t3 - t2, "tts_s": t3 - t0,
               "inner_iterations": u["inner_iterations"]}
    print(json.dumps(out))


def start_cpu_tts(args):
    """Launches cpu_tts_child pinned to the last usable core (the device run
    keeps its launching thread elsewhere); returns the Popen or None."""
    cores = sorted(os.sched_getaffinity(0))
    if len(cores) < 2:
        return None
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-tts-child", "--config", args.config,
           "--seed", str(args.seed)]
    try:
        return subprocess.Popen(["taskset", "-c", str(cores[-1])] + cmd, stdout=subprocess.PIPE,
                                stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)


def finish_cpu_tts(proc, timeout):
    if proc is None:
        return {"unavailable": "fewer than 2 host cores"}
    try:
        out, _ = proc.communicate(timeout=timeout)
        return json.loads(out.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        proc.kill()
        return {"unavailable": f"reference TTS child did not finish: {type(e).__name__}"}


def krylov_overhead(H, B, restart=0):
    """Per-iteration cost of the device Krylov loop (slope of capped solves,
    best of 5: PCG 5 and 45 iterations, GMRES 5 and 25, i.e. Arnoldi steps
    j = 5..25) against the V-cycle and the operator apply it contains."""
    rhs = B.rhs()
    solver = H.pcg if B.symmetric() else H.gmres
    hi = 45 if B.symmetric() else 25

    # device time on the library's stream: CUDA events around the solve (it
    # returns after its own synchronisation), so host jitter stays out
    import torch

    ext = torch.cuda.ExternalStream(B.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def t(k):
        best = 1e9
        for _ in range(5):
            e0.record(ext)
            solver(B, rhs, opt=H.KrylovOptions(max_iterations=k, rel_tol=1e-30, abs_tol=0.0, restart=restart))
            e1.record(ext)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        return best

    _, st = solver(B, rhs, opt=H.KrylovOptions(max_iterations=hi, rel_tol=1e-30, abs_tol=0.0, restart=restart))
    if st.iterations != hi:  # stopped early (breakdown past machine precision): the shorter window
        hi = 25
    t(3)
    per_it = (t(hi) - t(5)) / (hi - 5) * 1e3
    vc = B.time_apply(20)[0]
    sp = B.time_spmv(20)[0]
    return {"solver": solver.__name__ + (f"({restart})" if restart else ""), "ms_per_iteration": per_it,
            "vcycle_ms": vc, "spmv_ms": sp, "overhead_ms": per_it - vc - sp,
            "overhead_frac_of_vcycle": (per_it - vc - sp) / vc}


def workload_config(args, cfg, n):
    """The config dict both arms print (same keys, same values)."""
    return {"workload": args.config, **cfg, "cycle": "V(1,1)", "smoother": "multiplicative vertex-patch",
            "n_dofs": int(n)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle_lib as O
    cfg = CONFIGS[args.config]
    n_f = cfg["base_n"] << (cfg["levels"] - 1)
    F = O.seeded_load(n_f, args.seed)
    use_ref, kind = cpu_lib()
    B = O.OracleMG(reference=use_ref, **cpu_problem(cfg, F))
    per_step = max(1, args.ref_vcycles_per_step)
    for _ in range(min(args.warmup, 3)):
        B.time_apply(1)
    secs = sum(B.time_apply(per_step) for _ in range(args.steps))
    v = args.steps * per_step / secs
    what = ("oracle/_ref/libref.so: the reference's unmodified headers (MGPreconditioner::apply) over the "
            "Eigen-API shim" if use_ref else "oracle/ restatement (reference library not built)")
    return {"impl": "reference", "metric": METRIC if args.config == "config2" else f"hp-MG V-cycles/sec ({args.config})",
            "value": v, "unit": "V-cycles/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeded force as the GPU arm)",
            "config": {**workload_config(args, cfg, B.n), "parallelism": "replicas x1",
                       "l2": L2_NOTE},
            "cpu_baseline": {"value": v, "unit": "V-cycles/s", "cores": 1, "kind": kind,
                             "sample": f"{args.steps} x {per_step} V-cycles, {what}", **host_info()},
            "e2e": {"value": v, "unit": "V-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hpmg", choices=["hpmg", "reference"])
    ap.add_argument("--config", default="config2", choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-baseline", dest="cpu_baseline", action="store_true", default=True)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-vcycles", type=int, default=3)
    ap.add_argument("--ref-vcycles-per-step", type=int, default=1)
    ap.add_argument("--no-cpu-tts", dest="cpu_tts", action="store_false", default=True)
    ap.add_argument("--no-krylov", dest="krylov", action="store_false", default=True)
    ap.add_argument("--cpu-tts-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_tts_child:
        cpu_tts_child(args.config, args.seed)
        return
    args.warmup = max(args.warmup, 3) if args.impl == "hpmg" else args.warmup
    if args.impl == "reference":
        out = run_reference(args)
    else:
        rank, world, local, dist = dist_init()
        out = run_hpmg(args, rank, world, local, dist)
        if dist:
            dist.barrier()
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
