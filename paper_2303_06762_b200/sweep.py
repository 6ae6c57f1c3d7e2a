"""Replica-parallel configuration sweeps (the path does not
shard, so several GPUs serve independent solves). Every BASELINE.json run the
device path expresses is one job: config 1, config 2, config 3's robustness
sweep (k in {2, 4, 6} x AL in {1, 1e2, 1e4} x mass in {0, 1e2}: 6 runs the
reference can express, 12 beyond its k <= 3) and config 5's Oseen solves
(Re in {1, 100, 1000}). Under torchrun, rank r takes jobs r, r + N, ...; the
rows are gathered on rank 0 over a gloo group (no collective on the solve
path) and written as the reference's CSV (io.py) or JSON lines.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        -m paper_2303_06762_b200.sweep --only config3 --csv sweep.csv
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time


def config_runs():
    """All jobs, in a fixed order (every rank enumerates the same list)."""
    jobs = [dict(name="config1", base_n=8, levels=5, k=1, nu=1.0, beta=1.0, inv_eps=1e3),
            dict(name="config2", base_n=16, levels=5, k=3, nu=1.0, beta=1e-2, inv_eps=1e3)]
    for k in (2, 4, 6):
        for al in (1.0, 1e2, 1e4):
            for beta in (0.0, 1e2):
                jobs.append(dict(name=f"config3_k{k}_al{al:g}_m{beta:g}", base_n=8, levels=5, k=k, nu=1.0,
                                 beta=beta, inv_eps=al, reference_order=k <= 3))
    for re in (1.0, 100.0, 1000.0):
        jobs.append(dict(name=f"config5_re{re:g}", base_n=8, levels=6, k=2, nu=1.0 / re, beta=0.0, inv_eps=1e3,
                         oseen=True, lo=-0.1, hi=0.1))
    return jobs


def partition(jobs, rank, world):
    """Round-robin share of `jobs` for `rank` (deterministic, disjoint, covering)."""
    return [j for i, j in enumerate(jobs) if i % world == rank]


def run_job(r, seed=1):
    """One solve on this rank's GPU: setup, V-cycle time, AL-Uzawa (PCG, or
    GMRES(50) for the Oseen runs); returns a JSON-able dict."""
    import paper_2303_06762_b200 as H
    n_f = r["base_n"] << (r["levels"] - 1)
    F = H.seeded_load(n_f, seed, r.get("lo", -1.0), r.get("hi", 1.0))
    oseen = r.get("oseen", False)
    t0 = time.perf_counter()
    B = H.MGPreconditioner(base_n=r["base_n"], levels=r["levels"], k=r["k"], nu=r["nu"], beta=r["beta"],
                           inv_eps=r["inv_eps"], cycle=H.CYCLE_V, structured_load=(n_f, F),
                           bc="lid_unit" if oseen else None, wind="config5_wind" if oseen else None)
    setup = time.perf_counter() - t0
    ms, _ = B.time_apply(10)
    kopt = H.KrylovOptions(restart=50) if oseen else H.KrylovOptions()
    t1 = time.perf_counter()
    sol = H.uzawa_solve(B, krylov=kopt)
    wall = time.perf_counter() - t1
    out = dict(config=r["name"], n=int(B.n), k=r["k"], nu=r["nu"], beta=r["beta"], inv_eps=r["inv_eps"],
               setup_s=round(setup, 3), vcycle_ms=round(ms, 4), inner_iterations=sol.report.inner_iterations,
               solve_device_s=round(sol.report.seconds, 4), solve_wall_s=round(wall, 4),
               tts_s=round(setup + wall, 3), converged=sol.report.converged,
               not_applicable=sol.report.not_applicable, final_divergence=sol.report.final_divergence,
               krylov="GMRES(50)" if oseen else "PCG", parity="pinned" if r.get("reference_order", True) else
               "unpinned (k > 3)")
    B.close()
    return out


def csv_row(res, run_id):
    from .io import CsvRow
    status = "NA" if res.get("not_applicable") else ("ok" if res.get("converged") else "fail")
    return CsvRow(run_id=run_id, subcommand=res["config"], k=res["k"], level=0, nu=res["nu"], beta=res["beta"],
                  m=1, cycle="v", outer=len(res["inner_iterations"]), inner_iters=list(res["inner_iterations"]),
                  div_u=res["final_divergence"] if status == "ok" else None, status=status)


def gather(rows, dist):
    """All ranks' rows on every rank, in job order (rows carry their job index)."""
    if dist is None:
        return sorted(rows, key=lambda t: t[0])
    group = dist.new_group(backend="gloo")
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, rows, group=group)
    return sorted((t for p in parts for t in p), key=lambda t: t[0])


def sweep(jobs, run=run_job, dist=None):
    """Runs this rank's share of `jobs` and returns every job's result (index order)."""
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    mine = [(i, j) for i, j in enumerate(jobs) if i % world == rank]
    rows = [(i, run(j)) for i, j in mine]
    return [r for _, r in gather(rows, dist)]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="", help="run the jobs whose name starts with this")
    ap.add_argument("--csv", default="", help="write the reference's CSV schema here (rank 0)")
    args = ap.parse_args(argv)
    dist = None
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch
        import torch.distributed as tdist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        tdist.init_process_group(backend="nccl" if torch.cuda.is_available() else "gloo")
        dist = tdist
    jobs = [j for j in config_runs() if j["name"].startswith(args.only)]
    results = sweep(jobs, dist=dist)
    if dist is None or dist.get_rank() == 0:
        for res in results:
            print(json.dumps(res), flush=True)
        if args.csv:
            from .io import write_csv_header, write_csv_row
            with open(args.csv, "w") as f:
                write_csv_header(f)
                for i, res in enumerate(results):
                    write_csv_row(f, csv_row(res, i + 1))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
