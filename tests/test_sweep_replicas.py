"""CPU (gloo, world size 2) check of the replica-parallel sweep driver
(paper_2303_06762_b200/sweep.py): every job runs exactly
once, round-robin over ranks, and every rank ends with all rows in job order.
The solve itself is stubbed (it needs a GPU); the partition and the gather
over the gloo group are the real code."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2303_06762_b200 import sweep  # noqa: E402


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import torch.distributed as dist
from paper_2303_06762_b200 import sweep
dist.init_process_group(backend="gloo")
rank = dist.get_rank()
jobs = sweep.config_runs()
res = sweep.sweep(jobs, run=lambda j: {{"config": j["name"], "rank": rank}}, dist=dist)
print(json.dumps({{"rank": rank, "rows": res}}))
dist.barrier()
dist.destroy_process_group()
"""


def test_job_list_covers_the_baseline_sweeps():
    jobs = sweep.config_runs()
    names = [j["name"] for j in jobs]
    assert len(names) == len(set(names)) == 2 + 18 + 3
    c3 = [j for j in jobs if j["name"].startswith("config3")]
    assert sum(j["reference_order"] for j in c3) == 6 and len(c3) == 18  # 6 pinned + 12 beyond k <= 3
    for world in (1, 2, 3, 8):
        parts = [sweep.partition(jobs, r, world) for r in range(world)]
        flat = [j["name"] for p in parts for j in p]
        assert sorted(flat) == sorted(names)


def test_two_rank_sweep_over_gloo():
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER.format(root=ROOT)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=120)
        assert p.returncode == 0, e[-2000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    names = [j["name"] for j in sweep.config_runs()]
    for o in outs:
        assert [r["config"] for r in o["rows"]] == names
        assert [r["rank"] for r in o["rows"]] == [i % 2 for i in range(len(names))]
