"""CPU (gloo, world size 2) checks of bench.py's multi-process plumbing.

The path does not shard: `bench.py --gpus N` runs N
independent replicas under torchrun, and the only collectives are the
barrier and the max over ranks of the device-timed region. These tests run
that plumbing in two real processes on the gloo backend, and the reference
arm's rank gating (rank 0 alone works, the others exit without output).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import bench
rank, world, local, dist = bench.dist_init()
ms = [3.0, 5.0][rank]
ms_max = bench.max_over_ranks(ms, dist)
rate = bench.whole_job_rate(20, ms_max, world)
dist.barrier()
print(json.dumps({{"rank": rank, "world": world, "backend": dist.get_backend(), "ms_max": ms_max, "rate": rate}}))
dist.destroy_process_group()
"""


def run_two_ranks(code, extra_env=None, timeout=120):
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        env.update(extra_env or {})
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            p.kill()
            raise
        assert p.returncode == 0, e[-2000:]
        outs.append(o)
    return outs


def test_max_over_ranks_and_whole_job_rate_gloo():
    outs = run_two_ranks(WORKER.format(root=ROOT))
    res = [json.loads(o.strip().splitlines()[-1]) for o in outs]
    for r in res:
        assert r["world"] == 2 and r["backend"] == "gloo"
        assert r["ms_max"] == 5.0  # the slowest replica sets the job time
        assert r["rate"] == pytest.approx(20 * 2 / 5e-3)  # weak scaling: total units / slowest time


def test_single_process_helpers():
    assert bench.max_over_ranks(4.0, None) == 4.0
    assert bench.whole_job_rate(10, 2.0, 1) == pytest.approx(5000.0)


def test_reference_arm_only_rank0_reports():
    # rank 1 of a 2-rank torchrun launch of the reference arm must exit 0
    # without doing work or printing a line (the driver reads rank 0's line)
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2", CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""
