"""Reference CPU time-to-solution at every BASELINE configuration with a
reference path (configs 1, 3, 5; config 2 is timed by bench.py): the
reference itself (oracle/_ref/libref.so), one single-threaded process per
configuration, each pinned to its own host core and run concurrently
(the reference never uses more than one thread; concurrent runs share the
host's memory bandwidth, so these times are upper bounds of a solo run).
TTS = MGPreconditioner construction + uzawa_solve (2 outer steps) +
recover_locals, as bench.py's cpu_reference. Config 5 uses the reference's
own (unrestarted) GMRES. Prints one JSON line per configuration.
Usage (GPU box or build container): python tools/ref_tts.py [names...]"""
import concurrent.futures as cf
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

NAMES = ["config1"] + [f"config3_k2_al{al}_b{b}" for al in ("1", "100", "10000") for b in ("0", "100")] + \
        ["config5_re1", "config5_re100"]


def one(name, core):
    os.sched_setaffinity(0, {core})
    import oracle_lib as O
    from ref_runs import oracle_kwargs

    t0 = time.perf_counter()
    m = O.OracleMG(reference=True, **oracle_kwargs(name))
    t1 = time.perf_counter()
    u = m.uzawa()
    t2 = time.perf_counter()
    m.recover(u["velocity"])
    t3 = time.perf_counter()
    return dict(config=name, kind="reference", core=core, n=int(m.n), setup_s=t1 - t0, uzawa_s=t2 - t1,
                recover_s=t3 - t2, tts_s=t3 - t0, inner_iterations=u["inner_iterations"], converged=u["converged"])


def main():
    import oracle_lib as O

    if not O.ref_available():
        raise SystemExit("oracle/_ref/libref.so not built")
    names = sys.argv[1:] or NAMES
    cores = sorted(os.sched_getaffinity(0))
    with cf.ProcessPoolExecutor(max_workers=min(len(names), len(cores)), mp_context=mp.get_context("spawn")) as ex:
        futs = [ex.submit(one, n, cores[i % len(cores)]) for i, n in enumerate(names)]
        for f in futs:
            r = f.result()
            r["host"] = platform.processor() or platform.machine()
            r["nproc"] = len(cores)
            r["concurrent_runs"] = len(names)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
