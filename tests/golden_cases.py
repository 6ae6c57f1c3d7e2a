"""Loader of the committed reference outputs in tests/golden/ (written by
tools/make_golden.py from the reference itself, oracle/_ref/libref.so)."""
import json
import os

import numpy as np

import oracle_lib as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        idx = json.load(f)
    idx.pop("_source", None)
    return idx


NAMES = sorted(index())


def load(name):
    meta = index()[name]
    data = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return meta, data


def gpu_kwargs(meta, data):
    """MGPreconditioner arguments equal to the reference run's OracleMG ones."""
    kw = dict(meta["kwargs"])
    if kw.pop("bc", O.BC_NONE) == O.BC_LID_UNIT:
        kw["bc"] = "lid_unit"
    if kw.pop("wind", O.WIND_NONE) == O.WIND_CURL:
        kw["wind"] = "config5_wind"
    n_f = kw["base_n"] << (kw["levels"] - 1)
    kw["structured_load"] = (n_f, data["load"])
    return kw


def oracle_kwargs(meta, data):
    return dict(meta["kwargs"], load_kind=O.LOAD_ARRAY, load=data["load"])


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
