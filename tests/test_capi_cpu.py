"""CPU-side checks of the C ABI library (no GPU): exported symbols, host-side
plan (wave schedule) logic, problem sizes against SURVEY.md 8 and the
no-CPU-fallback contract."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2303_06762_b200 as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hpmg", "capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpmg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = H.lib()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def plan(base_n, levels, k, level=-1, mesh="unit_square"):
    L = H.lib()
    md = H._Mesh()
    (L.hpmg_unit_square_mesh if mesh == "unit_square" else L.hpmg_step_mesh)(base_n, levels, C.byref(md))
    out = np.zeros(128, np.int64)
    L.hpmg_plan_check.argtypes = [C.POINTER(H._Mesh), C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_int]
    n = L.hpmg_plan_check(C.byref(md), k, level, out.ctypes.data_as(C.POINTER(C.c_int64)), 128)
    assert n > 0, L.hpmg_last_error().decode()
    nw = int(out[2])
    return dict(n=int(out[0]), patches=int(out[1]), waves=nw, cover=bool(out[3]), indep=bool(out[4]),
                order=bool(out[5]), max_nf=int(out[6]), sizes=[int(v) for v in out[7:7 + nw]],
                asap=[int(v) for v in out[7 + nw:7 + 2 * nw]])


@pytest.mark.parametrize("base_n,levels,k,n_expect", [
    (8, 5, 1, 195584),      # config 1
    (16, 5, 3, 1568768),    # config 2
    (8, 5, 2, 293376),      # config 3, k=2
    (8, 6, 2, 1176576),     # config 5
    (8, 5, 4, 488960),      # config 3, k=4 (beyond the reference's k <= 3)
    (8, 5, 6, 684544),      # config 3, k=6
])
def test_config_sizes_and_wave_schedule(base_n, levels, k, n_expect):
    p = plan(base_n, levels, k)
    assert p["n"] == n_expect
    assert p["cover"] and p["indep"] and p["order"]
    assert p["waves"] == 9  # exact parallel schedule of the ascending sweep on refined levels
    assert sum(p["sizes"]) == p["patches"] == sum(p["asap"])
    assert p["sizes"] == p["asap"]  # wide schedules keep the as-soon-as-possible levelling


def test_wave_sizes_match_survey_appendix_b():
    # 256^2 mesh from an 8x8 base
    p = plan(8, 6, 0, level=5)
    assert p["asap"] == [16639, 8376, 10511, 11415, 7128, 5576, 3936, 1521, 945]
    assert p["sizes"] == p["asap"] and p["indep"] and p["order"]


@pytest.mark.parametrize("base_n,levels,level,waves", [(8, 5, 1, 26), (16, 5, 1, 50), (8, 5, 2, 9)])
def test_coarse_level_wave_counts(base_n, levels, level, waves):
    # 26 waves on level 1 of an 8x8 base, 50 for 16x16, then 9
    p = plan(base_n, levels, 0, level=level)
    assert p["waves"] == waves and p["indep"] and p["order"] and p["cover"]
    if waves > 12:  # the one-CTA level: every wave fits one 24-patch pass (ASAP: 79 / 287 in wave 0)
        assert max(p["sizes"]) <= 24 < max(p["asap"])


def test_step_domain_plan():
    p = plan(2, 3, 1, mesh="step")
    assert p["cover"] and p["indep"] and p["order"]


def test_no_cpu_fallback():
    """Without a CUDA device the product must refuse to run (no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HpmgError, match="no CPU fallback"):
        H.MGPreconditioner(base_n=2, levels=2)


def test_seeded_load_matches_oracle_generator():
    import oracle_lib as O
    assert np.array_equal(H.seeded_load(16, 3), O.seeded_load(16, 3))
