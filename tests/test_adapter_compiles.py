"""The C++ drop-in adapter (include/hpmg/hdivmg_gpu.hpp) needs the reference's
Eigen-based headers, absent here; it is compiled -fsyntax-only against a
declaration-only stand-in of those headers (tests/native/stub_hdivmg) so its
use of the C ABI (argument counts, struct layouts) is checked on every run."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_hdivmg_adapter_compiles(tmp_path):
    src = tmp_path / "use_adapter.cpp"
    src.write_text('#include "hpmg/hdivmg_gpu.hpp"\n'
                   "hdivmg::NSSolution f(const hdivmg::MeshHierarchy& h) {\n"
                   "  hpmg::MGPreconditioner B(h, 2, hdivmg::VelocityBC{}, hdivmg::AssemblyOptions{}, 1e3, {});\n"
                   "  hdivmg::Vec x(B.rhs().size());\n"
                   "  hpmg::pcg(B, B.rhs(), x);\n"
                   "  hpmg::uzawa_solve(B);\n"
                   "  auto sol = hpmg::navier_stokes_solve(h, 2, hdivmg::VelocityBC{}, 1e-2, {}, 1e3);\n"
                   "  auto post = hpmg::postprocess_velocity(B, sol.velocity, sol.locals.grad_coeffs);\n"
                   "  hpmg::measure_errors(B, sol.velocity, sol.locals.grad_coeffs, post,\n"
                   "                       [](const hdivmg::Vec2& x) { return x; },\n"
                   "                       [](const hdivmg::Vec2&) { return hdivmg::Mat2{}; });\n"
                   "  return sol;\n"
                   "}\n")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(ROOT, "tests", "native", "stub_hdivmg"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
