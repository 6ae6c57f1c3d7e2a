"""Host build of the product's element-condensation routine (condense.cuh)
checked element by element against the oracle (tests/native/check_condense.cpp).
Test infrastructure only: the product launches the same code as a CUDA kernel."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_condense_element_matches_oracle(tmp_path):
    exe = tmp_path / "check_condense"
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe),
                    os.path.join(ROOT, "tests", "native", "check_condense.cpp")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "RESULT PASS" in out.stdout
