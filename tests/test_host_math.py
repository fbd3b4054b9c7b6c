"""Host FP64 check of the FMM translation conventions (harmonics.h +
operators.cpp, the code that generates the device operators): P2M, M2M, M2L,
L2L, L2P, P2L, M2P against direct 1/r sums (tools/fmm_math_check.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fmm_translation_math(tmp_path):
    exe = tmp_path / "fmm_math_check"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", str(exe),
                           os.path.join(ROOT, "tools", "fmm_math_check.cpp"),
                           os.path.join(ROOT, "paper_2409_12375_b200", "csrc", "operators.cpp")])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert "ALL OK" in r.stdout
