"""A C++ program using the drop-in facade (include/moe_b200.hpp -> C ABI) reproduces the fp64
oracle within the fp32 tolerance (1e-5) and raises the reference's exception types."""
import subprocess
from pathlib import Path

import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_facade_against_oracle(cuda, tmp_path):
    oracle.build()
    exe = tmp_path / "facade_test"
    pkg = ROOT / "paper_2206_03382_b200"
    cmd = ["g++", "-std=c++17", "-O2", str(ROOT / "tests" / "cpp" / "facade_test.cpp"), "-o", str(exe),
           f"-I{ROOT / 'include'}", f"-L{pkg}", "-lmoe_b200", f"-L{ROOT / 'oracle' / 'build'}",
           "-loracle", f"-Wl,-rpath,{pkg}:{ROOT / 'oracle' / 'build'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "FACADE PASS" in r.stdout
