"""The GPU suite against the bounds-checked build (compute-sanitizer is closed on this pool):
libmoe_b200_checks.so is the product source compiled with -DMOE_CHECKS, whose device-side
MOE_CHECK traps (csrc/checks.cuh) verify token / slot / expert / rank / list-entry ranges in
encode, decode(-backward), encode-backward, assign, BPR ranking, the certified gate's fix-up
list, the ReLU fix-up and the up-GEMM certificate packing. A violated check traps the kernel and
fails the wrapped tests. Runs in a subprocess (MOE_LIB_PATH selects the library at import)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2206_03382_b200" / "libmoe_b200_checks.so"


@pytest.mark.skipif(os.environ.get("MOE_CHECKS_RUN") == "1", reason="already inside the checks run")
def test_gpu_suite_under_bounds_checks(cuda):
    if not LIB.exists():
        pytest.fail("libmoe_b200_checks.so missing: run __graft_entry__.build()")
    env = dict(os.environ, MOE_LIB_PATH=str(LIB), MOE_CHECKS_RUN="1")
    files = ["tests/test_gpu_ops.py", "tests/test_gpu_layer.py", "tests/test_gpu_gate_tc.py",
             "tests/test_gpu_guard.py", "tests/test_gpu_gemm.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        *files], env=env, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "MOE_CHECK failed" not in r.stdout + r.stderr
