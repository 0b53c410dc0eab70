"""In-tree build of libmoe_b200.so (sm_100a) with nvcc.

Objects go to paper_2206_03382_b200/build/, the shared library next to this file so it travels
with the repo snapshot to the GPU box. Incremental: a source is recompiled when it or any
header under csrc/ or include/ is newer than its object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = Path(os.environ.get("MOE_BUILD_DIR", PKG / "build"))
LIB = Path(os.environ.get("MOE_LIB_OUT", PKG / "libmoe_b200.so"))
EXTRA = os.environ.get("MOE_NVCC_EXTRA", "").split()  # e.g. tuning variants: -DMOE_GEMM_STAGES=4

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
    "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + EXTRA + ["-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd.insert(1, "-Xptxas=-v") if verbose else None
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    hm = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest or force:
        cmd = [nvcc()] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + [
            "-lnccl", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_checks(force: bool = False) -> Path:
    """The bounds-checked variant (-DMOE_CHECKS: device-side MOE_CHECK traps, csrc/checks.cuh),
    in-tree beside the product library; tests/test_gpu_checks.py runs the GPU suite against it."""
    global OBJ, LIB, EXTRA
    saved = (OBJ, LIB, EXTRA)
    try:
        OBJ, LIB, EXTRA = PKG / "build_checks", PKG / "libmoe_b200_checks.so", EXTRA + ["-DMOE_CHECKS"]
        return build(force=force)
    finally:
        OBJ, LIB, EXTRA = saved


if __name__ == "__main__":
    if "--checks" in sys.argv:
        print(build_checks(force="-f" in sys.argv))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
