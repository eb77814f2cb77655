"""Build recipes: the sm_100a CUDA library (product) and the oracle (tests).

The product library ``libstripefrac_cuda.so`` is built in-tree with nvcc for
``sm_100a`` only. The oracle pieces (``oracle/liboracle_port.so``, the C
restatement, and ``oracle/_ref/`` built from the reference sources when
``/root/reference`` is present) are test infrastructure.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libstripefrac_cuda.so"
ORACLE = ROOT / "oracle"
ORACLE_LIB = ORACLE / "liboracle_port.so"
REFERENCE = Path("/root/reference/proj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
    "-Xptxas", "-warn-spills",
    "-lcublasLt", "-Xlinker", "-rpath", "-Xlinker", "/usr/local/cuda/lib64",
]
SOURCES = ["sf_api.cu", "host_prep.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build stripefrac-b200")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).exists() and Path(d).stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False, out: Path = LIB, defines=()) -> Path:
    """The product library; `defines` (-D...) and `out` build A/B variants
    of the same sources (tools/build_ab.sh), never the product path."""
    deps = ([CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) +
            list((ROOT / "include").glob("*.h")))
    if force or _stale(out, deps):
        cmd = [_nvcc(), *NVCC_FLAGS, *defines, f"-I{ROOT / 'include'}", f"-I{CSRC}",
               *[str(CSRC / s) for s in SOURCES], "-o", str(out)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return out


PEAKS_SRC = ROOT / "tools" / "fp_peaks.cu"
PEAKS_LIB = ROOT / "tools" / "libsf_peaks.so"


def build_tools(force: bool = False, verbose: bool = False) -> None:
    """Measurement tooling: FP64/FP32 FMA peak microbenchmark (roofline denominators)."""
    if force or _stale(PEAKS_LIB, [PEAKS_SRC]):
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler",
               "-fPIC", "-shared", str(PEAKS_SRC), "-o", str(PEAKS_LIB)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)


def build_oracle(force: bool = False, verbose: bool = False) -> None:
    """Test infrastructure: C restatement + (when present) the reference build."""
    src = ORACLE / "stripefrac_oracle.c"
    if force or _stale(ORACLE_LIB, [src]):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
               str(src), "-o", str(ORACLE_LIB), "-lm"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    if REFERENCE.exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE), "-j8"], check=True,
                       stdout=None if verbose else subprocess.DEVNULL)


def build_dropin(verbose: bool = False) -> None:
    """Test infrastructure: the reference's own suites linked against the drop-in
    (tests/dropin/Makefile; needs the reference sources, so build container only)."""
    if REFERENCE.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "dropin"), "-j8"], check=True,
                       stdout=None if verbose else subprocess.DEVNULL)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_native(force=force, verbose=verbose)
    build_tools(force=force, verbose=verbose)
    build_oracle(force=force, verbose=verbose)
    build_dropin(verbose=verbose)


if __name__ == "__main__":
    build_all(force=True, verbose=True)
