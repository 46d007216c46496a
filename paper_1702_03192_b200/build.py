"""Build libmtnn_b200.so in-tree (sm_100a only).

Every .cu is compiled by nvcc for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` (ncu source pages); host C++ by g++ with
``-ffp-contract=off`` so the float64 tree walk rounds exactly like the
reference. The library links cudart statically and resolves the driver's
tensor-map encoder at run time, so it loads on a machine with no GPU/driver
(the C-ABI symbol tests) and carries no dependency on torch's CUDA runtime.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libmtnn_b200.so"
BUILD = PKG.parent / "build" / "mtnn_b200"
INCLUDE = PKG.parent / "include"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
    "-Xptxas", "-v", f"-I{INCLUDE}",
]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall",
             f"-I{CUDA_HOME / 'include'}", f"-I{INCLUDE}"]

SOURCES = ["transpose.cu", "gemm_ffma.cu", "gemm_tc.cu", "split_f16.cu", "fixup.cu", "operands.cu", "peer.cu", "gate.cu", "mtnn_abi.cpp", "model.cpp", "profile.cpp",
           "ipc.cpp"]
HEADERS = ["common.h", "workspace.h", "model.h", "fix.h", "sgemm_tile.cuh", "pdl.h"]


def _run(cmd, log):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    return proc


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    headers = [CSRC / h for h in HEADERS] + [INCLUDE / "mtnn_b200.h", Path(__file__)]
    objs = []
    log_path = BUILD / "build.log"
    with open(log_path, "w") as log:
        for src in SOURCES:
            path = CSRC / src
            obj = BUILD / (src + ".o")
            objs.append(obj)
            if not force and not _stale(obj, [path, *headers]):
                continue
            if src.endswith(".cu"):
                cmd = [NVCC, *NVCC_FLAGS, "-c", str(path), "-o", str(obj)]
            else:
                cmd = [shutil.which("g++") or "g++", *CXX_FLAGS, "-c", str(path), "-o", str(obj)]
            proc = _run(cmd, log)
            if verbose:
                sys.stderr.write(proc.stderr)
        if force or _stale(LIB, objs):
            tmp = LIB.with_suffix(".so.tmp")
            cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp),
                   *map(str, objs), "-lpthread", "-ldl", "-lrt"]
            _run(cmd, log)
            os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
