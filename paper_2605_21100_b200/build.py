"""Build recipes: the sm_100a product library and the CPU oracle.

Product:  paper_2605_21100_b200/_build/libdcp_b200.so
          = every csrc/*.cu (kernels + C ABI) + host/*.cpp (dcpsim C++ drop-in),
          nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo, static cudart.
Oracle:   make -C oracle  (test infrastructure; see oracle/Makefile).

The env CXX (/opt/gcc/bin/g++) is a wrapper without libgomp, so both nvcc's
host compiler and the oracle use /usr/bin/g++ explicitly.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
REPO = ROOT.parent
CSRC = ROOT / "csrc"
HOST = ROOT / "host"
BUILD = ROOT / "_build"
LIB = BUILD / "libdcp_b200.so"

NVCC = os.environ.get("DCP_NVCC", "/usr/local/cuda/bin/nvcc")
HOST_CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++20", "-ccbin", HOST_CXX,
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    f"-I{REPO / 'include'}", f"-I{CSRC}",
]


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(HOST.glob("*.cpp")) if HOST.exists() else []
    return cu, cpp


def _deps():
    return (sorted(CSRC.glob("*.cu*")) + sorted(CSRC.glob("*.h")) + sorted(HOST.glob("*.[ch]pp"))
            + sorted((REPO / "include").rglob("*.h*")))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_product(verbose: bool = True, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    cu, cpp = _sources()
    deps = _deps()
    objs = []
    for src in cu + cpp:
        obj = BUILD / (src.name + ".o")
        objs.append(obj)
        if force or _stale(obj, deps):
            if src.suffix == ".cu":
                _run([NVCC, *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj], verbose)
            else:
                _run([NVCC, *ARCH, *NVCC_FLAGS, "-x", "cu", "-c", src, "-o", obj], verbose)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-ccbin", HOST_CXX, "-cudart", "static",
              "-o", LIB, *objs, "-lrt"], verbose)
    return LIB


def build_oracle(verbose: bool = True) -> None:
    _run(["make", "-s", "-C", REPO / "oracle"], verbose)


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    build_product(force=force)
    build_oracle()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
