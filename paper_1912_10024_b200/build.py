"""Build every native artefact in-tree (no JIT cache; the .so files travel to the GPU box).

  paper_1912_10024_b200/libqtsse.so   product: C-ABI (qt_sse.h, qt_rgf.h) + sm_100a kernels (nvcc)
  qtgen/libqtgen_host.so              input generator, host side (gcc, OpenMP)
  qtgen/libqtgen_dev.so               input generator, device side (nvcc, sm_100a)
  oracle/liboracle.so                 CPU oracle + brute force (gcc; test infrastructure)

Usage: python -m paper_1912_10024_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1912_10024_b200"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> Path:
    """NCCL of the torch wheel (nvidia-nccl), so one libnccl.so.2 lives in the process with torch's."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL wheel) not found")
    return Path(list(spec.submodule_search_locations)[0])


NCCL_DIR = _nccl_dir()


def _cublas_dir() -> Path:
    """cuBLAS of the torch wheel (nvidia-cublas), so one libcublas.so.12 lives in the process with torch's."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.cublas")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.cublas (torch's cuBLAS wheel) not found")
    return Path(list(spec.submodule_search_locations)[0])


CUBLAS_DIR = _cublas_dir()


def _wheel_dir(mod: str) -> Path:
    import importlib.util
    spec = importlib.util.find_spec(mod)
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError(f"{mod} (torch's CUDA library wheel) not found")
    return Path(list(spec.submodule_search_locations)[0])


CUSOLVER_DIR = _wheel_dir("nvidia.cusolver")

TARGETS = {
    "libqtsse": dict(
        out=PKG / "libqtsse.so",
        srcs=sorted((PKG / "csrc").glob("*.cu")),
        deps=sorted((PKG / "csrc").glob("*.cuh")) + [ROOT / "include" / "qt_sse.h", ROOT / "include" / "qt_rgf.h"],
        cmd=lambda srcs, out: [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
                               "-Xcompiler", "-fPIC,-O2", "-shared", f"-I{ROOT / 'include'}",
                               f"-I{NCCL_DIR / 'include'}", *map(str, srcs), "-o", str(out), "-lcudart",
                               f"-L{NCCL_DIR / 'lib'}", "-l:libnccl.so.2", f"-Xlinker=-rpath,{NCCL_DIR / 'lib'}",
                               f"-L{CUBLAS_DIR / 'lib'}", "-l:libcublas.so.12", f"-Xlinker=-rpath,{CUBLAS_DIR / 'lib'}",
                               f"-L{CUSOLVER_DIR / 'lib'}", "-l:libcusolver.so.11",
                               f"-Xlinker=-rpath,{CUSOLVER_DIR / 'lib'}"],
    ),
    "qtgen_dev": dict(
        out=ROOT / "qtgen" / "libqtgen_dev.so",
        srcs=[ROOT / "qtgen" / "gen_dev.cu"],
        deps=[ROOT / "include" / "qt_gen.h"],
        cmd=lambda srcs, out: [NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               f"-I{ROOT / 'include'}", *map(str, srcs), "-o", str(out), "-lcudart"],
    ),
    "qtgen_host": dict(
        out=ROOT / "qtgen" / "libqtgen_host.so",
        srcs=[ROOT / "qtgen" / "gen_host.c"],
        deps=[ROOT / "include" / "qt_gen.h"],
        cmd=lambda srcs, out: ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               f"-I{ROOT / 'include'}", *map(str, srcs), "-o", str(out), "-lm"],
    ),
    "oracle": dict(
        out=ROOT / "oracle" / "liboracle.so",
        srcs=[ROOT / "oracle" / "oracle.c", ROOT / "oracle" / "brute.c"],
        deps=[],
        # portable flags: the .so is built here and may run on another host CPU
        cmd=lambda srcs, out: ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", *map(str, srcs), "-o", str(out)],
    ),
}


def _stale(t) -> bool:
    out = t["out"]
    if not out.exists():
        return True
    mt = out.stat().st_mtime
    return any(Path(p).stat().st_mtime > mt for p in list(t["srcs"]) + list(t["deps"]))


def build(force: bool = False, only: list[str] | None = None, verbose: bool = False) -> None:
    for name, t in TARGETS.items():
        if only and name not in only:
            continue
        if not force and not _stale(t):
            continue
        cmd = t["cmd"](t["srcs"], t["out"])
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"build of {name} failed")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
