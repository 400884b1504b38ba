"""In-tree build of the native engine (libttutv_b200.so) for sm_100a.

The shared library is written next to this file under ``lib/`` so that it travels with
the repository snapshot to the GPU box (no JIT cache). Every CUDA translation unit is
compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
OBJDIR = PKG / "lib" / "obj"
LIBNAME = "libttutv_b200.so"
ROOT = PKG.parent

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr", "-I" + str(ROOT / "include"), "-I" + str(CSRC),
]
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-I" + str(ROOT / "include"), "-I" + str(CSRC)]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return cand


def _cuda_home() -> Path:
    return Path(_nvcc()).resolve().parent.parent


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJDIR / (src.stem + ".o")
    deps = [src] + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + sorted((ROOT / "include").rglob("*.h*"))
    if obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return obj
    if src.suffix == ".cu":
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["/usr/bin/g++", *CXX_FLAGS, "-I" + str(_cuda_home() / "include"), "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, env=_env())
    return obj


def _env() -> dict:
    env = dict(os.environ)
    # The image's CXX points at a wrapper that lacks libgomp's spec; nvcc must use the system g++.
    env.pop("CXX", None)
    env.pop("CC", None)
    return env


def build(verbose: bool = False) -> Path:
    """Compile every CUDA/C++ source and link ``lib/libttutv_b200.so``."""
    OBJDIR.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    out = LIBDIR / LIBNAME
    if not out.exists() or out.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, env=_env())
    return out


def build_inputs(verbose: bool = False) -> Path:
    """hostgen/inputs.cpp -> lib/libttutv_inputs.so: the seeded input generators of the
    BASELINE configs (harness code for bench.py and the tests, not the product path).
    Default x86-64 target and no FP contraction, like the reference build, so the buffers
    are bitwise those of the reference's own generators."""
    src = PKG / "hostgen" / "inputs.cpp"
    out = LIBDIR / "libttutv_inputs.so"
    LIBDIR.mkdir(parents=True, exist_ok=True)
    if out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", str(src), "-o", str(out)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, env=_env())
    return out


def build_dropin_check(verbose: bool = False) -> Path:
    """tests/cpp/dropin_check.cpp: a caller written against the reference headers,
    compiled through the compat forwarding headers and linked to libttutv_b200.so."""
    src = ROOT / "tests" / "cpp" / "dropin_check.cpp"
    out = LIBDIR / "dropin_check"
    lib = LIBDIR / LIBNAME
    if out.exists() and out.stat().st_mtime >= max(src.stat().st_mtime, lib.stat().st_mtime):
        return out
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-I" + str(ROOT / "include" / "ttutv_b200" / "compat"),
           "-I" + str(ROOT / "include"), str(src), "-o", str(out), "-L" + str(LIBDIR), "-lttutv_b200",
           "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, env=_env())
    return out


if __name__ == "__main__":
    print(build(verbose=True))
    print(build_inputs(verbose=True))
    print(build_dropin_check(verbose=True))
