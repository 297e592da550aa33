"""In-tree build of libspikecam_b200.so (nvcc, sm_100a only).

The shared library is a plain C-ABI (include/spikecam_b200.h); Python binds it
with ctypes and the C++ drop-in layer (cpp/) links it.  It is built into the
package directory so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libspikecam_b200.so"
CHECKED_LIB = PKG / "libspikecam_b200_checked.so"  # bounds-checked build (SPK_CHECK traps)
CPP_LIB = PKG / "libspikecam_cpp.so"
CXX = "/usr/bin/g++"  # the system compiler (the image's CC/CXX env may point elsewhere)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-static-global-template-stub=false",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libspikecam_b200.so")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def source_sha16() -> str:
    """SHA-256 (16 hex) of what libspikecam_b200.so is built from: the kernel
    sources, the C-ABI header and the nvcc flags.  nvcc's output is not
    byte-reproducible, so profiles are tied to a build by this hash
    (bench.py, profiles/ncu_step_profile.py).  build_library() rebuilds the
    library whenever a source is newer, so the library on disk is the build
    of these sources."""
    import hashlib
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "spikecam_b200.h"]
    if not LIB.exists():
        return "missing"
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for d in deps:
        h.update(d.name.encode())
        h.update(d.read_bytes())
    return h.hexdigest()[:16]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "spikecam_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, f"-I{ROOT / 'include'}", "-o", str(tmp), *map(str, sources())]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    tmp.replace(LIB)
    return LIB


def build_checked(force: bool = False, verbose: bool = False) -> Path:
    """The same library with the kernels' index invariants asserted
    (-DSPK_CHECKED: SPK_CHECK traps).  compute-sanitizer is closed on the GPU
    pool; tests/test_checked_build.py runs GPU tests against this build
    (SPIKECAM_B200_LIB points the package at it)."""
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "spikecam_b200.h"]
    if not force and not _stale(CHECKED_LIB, deps):
        return CHECKED_LIB
    tmp = CHECKED_LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-DSPK_CHECKED", f"-I{ROOT / 'include'}", "-o", str(tmp), *map(str, sources())]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    tmp.replace(CHECKED_LIB)
    return CHECKED_LIB


def build_cpp(force: bool = False, verbose: bool = False) -> Path:
    """C++ drop-in (include/spikecam/b200.hpp) over the C-ABI: g++ only, linked
    against libspikecam_b200.so with an $ORIGIN rpath (no CUDA runtime of its own)."""
    lib = build_library(force=force, verbose=verbose)
    srcs = sorted((PKG / "cpp").glob("*.cpp"))
    deps = srcs + [ROOT / "include" / "spikecam" / "b200.hpp", ROOT / "include" / "spikecam_b200.h", lib]
    if not force and not _stale(CPP_LIB, deps):
        return CPP_LIB
    tmp = CPP_LIB.with_suffix(".so.tmp")
    cmd = [CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           "-o", str(tmp), *map(str, srcs), f"-L{PKG}", "-lspikecam_b200", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    tmp.replace(CPP_LIB)
    return CPP_LIB


def build_cpp_program(src: Path, out: Path, verbose: bool = False) -> Path:
    """A C++ program against the drop-in (tests/native/*.cpp)."""
    lib = build_cpp(verbose=verbose)
    if not _stale(out, [src, lib, ROOT / "include" / "spikecam" / "b200.hpp"]):
        return out
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", f"-I{ROOT / 'include'}", "-o", str(out), str(src),
           f"-L{PKG}", "-lspikecam_cpp", "-lspikecam_b200", f"-Wl,-rpath,{PKG}"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
    print(build_cpp(force=True, verbose=True))
    print(build_checked(force=True, verbose=True))
