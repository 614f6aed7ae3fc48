"""Builds libpot3d.so in-tree with nvcc for sm_100a (no JIT cache, no pip install).

Compiled here on the CPU box by __graft_entry__.build(); the .so travels to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpot3d.so"
SOURCES = ["kernels.cu", "passes.cu", "cg1.cu", "poly.cu", "pc2.cu", "abi.cu"]
HEADERS = ["pot3d_internal.cuh", "device_common.cuh", "pass_common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        base = Path(list(spec.submodule_search_locations)[0])
        inc, lib = base / "include", base / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return inc, lib
    return Path("/usr/include"), Path("/usr/lib/x86_64-linux-gnu")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "pot3d.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Build libpot3d.so (or a tuning variant `out` with extra -D `defines`).  Processes
    that build at once (the ranks of a torchrun job finding a stale library) take turns
    on a file lock: the object files are shared, and the later ones find it fresh."""
    import fcntl

    target = LIB if out is None else Path(out)
    if out is None and not force and not _stale():
        return LIB
    (PKG / "build").mkdir(parents=True, exist_ok=True)
    with open(PKG / "build" / ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if out is None and not force and not _stale():
            return LIB
        return _build_locked(target, verbose, defines, out)


def _build_locked(target: Path, verbose: bool, defines, out) -> Path:
    nvcc = os.environ.get("NVCC", "nvcc")
    inc, libdir = nccl_dirs()
    objs = []
    tmpdir = PKG / "build" / (target.stem if out is not None else "")
    tmpdir.mkdir(parents=True, exist_ok=True)
    common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *ARCH,
              f"-I{inc}", f"-I{ROOT / 'include'}", "-Xptxas", "-v" if verbose else "-O3",
              *[f"-D{d}" for d in defines]]
    for s in SOURCES:
        o = tmpdir / (Path(s).stem + ".o")
        cmd = [nvcc, *common, "-c", str(CSRC / s), "-o", str(o)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(str(o))
    tmp = target.with_suffix(f".so.tmp{os.getpid()}")
    link = [nvcc, "-shared", *ARCH, "-o", str(tmp), *objs, f"-L{libdir}", "-lnccl",
            f"-Xlinker", f"-rpath={libdir}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libpot3d.so failed")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
