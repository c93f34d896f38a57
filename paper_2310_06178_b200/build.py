"""Build the in-tree C-ABI CUDA library (sm_100a) with nvcc.

    python -m paper_2310_06178_b200.build [--force] [-v]

Produces paper_2310_06178_b200/_lib/libmsgemm_b200.so (git-ignored; it
travels to the GPU box with the repo snapshot).  nvcc cross-compiles here
without a GPU.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OUTDIR = PKG / "_lib"
LIB = OUTDIR / "libmsgemm_b200.so"
# debug variant (device-side bounds asserts + race-provoking barrier jitter,
# csrc/msg_common.cuh MSG_DEBUG_CHECKS); loaded when MSG_LIB_VARIANT=debug
LIB_DEBUG = OUTDIR / "libmsgemm_b200_debug.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden", "-I", str(INCLUDE), "-I", str(CSRC),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
          debug: bool = False, defines: tuple = (), name: str | None = None) -> Path:
    """defines/name: an experiment build (-D flags) into _lib/<name>.so."""
    lib = OUTDIR / f"{name}.so" if name else (LIB_DEBUG if debug else LIB)
    if not force and not _stale(lib):
        return lib
    OUTDIR.mkdir(exist_ok=True)
    objdir = OUTDIR / (f"obj_{name}" if name else ("obj_debug" if debug else "obj"))
    objdir.mkdir(exist_ok=True)
    cc = nvcc()
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    if debug:
        extra += ["-DMSG_DEBUG_CHECKS=1"]
    extra += [f"-D{d}" for d in defines]

    shared = [p for p in list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]]
    newest_shared = max(p.stat().st_mtime for p in shared)

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if (not force and not ptxas_verbose and obj.exists()
                and obj.stat().st_mtime > max(src.stat().st_mtime, newest_shared)):
            return obj  # up to date: only changed sources are recompiled
        cmd = [cc, *NVCC_FLAGS, *extra, "-dc" if False else "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
        if (verbose or ptxas_verbose) and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print ptxas register/smem usage")
    ap.add_argument("--debug", action="store_true", help="build the debug-checks variant")
    a = ap.parse_args()
    print(build(force=a.force or a.ptxas, verbose=a.verbose, ptxas_verbose=a.ptxas, debug=a.debug))


if __name__ == "__main__":
    main()
