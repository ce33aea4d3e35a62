"""In-tree build of the native library for sm_100a.

    python -m paper_2104_13542_b200.build          # -> paper_2104_13542_b200/_mppi_b200.so

Each translation unit is compiled in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
one shared object exporting the C ABI of include/mppi_b200.h.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# MPPI_BUILD_TAG=<tag>: a variant build (e.g. with MPPI_NVCC_FLAGS=-DMPPI_DEBUG_TIMERS)
# next to the production library, loaded with MPPI_LIB for A/B runs
TAG = os.environ.get("MPPI_BUILD_TAG", "")
OUT = PKG / (f"_mppi_b200_{TAG}.so" if TAG else "_mppi_b200.so")
OBJ = ROOT / "build" / (f"obj-{TAG}" if TAG else "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}"] + os.environ.get("MPPI_NVCC_FLAGS", "").split()
SOURCES = ["mppi_abi.cu", "mppi_seam.cu", "mppi_launch_f32.cu", "mppi_launch_f64.cu", "mppi_train.cu"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(exe).exists():
        raise RuntimeError("nvcc not found")
    return exe


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "mppi_b200.h"]
    objs = []
    jobs = []
    for src in SOURCES:
        obj = OBJ / (Path(src).stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src] + headers):
            cmd = [nvcc(), *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                print(log, file=sys.stderr)
    if force or _stale(OUT, objs):
        link = [nvcc(), *ARCH, "-shared", "-o", str(OUT), *map(str, objs)]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {r.stdout}\n{r.stderr}")
    if not TAG:
        build_fast(force)
    return OUT


FAST_SRC = CSRC / "mppi_fast.c"


def fast_path() -> Path:
    import sysconfig

    return PKG / ("_mppi_fast" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_fast(force: bool = False) -> Path:
    """The CPython entry of the latency path (csrc/mppi_fast.c): a plain C
    extension that passes the caller's float64 state arrays to mppi_step."""
    import sysconfig

    out = fast_path()
    if force or _stale(out, [FAST_SRC]):
        cc = shutil.which("gcc") or "cc"
        cmd = [cc, "-O2", "-shared", "-fPIC", f"-I{sysconfig.get_paths()['include']}", str(FAST_SRC), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"cc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
