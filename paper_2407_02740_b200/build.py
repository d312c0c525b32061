"""In-tree build of the native libraries (no JIT cache: the .so files live in
``paper_2407_02740_b200/lib/`` so they travel with the repository snapshot).

    libvecchia_b200.so  nvcc, sm_100a only: CUDA kernels + the C ABI of include/vecchia_b200.h
    libvecchia_host.so  g++ -ffp-contract=off -fopenmp: host ordered-neighbor search
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
CUDA_LIB = LIBDIR / "libvecchia_b200.so"
HOST_LIB = LIBDIR / "libvecchia_host.so"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def _newer(target: Path, sources) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(s.stat().st_mtime <= t for s in sources)


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _gxx() -> str:
    # the image's default /opt/gcc cannot link -fopenmp (no libgomp.spec); /usr/bin/g++ can
    for cand in (os.environ.get("VB200_CXX"), "/usr/bin/g++", shutil.which("g++")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("g++ not found")


def build_cuda(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    """Compile csrc/vecchia_b200.cu and every csrc/gen/tiled_part_*.cu to objects (in parallel)
    and link them into lib/libvecchia_b200.so.  sm_100a only, -lineinfo for ncu source pages."""
    from concurrent.futures import ThreadPoolExecutor

    headers = sorted(CSRC.glob("*.cuh")) + sorted((CSRC / "gen").glob("*.inc")) + [ROOT / "include" / "vecchia_b200.h"]
    units = ([CSRC / "vecchia_b200.cu"] + sorted((CSRC / "gen").glob("tiled_part_*.cu"))
             + sorted((CSRC / "gen").glob("krige_part_*.cu")))
    if not force and _newer(CUDA_LIB, headers + units):
        return CUDA_LIB
    LIBDIR.mkdir(exist_ok=True)
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
             "-I", str(ROOT / "include")]
    if verbose:
        flags.append("-Xptxas=-v")
    flags += os.environ.get("VB200_NVCC_FLAGS", "").split()  # development knob (e.g. -DTILED_WPB=2)

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if force or not _newer(obj, headers + [src]):
            subprocess.run([nvcc, *flags, "-c", str(src), "-o", str(obj)], check=True)
        return obj

    jobs = jobs or min(len(units), os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=jobs) as pool:
        objs = list(pool.map(compile_one, units))
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(CUDA_LIB),
                    *map(str, objs)], check=True)
    return CUDA_LIB


def build_host(force: bool = False) -> Path:
    sources = [CSRC / "host_neighbors.cpp"]
    if not force and _newer(HOST_LIB, sources):
        return HOST_LIB
    LIBDIR.mkdir(exist_ok=True)
    cmd = [_gxx(), "-O3", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
           "-o", str(HOST_LIB), *map(str, sources)]
    subprocess.run(cmd, check=True)
    return HOST_LIB


def build_all(force: bool = False, verbose: bool = False):
    return build_cuda(force, verbose), build_host(force)


if __name__ == "__main__":
    import sys
    print(*build_all(force="--force" in sys.argv, verbose="-v" in sys.argv), sep="\n")
