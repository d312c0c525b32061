#!/usr/bin/env python
"""Build an EXPERIMENT variant of libvecchia_b200.so with a single translation unit of likelihood
instances (seconds instead of minutes) and arbitrary -D flags:

    python tools/build_variant.py NAME [--flags "-DTILED_CLOCKS -DTILED_PD=5"] [--inst "16,2,FAM_MATERN15,2,1;..."] [--pt]

writes paper_2407_02740_b200/lib/variants/libvb_NAME.so (git-ignored; travels to the GPU box).  Load it with
VB200_LIB=<path> (see _cabi.load).  Kriging / simulation kernels are not part of variant builds.
"""
import argparse, os, subprocess, sys, tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2407_02740_b200" / "csrc"
OUT = ROOT / "paper_2407_02740_b200" / "lib" / "variants"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--flags", default="")
    ap.add_argument("--inst", default="16,2,FAM_MATERN15,2,1")
    ap.add_argument("--pt", action="store_true", help="pair-table kernel variant for the listed instances")
    ap.add_argument("--header", default="../kernel_tiled.cuh")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    tmp = Path(tempfile.mkdtemp(prefix="vbvar_"))
    gen = CSRC / "gen"
    part = gen / f"_variant_{a.name}.cu"
    macro = "TILED_INST_PT" if a.pt else "TILED_INST"
    items = [tuple(x.strip() for x in it.split(",")) for it in a.inst.split(";") if it.strip()]
    lines = [f'#include "{a.header}"', "", "extern const TiledInstance kTiledPart0[] = {"]
    for it in items:
        m = macro
        if len(it) == 7:    # g,s,fam,d,p,TILED_INST_PTN,np
            m, it = it[5], it[:5] + it[6:]
        elif len(it) == 6:
            m, it = it[5], it[:5]
        lines.append(f"    {m}({', '.join(it)}),")
    lines += ["};", f"extern const int kTiledPart0Count = {len(items)};", ""]
    part.write_text("\n".join(lines))
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
             "-I", str(ROOT / "include"), "-DVB200_SINGLE_PART", "-DVB200_EXPERIMENTS"] + a.flags.split()
    if a.v:
        flags.append("-Xptxas=-v")
    try:
        procs = []
        objs = []
        for src in (CSRC / "vecchia_b200.cu", part):
            obj = tmp / (src.stem + ".o")
            objs.append(obj)
            procs.append(subprocess.Popen(["nvcc", *flags, "-c", str(src), "-o", str(obj)]))
        for pr in procs:
            if pr.wait() != 0:
                sys.exit(1)
        lib = OUT / f"libvb_{a.name}.so"
        subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(lib), *map(str, objs)],
                       check=True)
        print(lib)
    finally:
        part.unlink(missing_ok=True)


if __name__ == "__main__":
    main()
