#!/usr/bin/env python
"""Time experiment variants (tools/build_variant.py) of the headline kernel on the GPU, one subprocess per
variant (the library is chosen at load time by VB200_LIB).

    python tools/time_variants.py [--names a,b,c] [--pads 0,40000] [--clocks] [extra args for the child]
"""
import argparse, json, os, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
VAR = ROOT / "paper_2407_02740_b200" / "lib" / "variants"

CHILD = r'''
import sys, json, ctypes, os
sys.path.insert(0, %(root)r)
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine, _cabi
from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows
import bench
n, m, d, p, fam = %(n)d, %(m)d, %(d)d, %(p)d, %(family)r
y, X, locs = bench.make_workload(n, d, p)
nn = find_ordered_neighbor_rows(locs, m, 0, n)
q = vg.covariance_registry(fam).nparms(d)
theta = np.array([1.0] + [0.05] * (q - 2) + [0.1])
lib = _cabi.load()
with engine.DeviceProblem(vg.Dataset(y, X, locs), vg.NeighborArray(nn), fam) as prob:
    prob.enable_timing(True)
    ms = []
    tot = None
    for _ in range(%(reps)d + 3):
        tot = prob.totals(theta)
        ms.append(prob.last_kernel_ms())
    ms = np.array(ms[3:])
    out = {"ms_median": float(np.median(ms)), "ms_min": float(ms.min()), "kernel": prob.last_kernel_name,
           "loglik_parts": [float(tot[0]), float(tot[1])]}
    if %(clocks)d:
        fn = lib.vb200_debug_clocks
        fn.restype = ctypes.c_int
        buf = (ctypes.c_ulonglong * 160)()
        fn(buf, 160, 1)
        prob.totals(theta)
        fn(buf, 160, 1)
        out["clocks"] = [int(v) for v in buf]
    print("RESULT " + json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--names", default="")
    ap.add_argument("--pads", default="0")
    ap.add_argument("--clocks", action="store_true")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--p", type=int, default=1)
    ap.add_argument("--family", default="matern15_isotropic")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    names = [x for x in a.names.split(",") if x] or sorted(p.stem[6:] for p in VAR.glob("libvb_*.so"))
    results = {}
    for name in names:
        lib = VAR / f"libvb_{name}.so"
        for pad in [int(x) for x in a.pads.split(",")]:
            env = dict(os.environ, VB200_LIB=str(lib))
            if pad:
                env["VB200_TILED_SMEM_PAD"] = str(pad)
            code = CHILD % dict(root=str(ROOT), n=a.n, m=a.m, d=a.d, p=a.p, family=a.family, reps=a.reps,
                                clocks=int(a.clocks))
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            res = None
            for line in r.stdout.splitlines():
                if line.startswith("RESULT "):
                    res = json.loads(line[7:])
            if res is None:
                res = {"error": (r.stderr or r.stdout)[-600:]}
            results[f"{name}@pad{pad}"] = res
            print(name, pad, json.dumps(res), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
