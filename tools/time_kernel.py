"""Time the main kernel (CUDA events inside the library) for the bench workload or a variant.
usage: python tools/time_kernel.py [--family F] [--m M] [--d D] [--p P] [--n N] [--layout L] [--reps R]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine
from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="matern15_isotropic"); ap.add_argument("--m", type=int, default=30)
ap.add_argument("--d", type=int, default=2); ap.add_argument("--p", type=int, default=1)
ap.add_argument("--n", type=int, default=1 << 20); ap.add_argument("--layout", default="auto")
ap.add_argument("--reps", type=int, default=10); ap.add_argument("--theta", type=float, nargs="+", default=None)
a = ap.parse_args()
y, X, locs = bench.make_workload(a.n, a.d, a.p)
nn = find_ordered_neighbor_rows(locs, a.m, 0, a.n)
fam = vg.covariance_registry(a.family)
q = fam.nparms(a.d)
theta = np.array(a.theta) if a.theta else np.array([1.0] + [0.05] * (q - 2) + [0.1])
with engine.DeviceProblem(vg.Dataset(y, X, locs), vg.NeighborArray(nn), a.family, layout=a.layout) as prob:
    prob.enable_timing(True)
    ms = []
    for _ in range(a.reps + 3):
        prob.totals(theta)
        ms.append(prob.last_kernel_ms())
    ms = np.array(ms[3:])
    F = bench.algorithmic_flops(a.family, a.d, a.p, q, a.m)["F_min"]
    print(f"{a.family} d={a.d} p={a.p} m={a.m} n={a.n} layout={prob.layout_for(q)} kernel={prob.last_kernel_name}: "
          f"median {np.median(ms):.3f} ms  min {ms.min():.3f} ms  {a.n / np.median(ms) / 1e3:.1f} Mobs/s  "
          f"{F * a.n / np.median(ms) / 1e9:.2f} TFLOP/s(alg)")
