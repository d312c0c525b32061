#!/usr/bin/env python
"""General-order Matern on the GPU against the CPU oracle (central-difference smoothness derivative) at several
smoothness values, including near-integer / half-integer orders where mu is tiny or the order shift changes nup.

    [VB200_LIB=...] python tools/matern_check.py
"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine
from oracle import vecchia_oracle as vo

rng = np.random.default_rng(11)
n, m = 3000, 30
locs = rng.uniform(0, 1, (n, 2))
y = rng.normal(size=n)
X = np.ones((n, 1))
nn = vg.find_ordered_neighbors(locs, m)
worst = 0.0
for nu in (0.3, 0.5, 0.8, 1.0, 1.0 + 3e-6, 1.5, 1.5 - 4e-6, 2.0001, 2.5, 3.7, 0.05):
    for rho in (0.08, 0.6, 0.004):
        theta = np.array([1.3, rho, nu, 0.1])
        want = vo.run(y, X, locs, nn.idx, "matern_isotropic", theta)
        with engine.DeviceProblem(vg.Dataset(y, X, locs), nn, "matern_isotropic") as prob:
            got = prob.totals(theta)
            name = prob.last_kernel_name
        scale = np.maximum(np.abs(want), 1e-300)
        # compare field-wise against the largest entry of the same block of accumulators (coarse: whole vector scale per entry)
        rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-6 * np.abs(want).max())
        worst = max(worst, rel.max())
        print(f"nu={nu:<10} rho={rho:<6} max rel diff {rel.max():.2e} at {int(rel.argmax())}  ({name})")
print("worst", worst)
