"""Small workload for compute-sanitizer (memcheck / racecheck): every layout, a few tiers, kriging."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200.engine import DeviceProblem

rng = np.random.default_rng(0)
for family, d, p, theta, m in [("matern15_isotropic", 2, 1, [1.0, 0.1, 0.1], 30), ("exponential_spacetime", 3, 1, [1, .2, .5, .1], 30),
                               ("exponential_isotropic", 2, 1, [1.0, 0.1, 0.1], 10), ("matern15_isotropic", 2, 1, [1.0, 0.1, 0.1], 40),
                               ("matern_isotropic", 2, 1, [1.0, 0.1, 0.8, 0.1], 20), ("matern15_isotropic", 3, 4, [1.0, 0.2, 0.1], 30),
                               # exact-size tiers (static padding rows): m = 20 / 50 / 60, and a ragged m on each
                               ("matern15_isotropic", 2, 1, [1.0, 0.1, 0.1], 20), ("matern15_isotropic", 2, 1, [1.0, 0.1, 0.1], 50),
                               ("matern15_isotropic", 2, 1, [1.0, 0.1, 0.1], 60), ("exponential_isotropic", 2, 4, [1.0, 0.1, 0.1], 37),
                               ("matern25_isotropic", 2, 1, [1.0, 0.1, 0.1], 15), ("exponential_spacetime", 3, 4, [1, .2, .5, .1], 25),
                               ("matern_isotropic", 3, 1, [1.0, 0.3, 2.2, 0.1], 40)]:
    n = 600
    locs = rng.uniform(0, 1, (n, d)); y = rng.normal(size=n)
    X = np.column_stack([np.ones(n)] + [rng.normal(size=n) for _ in range(p - 1)])
    nn = vg.find_ordered_neighbors(locs, m)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        for layout in ("tiled_reg", "warp_smem"):
            prob.set_layout(layout)
            tot = prob.totals(np.array(theta))
            print(family, m, layout, prob.last_kernel_name, float(tot[0]))
# narrowed (int32) chunked upload of the neighbor table + device-side widening
locs = rng.uniform(0, 1, (901, 2))
nn = vg.find_ordered_neighbors(locs, 30)
with DeviceProblem(vg.Dataset(rng.normal(size=901), np.ones((901, 1)), locs), nn, "matern15_isotropic", upload_chunks=3,
                   upload_narrow=True) as prob:
    print("narrowed upload", float(prob.totals(np.array([1.0, 0.1, 0.1]))[0]))
cov = vg.CovarianceParameters("matern15_isotropic", [1.0, 0.1, 0.1])
fr = vg.FitResult(theta_hat=cov, beta_hat=np.array([0.1]), beta_cov=np.eye(1), loglik_trace=[0.0], fisher_info=np.eye(3), iterations=0, converged=True)
locs = rng.uniform(0, 1, (800, 2))
ps = vg.krige(fr, vg.Dataset(rng.normal(size=800), np.ones((800, 1)), locs), rng.uniform(0, 1, (100, 2)), np.ones((100, 1)), m_pred=60)
print("krige", ps.mean[:2], ps.sd[:2])
