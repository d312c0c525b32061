import time, sys, numpy as np
sys.path.insert(0, '.')
import paper_2407_02740_b200 as vg
n, m = 1 << 20, 30
rng = np.random.default_rng(2); locs = rng.uniform(0, 1, (n, 2))
t=time.time(); nn = vg.find_ordered_neighbors(locs, m); t_nn=time.time()-t
t=time.time(); order, lp = vg.dependency_levels(nn); t_lev=time.time()-t
cov = vg.CovarianceParameters("matern15_isotropic", [1.5, 0.05, 0.1])
X = np.ones((n, 1))
for rep in range(2):
    t=time.time(); y = vg.simulate_nn_gp(cov, [0.3], locs, X, nn, seed=9); t_sim=time.time()-t
print(f"n=2^20 m=30: neighbours {t_nn:.2f}s, levels {t_lev:.3f}s ({len(lp)-1} levels), simulate_nn_gp total {t_sim:.3f}s, var {y.var():.3f}")
