import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import _cabi
from paper_2407_02740_b200.engine import DeviceProblem
from oracle import vecchia_oracle as vo
from conftest import make_instance
names = {0: "exponential_isotropic", 1: "exponential_anisotropic", 2: "exponential_spacetime", 3: "matern15_isotropic", 4: "matern25_isotropic", 5: "matern_isotropic"}
rng = np.random.default_rng(77)
worst = []
for g, s_, cap, fam, d, p in _cabi.tiled_instances():
    family = names[fam]; q = _cabi.load().vb200_family_nparms(fam, d)
    theta = np.concatenate([[1.3], rng.uniform(0.15, 0.4, q - 2), [0.08]])
    if fam == 5: theta[2] = rng.uniform(0.4, 2.6)
    for m in sorted({cap - 2, max(2, cap // 2 - 3)}):
        n = 3 * cap + 40
        y, X, locs, _ = make_instance(1000 + cap + d + p + m, n, d, p)
        nn = vg.find_ordered_neighbors(locs, m)
        want = vo.run(y, X, locs, nn.idx, family, theta)
        with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
            prob.set_layout("tiled_reg"); got = prob.totals(theta)
            prob.set_layout("warp_smem"); got2 = prob.totals(theta)
        G, W, G2 = vo.split_acc(got, p, q), vo.split_acc(want, p, q), vo.split_acc(got2, p, q)
        for k in W:
            sc = max(float(np.max(np.abs(W[k]))), 1e-300)
            e = float(np.max(np.abs(np.asarray(G[k]) - np.asarray(W[k])))) / sc
            e2 = float(np.max(np.abs(np.asarray(G2[k]) - np.asarray(W[k])))) / sc
            worst.append((e, e2, k, (g, s_, cap, family, d, p, m)))
worst.sort(reverse=True)
for w in worst[:8]: print(w)
