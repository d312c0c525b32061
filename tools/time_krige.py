"""Kriging throughput on the GPU box: predictions/s of vg.krige (host neighbour query + vb200_krige)
and of the CPU oracle on the same points."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200.preprocess import find_nearest_training
from oracle import vecchia_oracle as vo

n, npred, m_pred = 1 << 20, 1 << 18, 60
rng = np.random.default_rng(1)
locs = rng.uniform(0, 1, (n, 2)); y = rng.normal(size=n); X = np.ones((n, 1))
star = rng.uniform(0, 1, (npred, 2)); Xs = np.ones((npred, 1))
cov = vg.CovarianceParameters("matern15_isotropic", [1.0, 0.05, 0.1])
fr = vg.FitResult(theta_hat=cov, beta_hat=np.array([0.1]), beta_cov=np.eye(1), loglik_trace=[0.0], fisher_info=np.eye(3),
                  iterations=0, converged=True)
train = vg.Dataset(y, X, locs)
t0 = time.perf_counter(); nb = find_nearest_training(locs, star, m_pred); t_q = time.perf_counter() - t0
for rep in range(3):
    t0 = time.perf_counter(); ps = vg.krige(fr, train, star, Xs, m_pred=m_pred); t_k = time.perf_counter() - t0
print(f"neighbour query {t_q:.3f} s; vg.krige total {t_k:.3f} s = {npred / t_k / 1e6:.2f} M predictions/s (m_pred={m_pred}, n_train=2^20)")
sub = 1 << 13
t0 = time.perf_counter(); mean, sd, _ = vo.krige(y, X, locs, "matern15_isotropic", cov.theta, fr.beta_hat, star[:sub], Xs[:sub], m_pred)
t_o = time.perf_counter() - t0
print(f"CPU oracle (exhaustive neighbour scan + Cholesky, all cores): {sub / t_o:.0f} predictions/s; max |mean diff| {np.max(np.abs(mean - ps.mean[:sub])):.2e}")
