"""Second CPU oracle: numpy/LAPACK restatement, one observation at a time.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Follows the algebra of
the reference's numpy core (/root/reference/pkg/src/vecchiagp/engine/fallback.py:
76-141: gather, covariance, derivative stack, dpotrf, triangular solves,
contraction) but is written against a family table that also carries the
families the reference lacks, so the C oracle's extension families can be
cross-checked by an arithmetically independent implementation.

Covariance definitions (relative nugget: diag = variance*(1+nugget) + jitter):
  exponential_isotropic   covariance.py:45-55      variance*exp(-r/range)
  exponential_anisotropic covariance.py:67-74      variance*exp(-||delta/range||)
  exponential_spacetime   derived: anisotropic with the spatial ranges tied
                          (theta = variance, range_space, range_time, nugget;
                          time is the last coordinate)
  matern15_isotropic      UNPINNED: variance*(1+x)exp(-x), x = r/range
  matern25_isotropic      UNPINNED: variance*(1+x+x^2/3)exp(-x)
  matern_isotropic        UNPINNED: theta = variance, range, smoothness, nugget;
                          variance * 2^(1-nu)/Gamma(nu) x^nu K_nu(x) with scipy.special.kv;
                          range derivative analytic (variance*nc*x^(nu+1) K_{nu-1}(x)/range),
                          smoothness derivative = central difference of step 1e-5
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import cholesky, solve_triangular

from .vecchia_oracle import acc_len


def _dist(pts):
    diff = pts[:, None, :] - pts[None, :, :]
    return np.sqrt((diff * diff).sum(axis=2))


MATERN_H = 1e-5


def _matern_corr(nu, x):
    from scipy.special import gammaln, kv
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        out = np.exp((1.0 - nu) * np.log(2.0) - gammaln(nu) + nu * np.log(x)) * kv(nu, x)
    return np.where(x < 1e-60, 1.0, out)


def cov_and_derivs(family, theta, pts, jitter=0.0):
    """K (k,k) and the derivative stack D (q,k,k) at local points pts (k,d)."""
    theta = np.asarray(theta, dtype=np.float64)
    k, d = pts.shape
    q = theta.shape[0]
    sig2, tau2 = theta[0], theta[-1]
    eye = np.eye(k)
    D = np.zeros((q, k, k))
    if family == "matern_isotropic":
        from scipy.special import gammaln, kv
        rho, nu = theta[1], theta[2]
        x = _dist(pts) / rho
        corr = _matern_corr(nu, x)
        with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
            drho = np.exp((1.0 - nu) * np.log(2.0) - gammaln(nu) + (nu + 1.0) * np.log(x)) * kv(nu - 1.0, x) / rho
        D[1] = sig2 * np.where(x < 1e-60, 0.0, drho)
        D[2] = sig2 * (_matern_corr(nu + MATERN_H, x) - _matern_corr(nu - MATERN_H, x)) / (2.0 * MATERN_H)
    elif family in ("exponential_isotropic", "exponential_sphere", "matern15_isotropic", "matern25_isotropic"):
        rho = theta[1]
        x = _dist(pts) / rho
        e = np.exp(-x)
        if family == "matern15_isotropic":
            corr = (1.0 + x) * e
            dcorr = x * x * e / rho
        elif family == "matern25_isotropic":
            corr = (1.0 + x + x * x / 3.0) * e
            dcorr = x * x * (1.0 + x) * e / (3.0 * rho)
        else:
            corr = e
            dcorr = x * e / rho
        D[1] = sig2 * dcorr
    elif family in ("exponential_anisotropic", "exponential_spacetime"):
        if family == "exponential_spacetime":
            rho = np.concatenate([np.full(d - 1, theta[1]), [theta[2]]])
        else:
            rho = theta[1:1 + d]
        delta = pts[:, None, :] - pts[None, :, :]
        s = np.sqrt(((delta / rho) ** 2).sum(axis=2))
        corr = np.exp(-s)
        with np.errstate(invalid="ignore", divide="ignore"):
            per_axis = [np.where(s == 0.0, 0.0, sig2 * corr * delta[:, :, a] ** 2 / (rho[a] ** 3 * s))
                        for a in range(d)]
        if family == "exponential_spacetime":
            D[1] = sum(per_axis[:-1])
            D[2] = per_axis[-1]
        else:
            for a in range(d):
                D[1 + a] = per_axis[a]
    else:
        raise KeyError(family)
    corr = corr.copy()
    np.fill_diagonal(corr, 1.0)
    K = sig2 * corr + sig2 * tau2 * eye + jitter * eye
    D[0] = corr + tau2 * eye
    for j in range(1, q - 1):
        np.fill_diagonal(D[j], 0.0)
    D[q - 1] = sig2 * eye
    return K, D


def contribution(i, y, X, locs, nn, family, theta, jitter=0.0):
    """Flat accumulator vector (L,) of observation i."""
    row = nn[i]
    g = row[row >= 0][::-1]
    pts, Xs, ys = locs[g], X[g], y[g]
    k, p = Xs.shape
    q = len(theta)
    K, D = cov_and_derivs(family, theta, pts, jitter)
    B = cholesky(K, lower=True)
    z = solve_triangular(B, ys, lower=True)
    W = solve_triangular(B, Xs, lower=True)
    e_last = np.zeros(k)
    e_last[-1] = 1.0
    u = solve_triangular(B, e_last, lower=True, trans="T")
    C = solve_triangular(B, (D @ u).T, lower=True)      # (k, q)
    e = k - 1
    ze, we, ce = z[e], W[e], C[e]
    zc = z @ C
    Wc = W.T @ C
    wewe = np.outer(we, we)
    pieces = [
        np.array([2.0 * np.log(B[e, e])]), np.array([ze * ze]), wewe.ravel(), (ze * we).ravel(),
        ce.copy(), ce * ze * ze - 2.0 * ze * zc,
        (ze * we[:, None] * ce[None, :] - ze * Wc - np.outer(we, zc)).ravel(),
        (ce[None, None, :] * wewe[:, :, None] - Wc[:, None, :] * we[None, :, None]
         - we[:, None, None] * Wc[None, :, :]).ravel(),
        (C.T @ C - 0.5 * np.outer(ce, ce)).ravel(),
    ]
    out = np.concatenate(pieces)
    assert out.shape[0] == acc_len(p, q)
    return out


def run(y, X, locs, nn, family, theta, jitter=0.0, i0=0, i1=None):
    y = np.asarray(y, dtype=np.float64).ravel()
    X = np.asarray(X, dtype=np.float64).reshape(y.shape[0], -1)
    locs = np.asarray(locs, dtype=np.float64).reshape(y.shape[0], -1)
    nn = np.asarray(nn)
    i1 = y.shape[0] if i1 is None else i1
    tot = np.zeros(acc_len(X.shape[1], len(theta)))
    for i in range(i0, i1):
        tot += contribution(i, y, X, locs, nn, family, theta, jitter)
    return tot


def dense_loglik(family, theta, y, X, locs):
    """Exact profiled Gaussian loglik from the full covariance (small n only);
    restates /root/reference/pkg/src/vecchiagp/oracle.py:40-68."""
    K, _ = cov_and_derivs(family, theta, np.asarray(locs, dtype=np.float64))
    L = cholesky(K, lower=True)
    hX = solve_triangular(L, X, lower=True)
    hy = solve_triangular(L, y, lower=True)
    beta = np.linalg.solve(hX.T @ hX, hX.T @ hy)
    r = hy - hX @ beta
    n = len(y)
    return -0.5 * (n * np.log(2 * np.pi) + 2.0 * np.log(np.diag(L)).sum() + r @ r), beta


def simulate_nn_gp(family, theta, beta, locs, X, nn, seed):
    """Sequential conditional draw from the neighbour-conditioned model -- restates the reference's
    oracle.simulate_nn_gp (/root/reference/pkg/src/vecchiagp/oracle.py:102-140) for every family of this
    package (locs are WORKING coordinates; the local matrix comes from cov_and_derivs, nugget on the diagonal).
    Pure-Python loop: small cases only."""
    theta = np.asarray(theta, dtype=np.float64)
    locs = np.atleast_2d(np.asarray(locs, dtype=np.float64))
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    n = locs.shape[0]
    xi = np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
    mean = X @ np.atleast_1d(beta)
    y = np.empty(n)
    var_prior = theta[0] * (1.0 + theta[-1])
    for i in range(n):
        row = nn[i]
        row = row[row >= 0]
        nbrs = row[1:][::-1]
        k = nbrs.shape[0]
        if k == 0:
            y[i] = mean[i] + np.sqrt(var_prior) * xi[i]
            continue
        K, _ = cov_and_derivs(family, theta, np.vstack([locs[nbrs], locs[i]]))
        L = cholesky(K[:k, :k], lower=True)
        w = solve_triangular(L, K[:k, k], lower=True)
        cond_mean = mean[i] + w @ solve_triangular(L, y[nbrs] - mean[nbrs], lower=True)
        y[i] = cond_mean + np.sqrt(max(var_prior - w @ w, 0.0)) * xi[i]
    return y

