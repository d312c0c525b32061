"""ctypes wrapper over the C oracle (``oracle/vecchia_oracle.c``).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The accumulator layout
(one flat vector of L doubles) follows the reference's slot order
(/root/reference/pkg/src/vecchiagp/engine/__init__.py:141-152):
logdet, ysy, xsx[p,p], ysx[p], dlogdet[q], dysy[q], dysx[p,q], dxsx[p,p,q],
ainfo[q,q].
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libvecchia_oracle.so"

FAMILY_CODES = {
    "exponential_isotropic": 0,
    "exponential_sphere": 0,  # isotropic kernel on embedded coordinates
    "exponential_anisotropic": 1,
    "exponential_spacetime": 2,
    "matern15_isotropic": 3,
    "matern25_isotropic": 4,
    "matern_isotropic": 5,  # general order: variance, range, smoothness, nugget
}

_c_dp = ctypes.POINTER(ctypes.c_double)
_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_i32p = ctypes.POINTER(ctypes.c_int32)
_lib = None


def build(force: bool = False) -> Path:
    """Compile the C oracle in place (gcc, flags in oracle/Makefile)."""
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "vecchia_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.vo_acc_len.restype = ctypes.c_int
        L.vo_acc_len.argtypes = [ctypes.c_int, ctypes.c_int]
        L.vo_max_threads.restype = ctypes.c_int
        L.vo_run.restype = ctypes.c_int
        L.vo_run.argtypes = [
            _c_dp, _c_dp, _c_dp, _c_i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _c_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int, ctypes.c_int, _c_dp, _c_i64p, _c_i32p,
        ]
        L.vo_observations.restype = ctypes.c_int64
        L.vo_observations.argtypes = [
            _c_dp, _c_dp, _c_dp, _c_i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _c_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int, _c_dp, _c_i32p,
        ]
        L.vo_krige.restype = ctypes.c_int64
        L.vo_krige.argtypes = [_c_dp, _c_dp, _c_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _c_dp, ctypes.c_int,
                               ctypes.c_int, _c_dp, _c_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               _c_dp, _c_dp, _c_i64p]
        L.vo_bessel_k.restype = ctypes.c_double
        L.vo_bessel_k.argtypes = [ctypes.c_double, ctypes.c_double]
        L.vo_neighbor_scan.restype = None
        L.vo_neighbor_scan.argtypes = [_c_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64p]
        _lib = L
    return _lib


def acc_len(p: int, q: int) -> int:
    return (1 + q) * (2 + p + p * p) + q * q


def split_acc(v: np.ndarray, p: int, q: int) -> dict:
    """Flat accumulator vector(s) (..., L) -> dict of named arrays."""
    v = np.asarray(v)
    lead = v.shape[:-1]
    o = 0

    def take(shape):
        nonlocal o
        size = int(np.prod(shape)) if shape else 1
        out = v[..., o:o + size].reshape(lead + tuple(shape))
        o += size
        return out

    parts = {
        "logdet": take(()), "ysy": take(()), "xsx": take((p, p)), "ysx": take((p,)),
        "dlogdet": take((q,)), "dysy": take((q,)), "dysx": take((p, q)),
        "dxsx": take((p, p, q)), "ainfo": take((q, q)),
    }
    assert o == acc_len(p, q)
    return parts


def _prep(y, X, locs, nn, theta):
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    locs = np.ascontiguousarray(locs, dtype=np.float64)
    if locs.ndim == 1:
        locs = locs.reshape(-1, 1)
    nn = np.ascontiguousarray(nn, dtype=np.int64)
    theta = np.ascontiguousarray(theta, dtype=np.float64).ravel()
    return y, X, locs, nn, theta


def _dp(a):
    return a.ctypes.data_as(_c_dp)


class OracleNotPositiveDefinite(Exception):
    def __init__(self, pivot, observation):
        super().__init__(f"observation {observation}: pivot {pivot}")
        self.pivot = int(pivot)
        self.observation = int(observation)


def run(y, X, locs, nn, family, theta, jitter=0.0, i0=0, i1=None, workers=None, deterministic=True):
    """Totals of the L accumulators over observations [i0, i1) (flat vector)."""
    y, X, locs, nn, theta = _prep(y, X, locs, nn, theta)
    n, p, d, mp1, q = y.shape[0], X.shape[1], locs.shape[1], nn.shape[1], theta.shape[0]
    if i1 is None:
        i1 = n
    workers = workers or os.cpu_count() or 1
    out = np.zeros(acc_len(p, q))
    first = ctypes.c_int64(-1)
    piv = ctypes.c_int32(-1)
    code = FAMILY_CODES[family] if isinstance(family, str) else int(family)
    rc = lib().vo_run(_dp(y), _dp(X), _dp(locs), nn.ctypes.data_as(_c_i64p), n, p, d, mp1,
                      _dp(theta), q, code, float(jitter), int(i0), int(i1), int(workers),
                      int(bool(deterministic)), _dp(out), ctypes.byref(first), ctypes.byref(piv))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    if first.value >= 0:
        raise OracleNotPositiveDefinite(piv.value, first.value)
    return out


def observations(y, X, locs, nn, family, theta, jitter=0.0, i0=0, i1=None, workers=1):
    """Per-observation accumulator rows, shape (i1-i0, L), plus the fail vector."""
    y, X, locs, nn, theta = _prep(y, X, locs, nn, theta)
    n, p, d, mp1, q = y.shape[0], X.shape[1], locs.shape[1], nn.shape[1], theta.shape[0]
    if i1 is None:
        i1 = n
    L = acc_len(p, q)
    slots = np.zeros((i1 - i0, L))
    fail = np.zeros(i1 - i0, dtype=np.int32)
    code = FAMILY_CODES[family] if isinstance(family, str) else int(family)
    lib().vo_observations(_dp(y), _dp(X), _dp(locs), nn.ctypes.data_as(_c_i64p), n, p, d, mp1,
                          _dp(theta), q, code, float(jitter), int(i0), int(i1), int(workers),
                          _dp(slots), fail.ctypes.data_as(_c_i32p))
    return slots, fail


def neighbor_scan(locs, m, workers=None):
    """Exhaustive ordered nearest-predecessor table (n, m+1), -1 padded."""
    locs = np.ascontiguousarray(np.atleast_2d(locs), dtype=np.float64)
    n, d = locs.shape
    m = min(int(m), max(n - 1, 1))
    out = np.full((n, m + 1), -1, dtype=np.int64)
    lib().vo_neighbor_scan(_dp(locs), n, d, m, int(workers or os.cpu_count() or 1),
                           out.ctypes.data_as(_c_i64p))
    return out


def krige(y, X, locs, family, theta, beta, locs_star, X_star, m_pred, latent=False, workers=None):
    """Kriging mean / sd at locs_star (working coordinates) -- restates the reference's predict.krige
    (predict.py:35-90).  Returns (mean, sd, neighbor indices)."""
    y, X, locs, _, theta = _prep(y, X, locs, np.zeros((1, 1), dtype=np.int64), theta)
    beta = np.ascontiguousarray(beta, dtype=np.float64).ravel()
    locs_star = np.ascontiguousarray(np.atleast_2d(locs_star), dtype=np.float64)
    X_star = np.ascontiguousarray(np.atleast_2d(X_star), dtype=np.float64)
    n, p, d, q, ns = y.shape[0], X.shape[1], locs.shape[1], theta.shape[0], locs_star.shape[0]
    mean = np.zeros(ns)
    var = np.zeros(ns)
    nbrs = np.zeros((ns, m_pred), dtype=np.int64)
    code = FAMILY_CODES[family] if isinstance(family, str) else int(family)
    bad = lib().vo_krige(_dp(y), _dp(X), _dp(locs), n, p, d, _dp(theta), q, code, _dp(beta), _dp(locs_star), ns,
                         int(m_pred), int(bool(latent)), int(workers or os.cpu_count() or 1), _dp(mean), _dp(var),
                         nbrs.ctypes.data_as(_c_i64p))
    if bad:
        raise OracleNotPositiveDefinite(-1, bad - 1)
    return X_star @ beta + mean, np.sqrt(np.maximum(var, 0.0)), nbrs


LOG_2PI = float(np.log(2.0 * np.pi))


def assemble(totals, n, p, q):
    """Profiled loglik / beta / grad / info from accumulator totals.

    Restates /root/reference/pkg/src/vecchiagp/inference.py:42-68 with numpy only.
    """
    P = split_acc(np.asarray(totals, dtype=np.float64), p, q)
    chol = np.linalg.cholesky(P["xsx"])
    beta = np.linalg.solve(chol.T, np.linalg.solve(chol, P["ysx"]))
    quad = float(P["ysy"]) - 2.0 * beta @ P["ysx"] + beta @ P["xsx"] @ beta
    loglik = -0.5 * (n * LOG_2PI + float(P["logdet"]) + quad)
    grad = -0.5 * (P["dlogdet"] + P["dysy"] - 2.0 * beta @ P["dysx"]
                   + np.einsum("a,abj,b->j", beta, P["dxsx"], beta))
    return {"loglik": float(loglik), "beta": beta, "grad": grad, "info": P["ainfo"], "betainfo": P["xsx"]}
