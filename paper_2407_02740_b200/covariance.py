"""Covariance family registry: names, parameter layouts, device kernel codes.

Keeps the reference's registry surface (/root/reference/pkg/src/vecchiagp/covariance.py:
``covariance_registry`` :187-198, ``validate_parameters`` :201-217, ``CovarianceFamily``
with ``kernel_code / nparms / prepare_locs / matrix / derivatives / cross`` :125-176) and
adds the families BASELINE.json names that the reference lacks:

    exponential_isotropic    [variance, range, nugget]                 code 0
    exponential_anisotropic  [variance, range_1..range_d, nugget]      code 1
    exponential_sphere       lon/lat degrees -> unit sphere, then isotropic (code 0)
    exponential_spacetime    [variance, range_space, range_time, nugget], time = last
                             coordinate                                 code 2
    matern15_isotropic       [variance, range, nugget], nu = 3/2        code 3
    matern25_isotropic       [variance, range, nugget], nu = 5/2        code 4
    matern_isotropic         [variance, range, smoothness, nugget], general order (Bessel K on the
                             device by Temme's method; smoothness derivative by central difference)
                                                                        code 5

The nugget is relative: every diagonal entry is variance * (1 + nugget).
The dense ``matrix`` / ``derivatives`` / ``cross`` helpers below are small-n host
utilities (kriging, diagnostics); the likelihood path never uses them -- it runs in
the CUDA core (csrc/common.cuh ``pair_terms``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UnknownFamily
from .model import CovarianceParameters

KERNEL_ISOTROPIC = 0
KERNEL_ANISOTROPIC = 1
KERNEL_SPACETIME = 2
KERNEL_MATERN15 = 3
KERNEL_MATERN25 = 4
KERNEL_MATERN = 5
MATERN_NU_MIN, MATERN_NU_MAX = 2e-5, 60.0  # supported smoothness range of matern_isotropic
MATERN_H = 1e-5  # smoothness central-difference step (csrc/common.cuh VB_MATERN_H)

FAMILY_NAMES = (
    "exponential_isotropic",
    "exponential_anisotropic",
    "exponential_sphere",
    "exponential_spacetime",
    "matern15_isotropic",
    "matern25_isotropic",
    "matern_isotropic",
)

_CODES = {
    "exponential_isotropic": KERNEL_ISOTROPIC,
    "exponential_anisotropic": KERNEL_ANISOTROPIC,
    "exponential_sphere": KERNEL_ISOTROPIC,
    "exponential_spacetime": KERNEL_SPACETIME,
    "matern15_isotropic": KERNEL_MATERN15,
    "matern25_isotropic": KERNEL_MATERN25,
    "matern_isotropic": KERNEL_MATERN,
}


def _axis_ranges(name, theta, d):
    if name == "exponential_anisotropic":
        return np.asarray(theta[1:1 + d], dtype=np.float64)
    if name == "exponential_spacetime":
        return np.concatenate([np.full(d - 1, theta[1]), [theta[2]]])
    return np.full(d, theta[1], dtype=np.float64)


def _scaled_distance(a, b, rho):
    diff = (a[:, None, :] - b[None, :, :]) / rho
    return np.sqrt(np.einsum("ijk,ijk->ij", diff, diff)), diff


def _log_xk(order, power, x):
    """log( x^power K_order(x) ) in log space (exponentially scaled Bessel function): K_nu(x) overflows for large nu at
    small x while x^nu underflows, their product is O(1)."""
    from scipy.special import kve
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        return power * np.log(x) + np.log(kve(order, x)) - x


def _matern_corr(nu, x):
    from scipy.special import gammaln
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        out = np.exp((1.0 - nu) * np.log(2.0) - gammaln(nu) + _log_xk(nu, nu, x))
    return np.where(x < 1e-60, 1.0, out)


def _correlation(code, x, nu=None):
    if code == KERNEL_MATERN:
        return _matern_corr(nu, x)
    e = np.exp(-x)
    if code == KERNEL_MATERN15:
        return (1.0 + x) * e
    if code == KERNEL_MATERN25:
        return (1.0 + x + x * x / 3.0) * e
    return e


@dataclass(frozen=True)
class CovarianceFamily:
    """Handle for one registered family."""

    name: str
    kernel_code: int

    def nparms(self, d: int) -> int:
        if self.name == "exponential_anisotropic":
            return d + 2
        if self.name in ("exponential_spacetime", "matern_isotropic"):
            return 4
        return 3

    def prepare_locs(self, locs) -> np.ndarray:
        """Working coordinates: identity, except the sphere embedding."""
        locs = np.ascontiguousarray(locs, dtype=np.float64)
        if self.name == "exponential_sphere":
            if locs.ndim != 2 or locs.shape[1] != 2:
                raise ValueError(f"exponential_sphere expects lon/lat input with d=2, got d={locs.shape[-1]}")
            from .preprocess import embed_lonlat
            return embed_lonlat(locs)
        return locs

    def matrix(self, theta, locs) -> np.ndarray:
        """Dense covariance (nugget on the diagonal) at raw coordinates."""
        theta = np.asarray(theta, dtype=np.float64)
        w = self.prepare_locs(np.atleast_2d(locs))
        s, _ = _scaled_distance(w, w, _axis_ranges(self.name, theta, w.shape[1]))
        K = theta[0] * _correlation(self.kernel_code, s, theta[2] if self.kernel_code == KERNEL_MATERN else None)
        np.fill_diagonal(K, theta[0] * (1.0 + theta[-1]))
        return K

    def derivatives(self, theta, locs) -> np.ndarray:
        """(nparms, k, k) stack of dK/dtheta_j, ordered as theta."""
        theta = np.asarray(theta, dtype=np.float64)
        w = self.prepare_locs(np.atleast_2d(locs))
        k, d = w.shape
        rho = _axis_ranges(self.name, theta, d)
        s, diff = _scaled_distance(w, w, rho)
        sig2, tau2 = theta[0], theta[-1]
        q = self.nparms(d)
        D = np.zeros((q, k, k))
        nu = theta[2] if self.kernel_code == KERNEL_MATERN else None
        D[0] = _correlation(self.kernel_code, s, nu)
        np.fill_diagonal(D[0], 1.0 + tau2)
        D[q - 1] = sig2 * np.eye(k)
        e = np.exp(-s)
        if self.kernel_code in (KERNEL_ANISOTROPIC, KERNEL_SPACETIME):
            with np.errstate(invalid="ignore", divide="ignore"):
                per_axis = [np.where(s == 0.0, 0.0, sig2 * e * diff[:, :, a] ** 2 / (rho[a] * s)) for a in range(d)]
            if self.kernel_code == KERNEL_ANISOTROPIC:
                for a in range(d):
                    D[1 + a] = per_axis[a]
            else:
                D[1] = sum(per_axis[:-1])
                D[2] = per_axis[-1]
        elif self.kernel_code == KERNEL_MATERN:
            from scipy.special import gammaln
            with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
                drho = np.exp((1.0 - nu) * np.log(2.0) - gammaln(nu) + _log_xk(abs(nu - 1.0), nu + 1.0, s)) / rho[0]
            D[1] = sig2 * np.where(s < 1e-60, 0.0, drho)
            D[2] = sig2 * (_matern_corr(nu + MATERN_H, s) - _matern_corr(nu - MATERN_H, s)) / (2.0 * MATERN_H)
        elif self.kernel_code == KERNEL_MATERN15:
            D[1] = sig2 * s * s * e / rho[0]
        elif self.kernel_code == KERNEL_MATERN25:
            D[1] = sig2 * s * s * (1.0 + s) * e / (3.0 * rho[0])
        else:
            D[1] = sig2 * e * s / rho[0]
        for j in range(1, q - 1):
            np.fill_diagonal(D[j], 0.0)
        return D

    def cross(self, theta, locs_a, locs_b) -> np.ndarray:
        """Cross covariance between two location sets (no nugget)."""
        theta = np.asarray(theta, dtype=np.float64)
        a = self.prepare_locs(np.atleast_2d(locs_a))
        b = self.prepare_locs(np.atleast_2d(locs_b))
        s, _ = _scaled_distance(a, b, _axis_ranges(self.name, theta, a.shape[1]))
        return theta[0] * _correlation(self.kernel_code, s, theta[2] if self.kernel_code == KERNEL_MATERN else None)


_REGISTRY = {name: CovarianceFamily(name, code) for name, code in _CODES.items()}


def covariance_registry(name: str) -> CovarianceFamily:
    """Family handle by exact name; UnknownFamily otherwise (e.g. plain "matern")."""
    try:
        return _REGISTRY[name]
    except (KeyError, TypeError):
        raise UnknownFamily(f"unknown covariance family {name!r}; available: {', '.join(FAMILY_NAMES)}") from None


def validate_parameters(params: CovarianceParameters, d: int) -> CovarianceFamily:
    """Arity / positivity check of theta against the data dimension d."""
    fam = covariance_registry(params.family)
    if fam.name == "exponential_spacetime" and d < 2:
        raise ValueError("exponential_spacetime needs at least one spatial and one time coordinate")
    want = fam.nparms(d)
    if params.nparms != want:
        raise ValueError(f"{params.family} with d={d} needs {want} parameters, got {params.nparms}")
    th = params.theta
    if not np.isfinite(th).all():
        raise ValueError("covariance parameters must be finite")
    if (th[:-1] <= 0.0).any():
        raise ValueError("variance and range parameters must be strictly positive")
    if th[-1] < 0.0:
        raise ValueError("nugget must be >= 0")
    if fam.name == "matern_isotropic" and not (MATERN_NU_MIN < th[2] <= MATERN_NU_MAX):
        # same bounds as the device library (csrc/vecchia_b200.cu fill_params): the smoothness derivative is
        # a central difference of step MATERN_H, and x^nu K_nu(x) is evaluated by an upward recurrence in nu
        raise ValueError(f"matern_isotropic: smoothness must lie in ({MATERN_NU_MIN}, {MATERN_NU_MAX}]")
    return fam
