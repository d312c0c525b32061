"""Conditional simulation from the neighbour-conditioned model on the GPU.

Same entry point as the reference's ``oracle.simulate_nn_gp`` (/root/reference/pkg/src/vecchiagp/oracle.py:102-140):
each y_i is drawn from its conditional distribution given the already drawn values of its conditioning set, which
is exactly the joint distribution the Vecchia approximation defines.  The reference walks the observations one by one
in Python (O(n m^3), single thread); here the observations are grouped by dependency level
(``preprocess.dependency_levels``, host C++) and every level is one launch of the kriging kernel
(csrc/kernel_krige.cuh in simulation mode, ``vb200_simulate``).  The normal draws come from the same
``numpy.random.Generator(PCG64(seed))`` stream as the reference's, so the two outputs agree to rounding.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _cabi
from .covariance import covariance_registry
from .errors import NotPositiveDefinite
from .model import CovarianceParameters, Dataset
from .preprocess import NeighborArray, dependency_levels


def simulate_nn_gp(cov: CovarianceParameters, beta, locs, X, nn: NeighborArray, seed: int) -> np.ndarray:
    """Sequential conditional draw y (n,) from the neighbour-conditioned model (mean ``X @ beta``)."""
    from .engine import DeviceProblem

    family = covariance_registry(cov.family)
    locs = np.atleast_2d(np.asarray(locs, dtype=np.float64))
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    n = locs.shape[0]
    if nn.idx.shape[0] != n:
        raise ValueError(f"neighbor table has {nn.idx.shape[0]} rows for {n} locations")
    theta = np.ascontiguousarray(cov.theta, dtype=np.float64)
    beta = np.ascontiguousarray(np.atleast_1d(beta), dtype=np.float64).ravel()
    if beta.shape[0] != X.shape[1]:
        raise ValueError(f"{beta.shape[0]} mean parameters for {X.shape[1]} design columns")
    rng = np.random.Generator(np.random.PCG64(seed))
    xi = np.ascontiguousarray(rng.standard_normal(n))
    if nn.idx.shape[1] < 2:  # no conditioning at all: independent draws with the prior variance
        return X @ beta + np.sqrt(theta[0] * (1.0 + theta[-1])) * xi
    order, level_ptr = dependency_levels(nn)
    y = np.empty(n)
    first = ctypes.c_int64(-1)
    dp, ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
    ds = Dataset(np.zeros(n), X, locs)  # the response column of the records is filled by the device
    with DeviceProblem(ds, nn, cov.family, upload_chunks=1) as prob:
        rc = prob._lib.vb200_simulate(prob._h, prob.kernel_code, theta.ctypes.data_as(dp), theta.shape[0],
                                      beta.ctypes.data_as(dp), xi.ctypes.data_as(dp), order.ctypes.data_as(ip),
                                      level_ptr.ctypes.data_as(ip), level_ptr.shape[0] - 1,
                                      y.ctypes.data_as(dp), ctypes.byref(first))
        _cabi.check(rc, "vb200_simulate")
    if first.value >= 0:
        raise NotPositiveDefinite(pivot=-1, observation=int(first.value))
    return y
