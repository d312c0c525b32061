"""Loader for the reference's OWN compiled core (oracle/_ref/_kernels*.so).

TEST INFRASTRUCTURE ONLY.  ``oracle/build_ref.sh`` compiles
/root/reference/pkg/src/vecchiagp/engine/_kernels.pyx (unmodified) into
``oracle/_ref/``; this module imports that shared object stand-alone and drives
it the way the reference facade does (engine/__init__.py:196-248: slot
allocation, head pass with run_sequential, tail pass with run_task, np.sum or
pairwise-tree reduction), so bench.py can time the real reference hot loop on
the GPU box's host cores, where /root/reference itself does not exist.
"""
from __future__ import annotations

import importlib.machinery
import importlib.util
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_mod = None


def available() -> bool:
    return any((HERE / "_ref").glob("_kernels*.so"))


def module():
    global _mod
    if _mod is None:
        paths = sorted((HERE / "_ref").glob("_kernels*.so"))
        if not paths:
            raise ImportError("oracle/_ref/_kernels*.so not built (run oracle/build_ref.sh)")
        loader = importlib.machinery.ExtensionFileLoader("_kernels", str(paths[0]))
        spec = importlib.util.spec_from_loader("_kernels", loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _mod = mod
    return _mod


def _tree_sum(a):
    x = a
    while x.shape[0] > 1:
        half = x.shape[0] // 2
        y = x[0:2 * half:2] + x[1:2 * half:2]
        if x.shape[0] % 2:
            y = np.concatenate([y, x[2 * half:]], axis=0)
        x = y
    return x[0]


def run(y, X, locs, nn, kcode, theta, jitter=0.0, workers=None, deterministic=False, backend="task"):
    """Flat accumulator totals (L,) from the reference's compiled runners.

    kcode: 0 isotropic, 1 anisotropic (the only kernels the reference has).
    """
    K = module()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    n = y.shape[0]
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(n, -1)
    locs = np.ascontiguousarray(locs, dtype=np.float64).reshape(n, -1)
    nn = np.ascontiguousarray(nn, dtype=np.int64)
    theta = np.ascontiguousarray(theta, dtype=np.float64).ravel()
    p, q, mp1 = X.shape[1], theta.shape[0], nn.shape[1]
    workers = workers or os.cpu_count() or 1
    cap = next((t for t in (8, 16, 32, 64) if mp1 <= t), mp1)
    slots = (np.zeros(n), np.zeros(n), np.zeros((n, p, p)), np.zeros((n, p)), np.zeros((n, q)),
             np.zeros((n, q)), np.zeros((n, p, q)), np.zeros((n, p, p, q)), np.zeros((n, q, q)))
    fail = np.zeros(n, dtype=np.int32)
    head = min(mp1 - 1, n)
    args = (y, X, locs, nn, theta, int(kcode), float(jitter), slots, fail)
    first = K.run_sequential(*args, 0, head, 1, cap)
    if first < 0 and head < n:
        first = K.RUNNERS[backend](*args, head, n, workers, cap)
    if first >= 0:
        raise FloatingPointError(f"reference core: observation {first} pivot {int(fail[first]) - 1}")
    red = _tree_sum if deterministic else (lambda s: np.sum(s, axis=0))
    return np.concatenate([np.atleast_1d(red(s)).ravel() for s in slots])
