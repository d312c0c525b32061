"""Binary on-disk formats for large problems, plus the reference's fit document.

SURVEY.md 8f rank 4: the reference stores datasets and neighbor caches as CSV
(/root/reference/pkg/src/vecchiagp/io.py:35-126), which is impractical at n >= 2^20 (a 2^24 x 31
index table).  Here a dataset is one ``.npz`` (y, X, locs as float64) and a neighbor table one
``.npy`` (int64, the reference's layout, memory-mappable).  The fit document keeps the reference's
JSON schema key for key (io.py:128-185) so that files are interchangeable.
"""
from __future__ import annotations

import json

import numpy as np

from .model import CovarianceParameters, Dataset, FitResult
from .preprocess import NeighborArray

FIT_SCHEMA_KEYS = ("version", "family", "theta_hat", "beta_hat", "beta_cov", "fisher_info", "loglik_trace",
                   "iterations", "converged", "phase_timings_ms", "config")


def write_dataset_npz(ds: Dataset, path) -> None:
    np.savez(path, y=ds.y, X=ds.X, locs=ds.locs)


def read_dataset_npz(path) -> Dataset:
    with np.load(path) as z:
        return Dataset(y=z["y"], X=z["X"], locs=z["locs"])


def write_neighbors_npy(nn: NeighborArray, path) -> None:
    np.save(path, nn.idx)


def read_neighbors_npy(path, mmap: bool = False) -> NeighborArray:
    """``mmap=True`` maps the file instead of reading it (rank r of a sharded run touches only its rows)."""
    idx = np.load(path, mmap_mode="r" if mmap else None)
    if idx.dtype != np.int64 or idx.ndim != 2:
        raise ValueError(f"{path}: expected a 2-D int64 neighbor table, got {idx.dtype} {idx.shape}")
    return NeighborArray(idx)


def fit_to_dict(fit: FitResult, config=None, version="0.1.0") -> dict:
    return {
        "version": version,
        "family": fit.theta_hat.family,
        "theta_hat": [float(v) for v in fit.theta_hat.theta],
        "beta_hat": [float(v) for v in fit.beta_hat],
        "beta_cov": [[float(v) for v in row] for row in np.atleast_2d(fit.beta_cov)],
        "fisher_info": [[float(v) for v in row] for row in np.atleast_2d(fit.fisher_info)],
        "loglik_trace": [float(v) for v in fit.loglik_trace],
        "iterations": int(fit.iterations),
        "converged": bool(fit.converged),
        "phase_timings_ms": {k: float(v) for k, v in fit.phase_timings.items()},
        "config": dict(config) if config else {},
    }


def write_fit_json(fit: FitResult, path, config=None, version="0.1.0") -> None:
    with open(path, "w") as handle:
        json.dump(fit_to_dict(fit, config=config, version=version), handle, indent=2)
        handle.write("\n")


def read_fit_json(path) -> dict:
    with open(path) as handle:
        return json.load(handle)


def fit_from_dict(doc: dict) -> FitResult:
    return FitResult(theta_hat=CovarianceParameters(family=doc["family"], theta=np.asarray(doc["theta_hat"])),
                     beta_hat=np.asarray(doc["beta_hat"]), beta_cov=np.asarray(doc["beta_cov"]),
                     loglik_trace=list(doc["loglik_trace"]), fisher_info=np.asarray(doc["fisher_info"]),
                     iterations=int(doc["iterations"]), converged=bool(doc["converged"]),
                     phase_timings=dict(doc.get("phase_timings_ms", {})))
