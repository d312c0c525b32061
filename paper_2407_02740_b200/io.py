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


# ---------------------------------------------------------------------------
# the reference's text formats (io.py:35-126): CSV datasets with a header row (response column, covariate
# columns, coordinate columns) and CSV neighbor tables, floats written with repr() so a round trip is exact
# ---------------------------------------------------------------------------
def write_csv_dataset(ds: Dataset, path, y_col: str = "y", x_prefix: str = "x", loc_prefix: str = "loc") -> None:
    names = [y_col] + [f"{x_prefix}{j}" for j in range(ds.p)] + [f"{loc_prefix}{j}" for j in range(ds.d)]
    with open(path, "w") as handle:
        handle.write(",".join(names) + "\n")
        for i in range(ds.n):
            row = [ds.y[i], *ds.X[i], *ds.locs[i]]
            handle.write(",".join(repr(float(v)) for v in row) + "\n")


def read_csv_dataset(path, y_col: str = "y", x_cols=None, loc_cols=None, x_prefix: str = "x",
                     loc_prefix: str = "loc") -> Dataset:
    """Columns are selected by name; by default every column named `x<j>` is a covariate and every `loc<j>` a
    coordinate (the layout write_csv_dataset produces).  A dataset without covariate columns gets an intercept."""
    with open(path) as handle:
        header = [h.strip() for h in handle.readline().rstrip("\n").split(",")]
        rows = [line.rstrip("\n").split(",") for line in handle if line.strip()]
    if y_col not in header:
        raise ValueError(f"no response column {y_col!r} in {path}")
    pick = lambda prefix: [h for h in header if h.startswith(prefix) and h[len(prefix):].isdigit()]
    x_cols = list(x_cols) if x_cols is not None else pick(x_prefix)
    loc_cols = list(loc_cols) if loc_cols is not None else pick(loc_prefix)
    missing = [c for c in x_cols + loc_cols if c not in header]
    if missing:
        raise ValueError(f"columns {missing} not in {path}")
    if not loc_cols:
        raise ValueError("no coordinate columns")
    col = {h: k for k, h in enumerate(header)}
    data = np.array([[float(v) for v in r] for r in rows], dtype=np.float64).reshape(len(rows), len(header))
    X = data[:, [col[c] for c in x_cols]] if x_cols else np.ones((len(rows), 1))
    return Dataset(data[:, col[y_col]], X, data[:, [col[c] for c in loc_cols]])


def write_neighbors_csv(nn: NeighborArray, path) -> None:
    with open(path, "w") as handle:
        for row in nn.idx:
            handle.write(",".join(str(int(v)) for v in row) + "\n")


def read_neighbors_csv(path) -> NeighborArray:
    with open(path) as handle:
        rows = [[int(v) for v in line.split(",")] for line in handle if line.strip()]
    return NeighborArray(np.array(rows, dtype=np.int64))
