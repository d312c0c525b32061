"""Ordering, sphere embedding and the ordered neighbor table (host side).

API of the reference's preprocess module (/root/reference/pkg/src/vecchiagp/
preprocess.py): ``Ordering`` :22-33, ``identity_ordering`` :36-37, ``random_permutation``
:40-49 (PCG64 Fisher-Yates via numpy), ``reorder_dataset`` :52-59, ``lonlat_to_xyz`` :62-74,
``embed_lonlat`` :77-92, ``NeighborArray`` :95-118, ``find_ordered_neighbors`` :135-154.

The neighbor table is produced on the host by csrc/host_neighbors.cpp, which returns
the same table as the reference's exhaustive scan (same d2 arithmetic, same
smaller-index tie rule) from a grid index, so n = 2^20 .. 2^24 is practical.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .errors import LatitudeOutOfRange, LengthMismatch
from .model import Dataset

SENTINEL = -1


@dataclass(frozen=True)
class Ordering:
    """Permutation of 0..n-1: new position -> original index."""

    perm: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "perm", np.ascontiguousarray(self.perm, dtype=np.int64))

    @property
    def n(self) -> int:
        return self.perm.shape[0]


def identity_ordering(n: int) -> Ordering:
    return Ordering(np.arange(n, dtype=np.int64))


def random_permutation(n: int, seed: int) -> Ordering:
    """Uniform permutation from numpy's PCG64 generator (same stream as the reference)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    gen = np.random.Generator(np.random.PCG64(seed))
    return Ordering(gen.permutation(n).astype(np.int64))


def maxmin_ordering(locs) -> Ordering:
    """Max-min distance ordering of working coordinates (an addition: the reference offers identity and
    random orderings only, model.py:135-136; BASELINE.json config 1 names maxmin).  Position 0 is the
    point nearest the centroid; each following point maximises its minimum distance to all earlier
    ones (smallest index on ties).  Exact greedy selection, ~O(n log n) (csrc/host_neighbors.cpp)."""
    locs = np.ascontiguousarray(np.atleast_2d(locs), dtype=np.float64)
    out = np.empty(locs.shape[0], dtype=np.int64)
    rc = host_library().vbh_order_maxmin(locs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), locs.shape[0],
                                         locs.shape[1], out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc == -3:
        from .errors import NonFiniteValue
        raise NonFiniteValue("non-finite coordinate in locs")
    if rc != 0:
        raise RuntimeError(f"maxmin ordering failed with code {rc}")
    return Ordering(out)


def reorder_dataset(ds: Dataset, ordering: Ordering) -> Dataset:
    if ordering.n != ds.n:
        raise LengthMismatch(f"permutation length {ordering.n} does not match n={ds.n}")
    idx = ordering.perm
    return Dataset(y=ds.y[idx], X=ds.X[idx], locs=ds.locs[idx])


def lonlat_to_xyz(lon: float, lat: float) -> np.ndarray:
    """One lon/lat degree pair on the unit sphere: (cos lat cos lon, cos lat sin lon, sin lat)."""
    if not -90.0 <= lat <= 90.0:
        raise LatitudeOutOfRange(f"latitude {lat} outside [-90, 90]")
    lam, phi = np.deg2rad(lon), np.deg2rad(lat)
    return np.array([np.cos(phi) * np.cos(lam), np.cos(phi) * np.sin(lam), np.sin(phi)])


def embed_lonlat(locs) -> np.ndarray:
    """Vectorised sphere embedding of an (n, 2) lon/lat degree array."""
    locs = np.atleast_2d(np.asarray(locs, dtype=np.float64))
    if locs.shape[1] != 2:
        raise ValueError(f"expected (n, 2) lon/lat input, got shape {locs.shape}")
    lat = locs[:, 1]
    outside = (lat < -90.0) | (lat > 90.0)
    if outside.any():
        row = int(np.argmax(outside))
        raise LatitudeOutOfRange(f"latitude {lat[row]} at row {row} outside [-90, 90]")
    lam, phi = np.deg2rad(locs[:, 0]), np.deg2rad(lat)
    xyz = np.empty((locs.shape[0], 3))
    xyz[:, 0] = np.cos(phi) * np.cos(lam)
    xyz[:, 1] = np.cos(phi) * np.sin(lam)
    xyz[:, 2] = np.sin(phi)
    return xyz


@dataclass(frozen=True)
class NeighborArray:
    """(n, m+1) int64 table: column 0 = the observation, then its nearest predecessors by
    increasing distance (ties -> smaller index), -1 in unused trailing cells."""

    idx: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "idx", np.ascontiguousarray(self.idx, dtype=np.int64))

    @property
    def n(self) -> int:
        return self.idx.shape[0]

    @property
    def m(self) -> int:
        return self.idx.shape[1] - 1

    def row_sizes(self) -> np.ndarray:
        return (self.idx >= 0).sum(axis=1)


_host = None


def host_library():
    """ctypes handle of libvecchia_host.so (built on first use)."""
    global _host
    if _host is None:
        from . import build
        lib = ctypes.CDLL(str(build.build_host()))
        dp, ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        for name in ("vbh_neighbors_exhaustive", "vbh_neighbors_grid"):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ip]
        lib.vbh_neighbors_grid_rows.restype = ctypes.c_int
        lib.vbh_neighbors_grid_rows.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int64, ctypes.c_int64, ip]
        lib.vbh_neighbors_query.restype = ctypes.c_int
        lib.vbh_neighbors_query.argtypes = [dp, ctypes.c_int64, ctypes.c_int, dp, ctypes.c_int64, ctypes.c_int,
                                            ctypes.c_int, ip]
        lib.vbh_order_maxmin.restype = ctypes.c_int
        lib.vbh_order_maxmin.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ip]
        lib.vbh_max_threads.restype = ctypes.c_int
        lib.vbh_narrow_indices.restype = ctypes.c_int
        lib.vbh_narrow_indices.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        lib.vbh_dependency_levels.restype = ctypes.c_int64
        lib.vbh_dependency_levels.argtypes = [ip, ctypes.c_int64, ctypes.c_int, ip, ip]
        _host = lib
    return _host


def _worker_count(workers=None) -> int:
    if workers is not None:
        return max(1, int(workers))
    env = os.environ.get("VECCHIAGP_WORKERS")
    if env:
        return max(1, int(env))
    return os.cpu_count() or 1


def find_ordered_neighbors(locs, m: int, workers: int | None = None, method: str = "auto") -> NeighborArray:
    """Conditioning-set table for already-ordered working coordinates.

    ``method``: "grid" (multi-resolution grid index), "exhaustive" (the reference's
    normative O(n^2) scan) or "auto" (exhaustive for small n).  Both give the same table.
    """
    if m < 1:
        raise ValueError("m must be >= 1")
    locs = np.ascontiguousarray(np.atleast_2d(locs), dtype=np.float64)
    n, d = locs.shape
    m = min(int(m), max(n - 1, 1))
    if method not in ("auto", "grid", "exhaustive"):
        raise ValueError(f"unknown neighbor search method {method!r}")
    if method == "auto":
        method = "exhaustive" if n <= 4096 else "grid"
    out = np.full((n, m + 1), SENTINEL, dtype=np.int64)
    lib = host_library()
    fn = lib.vbh_neighbors_grid if method == "grid" else lib.vbh_neighbors_exhaustive
    rc = fn(locs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, d, m, _worker_count(workers),
            out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc == -3:
        from .errors import NonFiniteValue
        raise NonFiniteValue("non-finite coordinate in locs")
    if rc != 0:
        raise RuntimeError(f"neighbor search failed with code {rc}")
    return NeighborArray(out)


def find_ordered_neighbor_rows(locs, m: int, row0: int, rows: int, workers: int | None = None) -> np.ndarray:
    """Rows [row0, row0+rows) of the table ``find_ordered_neighbors(locs, m)`` would return,
    as a (rows, m+1) int64 array -- each rank of a sharded run builds only its own rows."""
    if m < 1:
        raise ValueError("m must be >= 1")
    locs = np.ascontiguousarray(np.atleast_2d(locs), dtype=np.float64)
    n, d = locs.shape
    m = min(int(m), max(n - 1, 1))
    out = np.full((rows, m + 1), SENTINEL, dtype=np.int64)
    rc = host_library().vbh_neighbors_grid_rows(
        locs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, d, m, _worker_count(workers), int(row0), int(rows),
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc != 0:
        raise RuntimeError(f"neighbor search failed with code {rc}")
    return out


def find_nearest_training(work_train, work_star, m_pred: int, workers: int | None = None) -> np.ndarray:
    """(nstar, m_pred) int64 indices of the m_pred training rows nearest to each query point, ranked by
    (squared distance, index) -- the selection of the reference's kriging (predict.py:27-32)."""
    a = np.ascontiguousarray(np.atleast_2d(work_train), dtype=np.float64)
    b = np.ascontiguousarray(np.atleast_2d(work_star), dtype=np.float64)
    if a.shape[1] != b.shape[1]:
        raise ValueError("training and prediction coordinates differ in dimension")
    if not 1 <= m_pred <= a.shape[0]:
        raise ValueError(f"m_pred must be in [1, n]={a.shape[0]}, got {m_pred}")
    out = np.full((b.shape[0], m_pred), SENTINEL, dtype=np.int64)
    rc = host_library().vbh_neighbors_query(
        a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), a.shape[0], a.shape[1],
        b.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), b.shape[0], int(m_pred), _worker_count(workers),
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc != 0:
        raise RuntimeError(f"neighbor query failed with code {rc}")
    return out


def dependency_levels(nn: NeighborArray):
    """Level schedule of the conditioning DAG: ``(order, level_ptr)`` with ``order[level_ptr[l]:level_ptr[l+1]]``
    the observations of level ``l`` (level = 1 + max level of the row's neighbours; rows without neighbours
    are level 0), ascending within a level.  Observations of one level are conditionally independent of each
    other given the lower levels: the launch schedule of the device conditional simulator (``simulate``)."""
    idx = np.ascontiguousarray(nn.idx, dtype=np.int64)
    n, mp1 = idx.shape
    order = np.empty(n, dtype=np.int64)
    level_ptr = np.zeros(n + 1, dtype=np.int64)
    ip = ctypes.POINTER(ctypes.c_int64)
    nlev = host_library().vbh_dependency_levels(idx.ctypes.data_as(ip), n, mp1, order.ctypes.data_as(ip),
                                                level_ptr.ctypes.data_as(ip))
    if nlev < 0:
        raise ValueError("neighbor table is not causal: a row lists an index that is not smaller than its own")
    return order, level_ptr[:nlev + 1].copy()
