"""Engine facade: ``run`` sums the per-observation Vecchia contributions on the GPU.

Keeps the reference facade's call signature and result type
(/root/reference/pkg/src/vecchiagp/engine/__init__.py: ``run`` :196-248, ``VecchiaParts``
:103-121, ``available_cores`` / ``active_core_name`` :64-73, ``choose_capacity_tier``
:76-85) and plugs in ONE core, ``"cuda"``: the sm_100a kernels behind the C ABI of
include/vecchia_b200.h.  What the reference does per call on the host -- slot
allocation, head pass, tail pass, host reduction (:233-248) -- happens inside a single
fused kernel launch plus a fixed-order device reduction; only the L totals and a
failure word come back.

``backend``, ``workers`` and ``capacity_tier`` are accepted for signature
compatibility (and validated like the reference does) but do not select different
code: there is one CUDA schedule.  ``deterministic`` is always honoured -- the device
reduction order is fixed, so results are run-to-run reproducible for a given GPU.

The reference's "compiled" and "fallback" CPU cores are NOT part of this package
and there is no CPU fallback: without the built library and a CUDA device, ``run``
raises ``DeviceUnavailable``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _cabi
from ..covariance import covariance_registry, validate_parameters
from ..errors import DeviceUnavailable, NotPositiveDefinite
from ..model import CovarianceParameters, Dataset, normalize_backend
from ..preprocess import NeighborArray

_FALLBACK_WARNED: set = set()
CAPACITY_TIERS = (8, 16, 32, 64)
VB_MAX_Q = 22  # csrc/common.cuh VB_MAXQ
CORES = ("cuda",)
_REFERENCE_CORES = ("compiled", "fallback")


def available_cores() -> tuple:
    return CORES


def active_core_name() -> str:
    return "cuda"


def choose_capacity_tier(mp1: int) -> int:
    """Smallest tier holding a conditioning set of m+1 points (exact size above 64)."""
    for tier in CAPACITY_TIERS:
        if mp1 <= tier:
            return tier
    return mp1


@dataclass(frozen=True)
class VecchiaParts:
    """Totals over all observations: ``logdet``/``ysy`` build the log-likelihood, ``xsx``/``ysx``
    profile the mean, the d-fields are their parameter derivatives, ``ainfo`` is the Fisher
    information of the covariance parameters."""

    logdet: float
    ysy: float
    xsx: np.ndarray
    ysx: np.ndarray
    dlogdet: np.ndarray
    dysy: np.ndarray
    dysx: np.ndarray
    dxsx: np.ndarray
    ainfo: np.ndarray


def acc_len(p: int, q: int) -> int:
    return (1 + q) * (2 + p + p * p) + q * q


def parts_from_flat(v, p: int, q: int) -> VecchiaParts:
    """Split the flat accumulator vector (C order of the reference's slot arrays,
    engine/__init__.py:141-152) into ``VecchiaParts``."""
    v = np.asarray(v, dtype=np.float64)
    cuts = np.cumsum([1, 1, p * p, p, q, q, p * q, p * p * q, q * q])
    logdet, ysy, xsx, ysx, dlogdet, dysy, dysx, dxsx, ainfo = np.split(v[:cuts[-1]], cuts[:-1])
    return VecchiaParts(float(logdet[0]), float(ysy[0]), xsx.reshape(p, p).copy(), ysx.copy(), dlogdet.copy(),
                        dysy.copy(), dysx.reshape(p, q).copy(), dxsx.reshape(p, p, q).copy(),
                        ainfo.reshape(q, q).copy())


def flat_from_parts(parts: VecchiaParts) -> np.ndarray:
    return np.concatenate([np.atleast_1d(np.asarray(x, dtype=np.float64)).ravel() for x in (
        parts.logdet, parts.ysy, parts.xsx, parts.ysx, parts.dlogdet, parts.dysy, parts.dysx, parts.dxsx,
        parts.ainfo)])


def _torch():
    try:
        import torch
    except ImportError as err:  # pragma: no cover
        raise DeviceUnavailable("PyTorch is required for device buffers") from err
    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device is visible; the cuda core has no CPU fallback")
    return torch


_STREAMS: dict = {}


def _device_streams(torch, device):
    """One (compute, upload) stream pair per device, created once.  A fresh pair per problem made the first ~16
    problems of a process slow (torch hands out 32 pool streams round-robin and the first use of each costs
    10-30 ms with this library loaded: measured in bench.py's end-to-end leg); problems on one device share the
    pair, i.e. their device work serialises, which is what a single GPU does with it anyway."""
    key = (device.type, device.index)
    pair = _STREAMS.get(key)
    if pair is None:
        with torch.cuda.device(device):
            pair = (torch.cuda.Stream(device=device), torch.cuda.Stream(device=device))
        _STREAMS[key] = pair
    return pair


_STAGING: dict = {}


def _index_staging(torch, count: int, owner):
    """One pinned int32 host buffer per process for the narrowed neighbor-table upload (pinning 130 MB costs tens of
    milliseconds: done once, grown on demand) and the event that says its last user's copies have finished."""
    import weakref
    prev = _STAGING.get("owner")
    prev = prev() if prev is not None else None
    if prev is not None and prev is not owner and getattr(prev, "_pending", None):
        prev._settle_uploads()  # it still has pieces to narrow into this buffer
    _STAGING["owner"] = weakref.ref(owner)
    buf = _STAGING.get("buf")
    if buf is None or buf.numel() < count:
        buf = torch.empty(max(count, 1), dtype=torch.int32, pin_memory=True)
        _STAGING["buf"] = buf
        _STAGING["event"] = None
    ev = _STAGING.get("event")
    if ev is not None:
        ev.synchronize()  # a previous problem's host-to-device copies read this buffer
    return buf


class DeviceProblem:
    """Device-resident inputs of one dataset (or one contiguous shard of its rows).

    PyTorch owns the device buffers (``y``, ``X``, working ``locs``, ``nn`` rows
    ``[row0, row0+rows)``); the C library adopts their pointers and packs its own
    point records.  Upload happens once here -- a Fisher-scoring fit then only
    sends theta down and gets L doubles back per evaluation.
    """

    def __init__(self, ds: Dataset, nn: NeighborArray, family: str, device=None, row0: int = 0,
                 rows: int | None = None, layout: str = "auto", nn_is_shard: bool = False,
                 upload_chunks: int | None = None, upload_narrow: bool | None = None):
        """``nn`` is the full (n, m+1) table, or -- with ``nn_is_shard`` -- only its rows
        [row0, row0+rows) (what each rank of a sharded run builds for itself).

        The neighbor table is by far the largest input (8(m+1) bytes per observation).  It is
        uploaded in ``upload_chunks`` pieces (default 16 for large tables) on a side stream, and the FIRST evaluation is issued
        chunk by chunk behind the copies (the C ABI evaluates any row range), so host-to-device
        transfer and compute overlap; later evaluations see a fully resident table.

        ``upload_narrow`` (default OFF -- measured on the 16-core B200 host at n = 2^20, m = 30: 6.2 ms per
        end-to-end step against 5.78 ms for the plain int64 copy, because narrowing 260 MB costs the host threads
        3.7-4 ms in bulk and more piece by piece, i.e. as much as the 2.7 ms of PCIe time it saves; worth turning on
        where the host has the memory bandwidth to spare): every chunk is narrowed to int32 by all
        host threads (``vbh_narrow_indices``) into a pinned staging buffer, copied -- half the PCIe bytes -- and
        widened back to the int64 rows on the device (``vb200_widen_indices``).  The pieces are issued LAZILY, by
        the first evaluation: narrow piece k on the host, enqueue its copy, widening and evaluation, go on to
        piece k+1 -- so host narrowing, PCIe and the kernel overlap (done eagerly here, the evaluation launches
        would queue behind 4 ms of host work).  The device-side table is the same int64 array either way."""
        torch = _torch()
        lib = _cabi.load()
        fam = covariance_registry(family)
        n, p = ds.n, ds.p
        rows = (nn.idx.shape[0] if nn_is_shard else n - row0) if rows is None else rows
        if row0 < 0 or rows < 0 or row0 + rows > n:
            raise ValueError("shard rows outside [0, n)")
        if nn.idx.shape[0] != (rows if nn_is_shard else n):
            raise ValueError(f"neighbor table has {nn.idx.shape[0]} rows for n={n}")
        shard_rows = nn.idx if nn_is_shard else nn.idx[row0:row0 + rows]
        work = fam.prepare_locs(ds.locs)
        self.family_name, self.kernel_code = family, fam.kernel_code
        self.n, self.p, self.d, self.mp1 = n, p, work.shape[1], nn.idx.shape[1]
        self.row0, self.rows = row0, rows
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        with torch.cuda.device(self.device):
            # A private (non-blocking) stream: the legacy default stream would serialise the library's
            # work against the side-stream upload of the neighbor table.  Consumers on other streams are
            # ordered behind it with an event (see _publish).
            self._stream, side_stream = _device_streams(torch, self.device)
        with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
            stream = self._stream
            put = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.device, non_blocking=True)
            self._y, self._X, self._locs = put(ds.y), put(ds.X), put(work)
            # [first_row, end_row, event, narrow job] of table chunks whose upload may be in flight (event None: the
            # narrowed upload of the piece has not been issued yet -- the first evaluation does it, piece by piece)
            self._pending = []
            self._narrow = None
            if upload_chunks is None:
                # 16 pieces: the evaluation of a piece overlaps the copy of the next, so the un-overlapped tail is
                # 1/16 of the kernel (measured end to end at n = 2^20: 8 -> 6.02 ms, 12 -> 5.89, 16 -> 5.78, 32 -> 5.83)
                upload_chunks = 16 if rows * self.mp1 * 8 >= (32 << 20) else 1
            if upload_narrow is None:
                upload_narrow = False
            if upload_narrow and n >= 2 ** 31:
                raise ValueError("upload_narrow needs n < 2^31")
            self.upload_narrowed = False
            if rows > 0 and upload_chunks > 1:
                src = np.ascontiguousarray(shard_rows)
                host_nn = torch.from_numpy(src)
                self._nn = torch.empty((rows, self.mp1), dtype=torch.int64, device=self.device)
                side = side_stream
                side.wait_stream(self._stream)  # the block just handed out may still be in use by earlier work
                self._nn.record_stream(side)
                cuts = (np.linspace(0, rows, upload_chunks + 1).astype(np.int64) // 2) * 2  # even rows: aligned pieces
                cuts[-1] = rows
                if upload_narrow:
                    mp1 = self.mp1
                    self._narrow = {"src": src, "stage_h": _index_staging(torch, rows * mp1, self),
                                    "stage_d": torch.empty(rows * mp1, dtype=torch.int32, device=self.device),
                                    "flat": self._nn.view(-1), "side": side}
                    self._narrow["stage_d"].record_stream(side)
                    for a, b in zip(cuts[:-1], cuts[1:]):
                        if b > a:  # event None: not issued yet (see _issue_chunk)
                            self._pending.append([row0 + int(a), row0 + int(b), None, (int(a) * mp1, int(b - a) * mp1)])
                    self.upload_narrowed = True
                else:
                    with torch.cuda.stream(side):
                        for a, b in zip(cuts[:-1], cuts[1:]):
                            if b > a:
                                self._nn[a:b].copy_(host_nn[a:b], non_blocking=True)
                                ev = torch.cuda.Event()
                                ev.record(side)
                                self._pending.append([row0 + int(a), row0 + int(b), ev, None])
                self._host_nn = host_nn  # keep the source alive while the copies run
            else:
                self._nn = put(shard_rows) if rows > 0 else torch.zeros((1, self.mp1), dtype=torch.int64,
                                                                        device=self.device)
            # bytes this constructor put on the bus (bench.py's end-to-end accounting)
            self.h2d_bytes = int(8 * (ds.y.size + ds.X.size + work.size)
                                 + (4 if self.upload_narrowed else 8) * max(rows, 0) * self.mp1)
            self._out = torch.zeros(acc_len(p, VB_MAX_Q) + 2, dtype=torch.float64, device=self.device)
            self._out_chunks = None
            handle = ctypes.c_void_p()
            rc = lib.vb200_create(self.device.index or 0, n, p, self.d, self.mp1, self._y.data_ptr(),
                                  self._X.data_ptr(), self._locs.data_ptr(), self._nn.data_ptr(), row0, rows,
                                  ctypes.c_void_p(stream.cuda_stream), ctypes.byref(handle))
            _cabi.check(rc, "vb200_create")
        self._h = handle
        self._lib = lib
        if layout != "auto":
            self.set_layout(layout)

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            if getattr(self, "_pending", None):
                # never free buffers under a copy that is still in flight (pieces never issued have none)
                self._pending = [e for e in self._pending if e[2] is not None]
                self._settle_uploads()
            self._lib.vb200_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- configuration ----------------------------------------------------------
    def set_layout(self, layout: str):
        self._layout_name = layout
        _cabi.check(self._lib.vb200_set_layout(self._h, _cabi.LAYOUTS[layout]), "vb200_set_layout")

    def layout_for(self, q: int) -> str:
        return _cabi.LAYOUT_NAMES[self._lib.vb200_get_layout(self._h, self.kernel_code, q)]

    def use_current_stream(self):
        """Launch on torch's current stream from now on (so that torch CUDA events bracket the kernels)."""
        torch = _torch()
        if self._pending:
            self._settle_uploads()
        with torch.cuda.device(self.device):
            self._stream = torch.cuda.current_stream()
        _cabi.check(self._lib.vb200_set_stream(self._h, ctypes.c_void_p(self._stream.cuda_stream)),
                    "vb200_set_stream")

    def _publish(self):
        """Order torch's current stream behind everything enqueued on the problem's stream."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.device)
        if cur != self._stream:
            ev = torch.cuda.Event()
            ev.record(self._stream)
            cur.wait_event(ev)

    def enable_timing(self, on: bool = True):
        _cabi.check(self._lib.vb200_enable_timing(self._h, int(on)), "vb200_enable_timing")

    def last_kernel_ms(self) -> float:
        ms = ctypes.c_double(0.0)
        _cabi.check(self._lib.vb200_last_kernel_ms(self._h, ctypes.byref(ms)), "vb200_last_kernel_ms")
        return ms.value

    @property
    def last_launch_count(self) -> int:
        return int(self._lib.vb200_last_launch_count(self._h))

    @property
    def last_kernel_name(self) -> str:
        return (self._lib.vb200_last_kernel_name(self._h) or b"").decode()

    # -- evaluation ---------------------------------------------------------------
    def _theta(self, theta):
        th = np.ascontiguousarray(theta, dtype=np.float64).ravel()
        self._warn_if_fallback(th.shape[0])
        return th, th.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

    def _warn_if_fallback(self, q: int):
        """layout "auto" silently ran the shape-agnostic kernel in round 1 (about 10x slower): say so, once per
        shape.  The library counts those evaluations as well (vb200_fallback_count)."""
        key = (self.kernel_code, q, self.p, self.d, self.mp1)
        if key in _FALLBACK_WARNED:
            return
        _FALLBACK_WARNED.add(key)
        if self._lib.vb200_get_layout(self._h, self.kernel_code, q) == _cabi.LAYOUTS["warp_smem"] and \
                getattr(self, "_layout_name", "auto") == "auto":
            import warnings
            warnings.warn(f"no register-tiled kernel instance for family={self.family_name}, d={self.d}, p={self.p}, "
                          f"m+1={self.mp1}: falling back to the generic shared-memory kernel (roughly 10x slower)",
                          RuntimeWarning, stacklevel=3)

    def totals(self, theta, jitter: float = 0.0, i0: int | None = None, i1: int | None = None) -> np.ndarray:
        """Flat totals (L,) over [i0, i1) of this shard; raises NotPositiveDefinite."""
        th, thp = self._theta(theta)
        q = th.shape[0]
        i0 = self.row0 if i0 is None else i0
        i1 = self.row0 + self.rows if i1 is None else i1
        if self._pending:  # first evaluation: run it behind the chunked upload
            L = acc_len(self.p, q)
            host = self.totals_async(th, jitter, i0, i1).cpu().numpy()
            if host[L] == 0.0:
                return host[:L].copy()
            self._settle_uploads()  # a failure: fall through to the plain path for (observation, pivot)
        out = np.empty(acc_len(self.p, q))
        first, piv = ctypes.c_int64(-1), ctypes.c_int32(-1)
        rc = self._lib.vb200_eval(self._h, self.kernel_code, thp, q, float(jitter), int(i0), int(i1),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(first),
                                  ctypes.byref(piv))
        _cabi.check(rc, "vb200_eval")
        if first.value >= 0:
            raise NotPositiveDefinite(pivot=piv.value, observation=first.value)
        return out

    def totals_async(self, theta, jitter: float = 0.0, i0: int | None = None, i1: int | None = None):
        """Enqueue one evaluation; returns the device tensor (L+2,) described in
        include/vecchia_b200.h (totals, failure count, -(first failing index)-1)."""
        th, thp = self._theta(theta)
        q = th.shape[0]
        i0 = self.row0 if i0 is None else i0
        i1 = self.row0 + self.rows if i1 is None else i1
        L = acc_len(self.p, q)
        if self._pending:
            return self._totals_behind_upload(thp, q, float(jitter), int(i0), int(i1), L)
        rc = self._lib.vb200_eval_async(self._h, self.kernel_code, thp, q, float(jitter), int(i0), int(i1),
                                        ctypes.c_void_p(self._out.data_ptr()))
        _cabi.check(rc, "vb200_eval_async")
        self._publish()
        return self._out[:L + 2]

    def _issue_chunk(self, entry):
        """Narrowed upload of one piece of the table: host narrowing (all host threads), copy and device-side
        widening on the side stream; returns the event behind them."""
        if entry[2] is not None:
            return entry[2]
        torch = _torch()
        from ..preprocess import host_library
        nw = self._narrow
        lo, cnt = entry[3]
        bad = host_library().vbh_narrow_indices(nw["src"].ctypes.data + 8 * lo, nw["stage_h"].data_ptr() + 4 * lo, cnt, 0)
        if bad:
            raise ValueError("neighbor index outside the int32 range in a table with n < 2^31")
        with torch.cuda.device(self.device), torch.cuda.stream(nw["side"]):
            nw["stage_d"][lo:lo + cnt].copy_(nw["stage_h"][lo:lo + cnt], non_blocking=True)
            _cabi.check(self._lib.vb200_widen_indices(nw["stage_d"].data_ptr() + 4 * lo, nw["flat"].data_ptr() + 8 * lo,
                                                      cnt, ctypes.c_void_p(nw["side"].cuda_stream)),
                        "vb200_widen_indices")
            ev = torch.cuda.Event()
            ev.record(nw["side"])
        entry[2] = ev
        _STAGING["event"] = ev
        return ev

    def _settle_uploads(self):
        torch = _torch()
        with torch.cuda.device(self.device):
            for entry in self._pending:
                ev = entry[2] if entry[2] is not None else self._issue_chunk(entry)
                ev.synchronize()
        self._pending = []
        self._host_nn = None
        self._narrow = None  # the staging tensors go back to the allocator (stream-ordered: record_stream)

    def _totals_behind_upload(self, thp, q, jitter, i0, i1, L):
        """Evaluate [i0, i1) one upload chunk at a time, each piece waiting (on the device) for its
        chunk's copy event; the pieces' (L+2) vectors are combined on the device."""
        torch = _torch()
        with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
            compute = self._stream
            if self._out_chunks is None or self._out_chunks.shape[0] < len(self._pending):
                self._out_chunks = torch.zeros((len(self._pending), self._out.shape[0]), dtype=torch.float64,
                                               device=self.device)
            k = 0
            for entry in self._pending:
                a, b = entry[0], entry[1]
                lo, hi = max(a, i0), min(b, i1)
                if lo >= hi:
                    continue
                ev = entry[2] if entry[2] is not None else self._issue_chunk(entry)
                compute.wait_event(ev)
                rc = self._lib.vb200_eval_async(self._h, self.kernel_code, thp, q, jitter, lo, hi,
                                                ctypes.c_void_p(self._out_chunks[k].data_ptr()))
                _cabi.check(rc, "vb200_eval_async")
                k += 1
            if k == 0:
                self._out[:L + 2] = torch.tensor([0.0] * (L + 1) + [float("-inf")], dtype=torch.float64,
                                                 device=self.device)
            else:
                pieces = self._out_chunks[:k]
                self._out[:L + 1] = pieces[:, :L + 1].sum(dim=0)
                self._out[L + 1] = pieces[:, L + 1].max()
            if i0 <= self.row0 and i1 >= self.row0 + self.rows:
                # the compute stream now sits behind every copy: later work needs no more waits
                self._pending = []
                self._narrow = None
        self._publish()
        return self._out[:L + 2]

    def fail_info(self):
        if self._pending:
            self._settle_uploads()
        first, piv = ctypes.c_int64(-1), ctypes.c_int32(-1)
        _cabi.check(self._lib.vb200_fail_info(self._h, ctypes.byref(first), ctypes.byref(piv)), "vb200_fail_info")
        return first.value, piv.value

    def rows_host(self, theta, jitter: float = 0.0, i0: int | None = None, i1: int | None = None):
        """Per-observation accumulator rows (i1-i0, L) and pivot+1 failure flags (diagnostics)."""
        if self._pending:
            self._settle_uploads()
        th, thp = self._theta(theta)
        q = th.shape[0]
        i0 = self.row0 if i0 is None else i0
        i1 = self.row0 + self.rows if i1 is None else i1
        rows = np.zeros((max(i1 - i0, 0), acc_len(self.p, q)))
        flags = np.zeros(max(i1 - i0, 0), dtype=np.int32)
        rc = self._lib.vb200_eval_rows(self._h, self.kernel_code, thp, q, float(jitter), int(i0), int(i1),
                                       rows.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        _cabi.check(rc, "vb200_eval_rows")
        return rows, flags

    def run(self, cov: CovarianceParameters, jitter: float = 0.0) -> VecchiaParts:
        if cov.family != self.family_name:
            raise ValueError(f"problem was built for {self.family_name!r}, got {cov.family!r}")
        return parts_from_flat(self.totals(cov.theta, jitter), self.p, cov.nparms)


# ---------------------------------------------------------------------------
# facade.  `run` is STATELESS like the reference's (engine/__init__.py:196-248): every call uploads the
# arrays it is given, so in-place edits of y / X / locs / nn between calls are always honoured (round 1
# cached device copies keyed on host addresses; the advisor flagged the stale-data hazard).  Code that
# evaluates the same dataset repeatedly -- `inference.fit`, bench.py -- holds an explicit DeviceProblem.
# ---------------------------------------------------------------------------
def clear_cache() -> None:
    """Kept for API compatibility with round 1: there is no implicit device cache any more."""


def _validate_core(core):
    """The reference reads its default core from VECCHIAGP_CORE (engine/__init__.py:52-60); here the only
    core is "cuda", so the variable may be unset, empty or "cuda" -- anything else is an error, as an unknown
    name is in the reference."""
    import os
    core = core or os.environ.get("VECCHIAGP_CORE") or "cuda"
    if core in _REFERENCE_CORES:
        raise ValueError(f"core {core!r} is a CPU core of the reference package; this package provides 'cuda' only")
    if core != "cuda":
        raise ValueError(f"unknown core {core!r}")
    return core


def run(ds: Dataset, nn: NeighborArray, cov: CovarianceParameters, backend: str = "task",
        deterministic: bool = True, workers: int | None = None, capacity_tier: int | None = None,
        jitter: float = 0.0, core: str | None = None) -> VecchiaParts:
    """Sum of every observation's contribution (drop-in for the reference's ``engine.run``).

    Raises ``NotPositiveDefinite`` with the lowest failing observation index when a local
    factorization fails; no jitter is added unless requested.
    """
    normalize_backend(backend)
    _validate_core(core)
    validate_parameters(cov, ds.d)
    mp1 = nn.idx.shape[1]
    if nn.idx.shape[0] != ds.n:
        raise ValueError(f"neighbor table has {nn.idx.shape[0]} rows for n={ds.n}")
    if capacity_tier is not None and capacity_tier < mp1:
        raise ValueError(f"capacity tier {capacity_tier} too small for m+1={mp1}")
    with DeviceProblem(ds, nn, cov.family) as prob:
        return prob.run(cov, jitter=float(jitter))


def process_observation(i: int, ds: Dataset, nn: NeighborArray, cov: CovarianceParameters,
                        jitter: float = 0.0) -> VecchiaParts:
    """One observation's contribution (reference: engine/__init__.py:179-193), from the GPU."""
    if not 0 <= i < ds.n:
        raise IndexError(f"observation index {i} outside [0, {ds.n})")
    validate_parameters(cov, ds.d)
    with DeviceProblem(ds, nn, cov.family, upload_chunks=1) as prob:
        rows, flags = prob.rows_host(cov.theta, jitter, i, i + 1)
    if flags[0]:
        raise NotPositiveDefinite(pivot=int(flags[0]) - 1, observation=i)
    return parts_from_flat(rows[0], ds.p, cov.nparms)
