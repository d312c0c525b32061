"""ctypes binding of include/vecchia_b200.h (the C ABI of libvecchia_b200.so).

Thin by design: argument marshalling and error translation only.  There is no
CPU fallback here or anywhere in the package -- if the library is missing or no
CUDA device is visible, ``DeviceUnavailable`` is raised.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

from .errors import DeviceUnavailable

VB200_OK, VB200_EINVAL, VB200_ECUDA, VB200_ENOMEM, VB200_EUNSUPPORTED = 0, -1, -2, -3, -4

LAYOUTS = {"auto": 0, "warp_smem": 1, "tiled_reg": 2, "thread_smem": 3, "thread_local": 4}
LAYOUT_NAMES = {v: k for k, v in LAYOUTS.items()}

_dp, _ip = POINTER(c_double), POINTER(c_int64)
_lib = None

_SIGNATURES = {
    "vb200_abi_version": (c_int, []),
    "vb200_last_error": (c_char_p, []),
    "vb200_acc_len": (c_int, [c_int, c_int]),
    "vb200_family_nparms": (c_int, [c_int, c_int]),
    "vb200_device_count": (c_int, []),
    "vb200_create": (c_int, [c_int, c_int64, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_int64, c_int64, c_void_p, POINTER(c_void_p)]),
    "vb200_destroy": (c_int, [c_void_p]),
    "vb200_set_stream": (c_int, [c_void_p, c_void_p]),
    "vb200_set_layout": (c_int, [c_void_p, c_int]),
    "vb200_get_layout": (c_int, [c_void_p, c_int, c_int]),
    "vb200_eval": (c_int, [c_void_p, c_int, _dp, c_int, c_double, c_int64, c_int64, _dp, POINTER(c_int64),
                           POINTER(c_int32)]),
    "vb200_eval_async": (c_int, [c_void_p, c_int, _dp, c_int, c_double, c_int64, c_int64, c_void_p]),
    "vb200_sync": (c_int, [c_void_p]),
    "vb200_fail_info": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int32)]),
    "vb200_eval_rows": (c_int, [c_void_p, c_int, _dp, c_int, c_double, c_int64, c_int64, _dp, POINTER(c_int32)]),
    "vb200_krige": (c_int, [c_void_p, c_int, _dp, c_int, _dp, c_void_p, c_void_p, c_int64, c_int, c_int, _dp, _dp,
                            POINTER(c_int64)]),
    "vb200_simulate": (c_int, [c_void_p, c_int, _dp, c_int, _dp, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                               POINTER(c_int64)]),
    "vb200_last_launch_count": (c_int, [c_void_p]),
    "vb200_last_kernel_name": (c_char_p, [c_void_p]),
    "vb200_tiled_instance_count": (c_int, []),
    "vb200_tiled_instance": (c_int, [c_int] + [POINTER(c_int)] * 6),
    "vb200_enable_timing": (c_int, [c_void_p, c_int]),
    "vb200_last_kernel_ms": (c_int, [c_void_p, _dp]),
    "vb200_measure_fp64_peak": (c_int, [c_int, c_double, _dp, _dp]),
    "vb200_measure_fp64_peak_mma": (c_int, [c_int, c_double, _dp, _dp]),
    "vb200_release_memory": (c_int, [c_int]),
    "vb200_widen_indices": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "vb200_fallback_count": (ctypes.c_ulonglong, []),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def library_path():
    from . import build
    return build.CUDA_LIB


def load(build_if_missing: bool = True):
    """The loaded library; raises DeviceUnavailable when it cannot be loaded."""
    global _lib
    if _lib is None:
        from . import build
        try:
            import os
            override = os.environ.get("VB200_LIB")  # development: load an alternative build of the same ABI
            path = override or (build.build_cuda() if build_if_missing else build.CUDA_LIB)
            lib = ctypes.CDLL(str(path))
        except (OSError, RuntimeError, Exception) as err:  # noqa: BLE001 - anything here means "no CUDA core"
            raise DeviceUnavailable(f"cannot load the CUDA core ({err}); there is no CPU fallback") from err
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().vb200_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Translate a VB200_E* code into the Python exception the reference would raise."""
    if rc == VB200_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == VB200_EINVAL:
        raise ValueError(msg)
    if rc == VB200_ENOMEM:
        raise MemoryError(msg)
    if rc == VB200_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == VB200_ECUDA:
        raise DeviceUnavailable(msg)
    raise RuntimeError(f"{msg} (code {rc})")


def device_count() -> int:
    return int(load().vb200_device_count())


def tiled_instances():
    """List of (lanes_per_obs, rows_per_lane, cap, family_code, d, p) of the compiled TILED_REG kernels."""
    lib = load()
    out = []
    for k in range(lib.vb200_tiled_instance_count()):
        vals = [c_int() for _ in range(6)]
        check(lib.vb200_tiled_instance(k, *[ctypes.byref(v) for v in vals]), "vb200_tiled_instance")
        out.append(tuple(v.value for v in vals))
    return out
