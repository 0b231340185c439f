"""Locate and bind libaxhelm_sm100.so (the C ABI in include/axhelm.h).

There is no fallback: if the library is missing or cannot be loaded the
product path raises, so a GPU test can never pass on a silent CPU path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CodegenError

PKG = Path(__file__).resolve().parent
DEFAULT_LIB = PKG / "libaxhelm_sm100.so"

_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# every exported symbol and its ctypes prototype (restype, argtypes)
PROTOTYPES = {
    "__dace_ax_helm": (None, [_vp] * 15 + [ctypes.c_int, ctypes.c_int]),
    "axhelm_apply": (ctypes.c_int, [_vp] * 15 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _vp]),
    "axhelm_apply_sync": (ctypes.c_int, [_vp] * 15 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]),
    "axhelm_probe_stream": (ctypes.c_int, [_vp] * 9 + [ctypes.c_int64, _vp]),
    "axhelm_box_gid": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, _vp]),
    "axhelm_box_geometry": (ctypes.c_int, [_vp] * 9 + [ctypes.c_int] * 4 + [ctypes.c_int64, ctypes.c_int64,
                                                                          ctypes.c_double, _vp]),
    "axhelm_gs_sum": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int64, _vp]),
    "axhelm_gs_plane": (ctypes.c_int, [ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp, ctypes.c_int64,
                                       _vp, _vp]),
    "axhelm_gs_box": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp]),
    "axhelm_gs_box_range": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp]),
    "axhelm_reduce_blocks": (ctypes.c_int, [ctypes.c_int64]),
    "axhelm_peer_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p), _vp]),
    "axhelm_peer_open": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    "axhelm_peer_close": (ctypes.c_int, [_vp]),
    "axhelm_peer_free": (ctypes.c_int, [_vp]),
    "axhelm_peer_allreduce_bytes": (ctypes.c_int64, []),
    "axhelm_peer_allreduce": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_ulonglong, _vp, _vp]),
    "axhelm_gs_box_peer": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                           ctypes.c_ulonglong, _vp, _vp, _vp]),
    "axhelm_peer_seq_bump": (ctypes.c_int, [_vp, _vp]),
    "axhelm_ax_gs_box": (ctypes.c_int, [_vp] * 15 + [ctypes.c_int] * 3 + [ctypes.c_int64] * 6
                         + [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "axhelm_ax_gs_scratch": (ctypes.c_int, [ctypes.c_int64]),
    "axhelm_dot": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp]),
    "axhelm_cg_init": (ctypes.c_int, [_vp] * 7 + [ctypes.c_int64, _vp, _vp, _vp]),
    "axhelm_cg_update": (ctypes.c_int, [_vp] * 7 + [ctypes.c_int64, _vp, _vp, _vp]),
    "axhelm_apply_dot": (ctypes.c_int, [_vp] * 15 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "axhelm_cg_pupdate": (ctypes.c_int, [_vp] * 5 + [ctypes.c_int64, _vp]),
    "axhelm_cg_update_box": (ctypes.c_int, [_vp] * 4 + [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                       ctypes.c_int, _vp, _vp, _vp]),
    "axhelm_apply_box": (ctypes.c_int, [_vp] * 15 + [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                     _vp, _vp, _vp, _vp]),
    "axhelm_cg_xpupdate": (ctypes.c_int, [_vp] * 6 + [ctypes.c_int64, _vp]),
    "axhelm_diag": (ctypes.c_int, [_vp] * 14 + [ctypes.c_int64, ctypes.c_int, _vp]),
    "axhelm_set_mode": (ctypes.c_int, [ctypes.c_int]),
    "axhelm_get_mode": (ctypes.c_int, []),
    "axhelm_last_status": (ctypes.c_int, []),
    "axhelm_last_error": (ctypes.c_char_p, []),
    "axhelm_version": (ctypes.c_char_p, []),
    "axhelm_bytes_model": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int]),
    "axhelm_flops_model": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int]),
}

_CACHE: dict[str, ctypes.CDLL] = {}


def lib_path() -> Path:
    return Path(os.environ.get("AXHELM_LIB", DEFAULT_LIB))


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """dlopen the library once and attach prototypes to every known symbol."""
    p = str(Path(path) if path is not None else lib_path())
    if p in _CACHE:
        return _CACHE[p]
    if not Path(p).exists():
        raise CodegenError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(p)
    except OSError as exc:
        raise CodegenError(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype = res
            fn.argtypes = args
    _CACHE[p] = lib
    return lib


def last_error(lib: ctypes.CDLL) -> str:
    msg = lib.axhelm_last_error()
    return msg.decode() if msg else ""
