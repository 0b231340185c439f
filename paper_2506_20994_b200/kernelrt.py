"""Operator API: a drop-in for the reference's ``mdg.kernelrt.load_kernel``.

Reference: /root/reference/pkg/src/mdg/kernelrt.py:25 (``KernelFn``),
:77-108 (``load_kernel``).  The reference compiles generated C and returns
``invoke(arrays, nelv, lx)`` that checks every ABI array is a C-contiguous
float64 ndarray (:98-104) and calls the 15-pointer C function (:105-106).

Here ``load_kernel`` binds the prebuilt sm_100a library (include/axhelm.h)
and returns a ``KernelFn`` with the same call shape and the same error
behaviour (``BindingError`` naming the array, ``CodegenError`` for a missing
symbol), that accepts either

* torch CUDA tensors (device buffers) — the apply is enqueued on torch's
  current CUDA stream through ``axhelm_apply`` and ``arrays["wd"]`` is
  written in stream order, like any other torch op; or
* NumPy arrays / CPU tensors (host buffers) — routed through the exact
  reference symbol ``__dace_ax_helm``, which stages them through the GPU
  and returns with ``wd`` written, like the reference's CPU kernel.

There is no CPU compute path: without the library or a GPU this raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Any, Callable, Mapping

import numpy as np

from . import _lib
from .errors import BindingError, CodegenError, DeviceError, RangeError

# axprogram.py:32-48
ABI_CONTAINER_ORDER = (
    "wd", "ud", "dxd", "dyd", "dzd", "dxtd", "dytd", "dztd",
    "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d",
)
MATRICES = frozenset(("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd"))
MODES = {"strict": 0, "fast": 1}

KernelFn = Callable[[Mapping[str, Any], int, int], None]


def expected_shape(name: str, nelv: int, lx: int) -> tuple[int, ...]:
    """[lx,lx] for the six matrices, [nelv,lx,lx,lx] otherwise (abi.ts:25-29)."""
    return (lx, lx) if name in MATRICES else (nelv, lx, lx, lx)


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _check(name: str, a, nelv: int, lx: int):
    """Validate one argument; returns (pointer, on_device)."""
    if _is_torch(a):
        import torch

        if a.dtype != torch.float64 or not a.is_contiguous():
            raise BindingError(f"array {name!r} must be C-contiguous float64")
        on_dev = a.is_cuda
        ptr = a.data_ptr()
    else:
        if not isinstance(a, np.ndarray):
            raise BindingError(f"array {name!r} must be an ndarray or torch tensor")
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise BindingError(f"array {name!r} must be C-contiguous float64")
        on_dev = False
        ptr = a.ctypes.data
    want = expected_shape(name, nelv, lx)
    if tuple(a.shape) != want:
        raise BindingError(
            f"array {name!r} has shape {tuple(a.shape)}, expected {want} for nelv={nelv}, lx={lx}"
        )
    if name == "wd" and not on_dev and isinstance(a, np.ndarray) and not a.flags.writeable:
        raise BindingError("array 'wd' must be writeable")
    return ptr, on_dev


def load_kernel(
    libpath: str | os.PathLike | None = None,
    entry: str = "__dace_ax_helm",
    mode: str | None = None,
) -> KernelFn:
    """Bind the entry symbol and wrap it for dict-of-array invocation.

    Same signature and contract as mdg.kernelrt.load_kernel (kernelrt.py:77):
    the callable takes (arrays, nelv, lx) with every ABI container name
    mapped to a C-contiguous float64 array; ``wd`` is written in place.
    ``mode`` selects "strict" (bit-exact with the reference, the default) or
    "fast" (FMA) arithmetic; None keeps the library default (AXHELM_FP).
    """
    lib = _lib.load(libpath)
    path = libpath if libpath is not None else _lib.lib_path()
    fn = getattr(lib, entry, None)
    if fn is None:
        raise CodegenError(f"symbol {entry!r} not found in {path}")
    if mode is not None and mode not in MODES:
        raise RangeError(f"mode must be one of {sorted(MODES)}, got {mode!r}")
    if entry != "__dace_ax_helm":  # custom entry with the reference ABI
        fn.restype = None
        fn.argtypes = [ctypes.c_void_p] * 15 + [ctypes.c_int, ctypes.c_int]
    apply_dev = lib.axhelm_apply

    def invoke(arrays: Mapping[str, Any], nelv: int, lx: int) -> None:
        ptrs, dev = [], []
        for name in ABI_CONTAINER_ORDER:
            if name not in arrays:
                raise BindingError(f"missing kernel argument array {name!r}")
            p, d = _check(name, arrays[name], nelv, lx)
            ptrs.append(p)
            dev.append(d)
        m = MODES[mode] if mode is not None else lib.axhelm_get_mode()
        if all(dev) and entry == "__dace_ax_helm":
            import torch

            stream = torch.cuda.current_stream(arrays["wd"].device).cuda_stream
            rc = apply_dev(*ptrs, int(nelv), int(lx), m, ctypes.c_void_p(stream))
        else:
            if entry == "__dace_ax_helm":
                # the reference symbol's body with an explicit mode + status
                rc = lib.axhelm_apply_sync(*ptrs, int(nelv), int(lx), m)
            else:
                fn(*ptrs, int(nelv), int(lx))
                rc = lib.axhelm_last_status()
        if rc != 0:
            msg = _lib.last_error(lib)
            if rc == 1:
                raise RangeError(msg)
            raise DeviceError(msg)

    invoke.lib = lib  # type: ignore[attr-defined]
    invoke.entry = entry  # type: ignore[attr-defined]
    return invoke


def apply(arrays: Mapping[str, Any], nelv: int, lx: int, mode: str = "strict", stream=None) -> None:
    """One stream-ordered apply over torch CUDA tensors (no host staging)."""
    import torch

    lib = _lib.load()
    ptrs = []
    for name in ABI_CONTAINER_ORDER:
        if name not in arrays:
            raise BindingError(f"missing kernel argument array {name!r}")
        p, d = _check(name, arrays[name], nelv, lx)
        if not d:
            raise BindingError(f"array {name!r} must be a CUDA tensor for apply()")
        ptrs.append(p)
    if stream is None:
        stream = torch.cuda.current_stream(arrays["wd"].device)
    rc = lib.axhelm_apply(*ptrs, int(nelv), int(lx), MODES[mode], ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise (RangeError if rc == 1 else DeviceError)(_lib.last_error(lib))
