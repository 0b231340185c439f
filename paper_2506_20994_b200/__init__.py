"""paper_2506_20994_b200 — B200-native (sm_100a) ax_helm for the mdg operator API.

Drop-in for the reference's hot path (/root/reference/pkg/src/mdg):
``load_kernel(libpath=None, entry="__dace_ax_helm") -> KernelFn`` with the
call shape ``fn(arrays, nelv, lx)`` of mdg.kernelrt.load_kernel, backed by
hand-written FP64 CUDA kernels in libaxhelm_sm100.so (include/axhelm.h).
"""

from .errors import (  # noqa: F401
    BindingError, CodegenError, ContractError, DeviceError, MdgError, ParseError,
    RangeError, VersionError,
)
from .kernelrt import ABI_CONTAINER_ORDER, KernelFn, apply, expected_shape, load_kernel  # noqa: F401
from .basis import Basis, gll_basis  # noqa: F401

__version__ = "0.1.0"


def bytes_model(nel: int, lx: int) -> int:
    """Algorithmic HBM bytes of one apply: (u + 6 G + h1 + w) * 8 B per point."""
    return 72 * int(nel) * int(lx) ** 3


def flops_model(lx: int, nel: int) -> int:
    """nel * lx^3 * (12 lx + 18) (reference sem.py:367-375, same argument order)."""
    return int(nel) * int(lx) ** 3 * (12 * int(lx) + 18)
