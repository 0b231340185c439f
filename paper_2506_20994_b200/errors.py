"""Exception classes of the operator API: the reference's own, when present.

The reference's kernel runtime raises ``mdg.errors.BindingError`` /
``CodegenError`` (/root/reference/pkg/src/mdg/kernelrt.py:85-104; classes at
errors.py:26-100).  A caller written against it catches those exact classes,
so when ``mdg`` is importable this module re-exports them and everything
this package raises is an instance of the reference's class.  Without
``mdg`` (the GPU box, or a deployment that never installed the reference)
local classes with the same names, bases and constructor signatures stand
in.  ``DeviceError`` (CUDA runtime failures; the reference's void ABI has
no error channel) always derives from the active ``MdgError``.
"""

from __future__ import annotations

try:  # the reference's taxonomy, so `except mdg.errors.BindingError` works
    from mdg.errors import (  # type: ignore[import-not-found]
        BindingError, CodegenError, ContractError, MdgError, ParseError, RangeError, VersionError,
    )

    FROM_REFERENCE = True
except ImportError:
    FROM_REFERENCE = False

    class MdgError(Exception):  # type: ignore[no-redef]
        """Base class (reference errors.py:26)."""

    class RangeError(MdgError, ValueError):  # type: ignore[no-redef]
        """Argument outside its documented range (errors.py:30)."""

    class ContractError(MdgError, ValueError):  # type: ignore[no-redef]
        """Documented precondition violated (errors.py:34)."""

    class BindingError(MdgError, ValueError):  # type: ignore[no-redef]
        """Kernel argument arrays missing or wrongly typed / shaped."""

    class CodegenError(MdgError, ValueError):  # type: ignore[no-redef]
        """Kernel library or entry symbol cannot be loaded."""

    class ParseError(MdgError, ValueError):  # type: ignore[no-redef]
        """A file failed to parse; offset = byte offset when known."""

        def __init__(self, message: str, offset: int | None = None):
            if offset is not None:
                message = f"{message} (byte offset {offset})"
            super().__init__(message)
            self.offset = offset

    class VersionError(MdgError, ValueError):  # type: ignore[no-redef]
        """A file declared an unknown format version."""


class DeviceError(MdgError, RuntimeError):
    """The CUDA library reported a runtime failure (no reference analogue)."""


__all__ = ["MdgError", "RangeError", "ContractError", "BindingError", "CodegenError", "ParseError",
           "VersionError", "DeviceError", "FROM_REFERENCE"]
