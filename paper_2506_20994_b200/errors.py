"""Exception taxonomy of the operator API.

Mirrors the reference's ``mdg.errors`` (/root/reference/pkg/src/mdg/errors.py:
MdgError :26, RangeError :30, ContractError :34, BindingError :81,
CodegenError :97) so callers that catch the reference's error classes by
name keep working when they swap this package in.
"""

from __future__ import annotations


class MdgError(Exception):
    """Base class for all package errors (errors.py:26)."""


class RangeError(MdgError, ValueError):
    """An argument fell outside its documented range (errors.py:30)."""


class ContractError(MdgError, ValueError):
    """A documented precondition was violated (errors.py:34)."""


class BindingError(MdgError, ValueError):
    """Kernel argument arrays are missing or shaped/typed wrongly (errors.py:81)."""


class CodegenError(MdgError, ValueError):
    """The kernel library or its entry symbol cannot be loaded (errors.py:97)."""


class DeviceError(MdgError, RuntimeError):
    """The CUDA library reported a runtime failure (no reference analogue:
    the reference's void ABI has no error channel, SURVEY §7 hard part 6)."""


class ParseError(MdgError, ValueError):
    """A tensor or sizes file failed to parse (errors.py ParseError)."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (byte offset {offset})"
        super().__init__(message)
        self.offset = offset


class VersionError(MdgError, ValueError):
    """A tensor file declared an unknown version (errors.py VersionError)."""
