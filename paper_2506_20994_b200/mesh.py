"""Device-resident box mesh and geometric-factor store.

The reference has no mesh: its fixtures are random per-point
SPD metric blocks (sem.py:265-285) or identical axis-aligned cubes
(sem.py:239-262).  The B200 build needs a real mesh for the gather-scatter
and the Poisson solve: an nx x ny x nz brick of lx^3 spectral elements,
element order e = (ez*ny + ey)*nx + ex, partitioned into
z-slabs for multi-GPU runs, with a smooth interior deformation.  Node ids,
geometric factors and all work arrays live in HBM; they are generated on the
device (``axhelm_box_gid``, ``axhelm_box_geometry``) because a NumPy
generator at 2^18+ elements needs tens of GB of host RAM.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .basis import gll_basis
from .errors import DeviceError, RangeError

GEOM_FIELDS = ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")


def slab_range(nz: int, rank: int, world: int) -> tuple[int, int]:
    """Element layers [ez0, ez1) of rank's z-slab (contiguous, balanced)."""
    if world < 1 or not (0 <= rank < world):
        raise RangeError(f"bad rank {rank} of {world}")
    if nz < world:
        raise RangeError(f"nz={nz} element layers cannot be split over {world} ranks")
    base, extra = divmod(nz, world)
    ez0 = rank * base + min(rank, extra)
    return ez0, ez0 + base + (1 if rank < extra else 0)


@dataclass
class BoxMesh:
    """One rank's z-slab [ez0, ez1) of an nx x ny x nz brick of lx^3 elements."""

    nx: int
    ny: int
    nz: int
    lx: int
    rank: int = 0
    world: int = 1
    ez0: int = field(init=False)
    ez1: int = field(init=False)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise RangeError("mesh dimensions must be >= 1")
        gll_basis(self.lx)  # validates lx
        self.ez0, self.ez1 = slab_range(self.nz, self.rank, self.world)

    @property
    def n1(self) -> int:
        return self.lx - 1

    @property
    def NX(self) -> int:
        return self.nx * self.n1 + 1

    @property
    def NY(self) -> int:
        return self.ny * self.n1 + 1

    @property
    def plane(self) -> int:
        """Global nodes per z-plane."""
        return self.NX * self.NY

    @property
    def nel(self) -> int:
        """Local (slab) element count."""
        return self.nx * self.ny * (self.ez1 - self.ez0)

    @property
    def nel_global(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def e_offset(self) -> int:
        """Global index of the first local element."""
        return self.nx * self.ny * self.ez0

    @property
    def shape(self) -> tuple[int, int, int, int]:
        return (self.nel, self.lx, self.lx, self.lx)

    def layer_range(self, ez: int) -> tuple[int, int]:
        """Local element range of global element layer ez (must be in the slab)."""
        if not (self.ez0 <= ez < self.ez1):
            raise RangeError(f"layer {ez} not in slab [{self.ez0}, {self.ez1})")
        a = (ez - self.ez0) * self.nx * self.ny
        return a, a + self.nx * self.ny

    # ------------------------------------------------------ device builders

    def gid(self, torch, device):
        """int64 [nel, lx, lx, lx] global node ids on the device."""
        lib = _lib.load()
        out = torch.empty(self.shape, dtype=torch.int64, device=device)
        s = torch.cuda.current_stream(device).cuda_stream
        rc = lib.axhelm_box_gid(out.data_ptr(), self.nx, self.ny, self.lx, self.ez0, self.nel,
                                ctypes.c_void_p(s))
        if rc:
            raise DeviceError(_lib.last_error(lib))
        return out

    def geometry(self, torch, device, amp: float = 0.1) -> dict:
        """h1d and the six metric fields of the deformed brick, on the device."""
        lib = _lib.load()
        b = gll_basis(self.lx)
        pts = torch.from_numpy(np.ascontiguousarray(b.points)).to(device)
        wts = torch.from_numpy(np.ascontiguousarray(b.weights)).to(device)
        out = {k: torch.empty(self.shape, dtype=torch.float64, device=device) for k in GEOM_FIELDS}
        s = torch.cuda.current_stream(device).cuda_stream
        rc = lib.axhelm_box_geometry(*[out[k].data_ptr() for k in GEOM_FIELDS], pts.data_ptr(),
                                     wts.data_ptr(), self.nx, self.ny, self.nz, self.lx, self.ez0,
                                     self.nel, float(amp), ctypes.c_void_p(s))
        if rc:
            raise DeviceError(_lib.last_error(lib))
        torch.cuda.current_stream(device).synchronize()  # pts/wts go out of scope
        return out

    def matrices(self, torch, device) -> dict:
        a, b = gll_basis(self.lx).operator_matrices()
        d = {}
        for n in ("dxd", "dyd", "dzd"):
            d[n] = torch.from_numpy(a.copy()).to(device)
        for n in ("dxtd", "dytd", "dztd"):
            d[n] = torch.from_numpy(b.copy()).to(device)
        return d
