"""Gather-scatter (direct stiffness summation, DSSUM) on the device.

No reference implementation exists; the paper names it Neko's
second ingredient.  Contract (shared with the oracle,
oracle/oracle.py:dssum): each SHARED global node's value is the sum, from
0.0, of all its local copies in ascending flat local index, written back to
every copy; unshared points are untouched.  The order is fixed, so the
result is bit-exact and independent of the number of ranks.

Setup (once per mesh, torch ops on the device): a stable sort of the
global ids gives every node's copies in ascending local order; nodes are
split into
  * local shared nodes                          -> axhelm_gs_sum (CSR)
  * nodes on the slab's top interface plane     -> PARTIAL / WRITE  (lower role)
  * nodes on the slab's bottom interface plane  -> FINISH           (upper role)
The per-apply hot path is three CUDA kernels plus, across ranks, two
plane-sized point-to-point messages (dist.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .errors import DeviceError
from .mesh import BoxMesh

PARTIAL, FINISH, WRITE = 0, 1, 2


@dataclass
class CSR:
    offs: object  # int64 [n+1]
    idx: object  # int32 / int64 [copies]
    slot: object  # int64 [n] plane slot (interface CSRs) or None
    n: int

    @property
    def idx_bytes(self) -> int:
        return self.idx.element_size()

    def nbytes(self) -> int:
        b = self.offs.numel() * 8 + self.idx.numel() * self.idx_bytes
        return b + (self.slot.numel() * 8 if self.slot is not None else 0)


def _csr(torch, order, counts, starts, select, slot_of=None):
    """CSR over the nodes where select is True, copies in ascending local order."""
    cnt = counts[select]
    offs = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=counts.device)
    torch.cumsum(cnt, 0, out=offs[1:])
    per_entry = torch.repeat_interleave(select, counts)
    idx = order[per_entry]
    nloc = order.numel()
    idx = idx.to(torch.int32) if nloc < 2**31 else idx
    slot = slot_of[select].contiguous() if slot_of is not None else None
    return CSR(offs.contiguous(), idx.contiguous(), slot, int(cnt.numel()))


class GatherScatter:
    """DSSUM machinery for one rank's slab of a BoxMesh."""

    def __init__(self, mesh: BoxMesh, torch, device, gid=None):
        self.mesh = mesh
        self.torch = torch
        self.device = device
        lib = _lib.load()
        self.lib = lib
        gid = mesh.gid(torch, device) if gid is None else gid
        flat = gid.reshape(-1)
        order = torch.argsort(flat, stable=True)
        sg = flat[order]
        uniq, counts = torch.unique_consecutive(sg, return_counts=True)
        starts = torch.cumsum(counts, 0) - counts
        gz = uniq // mesh.plane
        top = (gz == mesh.ez1 * mesh.n1) & (mesh.rank < mesh.world - 1)
        bot = (gz == mesh.ez0 * mesh.n1) & (mesh.rank > 0)
        local = (counts > 1) & ~top & ~bot
        slot = uniq % mesh.plane
        self.local = _csr(torch, order, counts, starts, local)
        self.top = _csr(torch, order, counts, starts, top, slot) if mesh.rank < mesh.world - 1 else None
        self.bot = _csr(torch, order, counts, starts, bot, slot) if mesh.rank > 0 else None
        # multiplicity of every local point's global node, restricted to this rank;
        # the global multiplicity needs the interface exchange (dist.py)
        self.n_shared_local = self.local.n
        del order, sg, uniq, counts, starts, gz, slot

    # -------------------------------------------------------------- ops

    def _stream(self, stream):
        if stream is None:
            stream = self.torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(stream.cuda_stream)

    def sum_local(self, w, stream=None):
        c = self.local
        rc = self.lib.axhelm_gs_sum(w.data_ptr(), c.offs.data_ptr(), c.idx.data_ptr(), c.idx_bytes,
                                    c.n, self._stream(stream))
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def plane(self, op: int, which: str, w, buf, stream=None):
        c = self.top if which == "top" else self.bot
        if c is None:
            return
        rc = self.lib.axhelm_gs_plane(op, w.data_ptr(), c.offs.data_ptr(), c.idx.data_ptr(),
                                      c.idx_bytes, c.slot.data_ptr(), c.n, buf.data_ptr(),
                                      self._stream(stream))
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def new_plane_buffer(self):
        return self.torch.zeros(self.mesh.plane, dtype=self.torch.float64, device=self.device)

    def bytes_per_apply(self) -> int:
        """Algorithmic HBM bytes of one local DSSUM: every shared copy read and
        written once (16 B) plus the CSR arrays."""
        b = 0
        for c in (self.local, self.top, self.bot):
            if c is not None:
                b += c.idx.numel() * 16 + c.nbytes()
        return b


class BoxGatherScatter:
    """Structured DSSUM for a BoxMesh slab (axhelm_gs_box): the copies of each
    global node are computed arithmetically, so no setup sort and no index
    traffic.  Same ops interface and summation order as GatherScatter."""

    def __init__(self, mesh: BoxMesh, torch, device):
        self.mesh = mesh
        self.torch = torch
        self.device = device
        self.lib = _lib.load()
        self.has_below = mesh.rank > 0
        self.has_above = mesh.rank < mesh.world - 1

    def _stream(self, stream):
        if stream is None:
            stream = self.torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(stream.cuda_stream)

    def _call(self, op, w, buf, stream):
        m = self.mesh
        rc = self.lib.axhelm_gs_box(op, w.data_ptr(), m.nx, m.ny, m.lx, m.ez0, m.ez1,
                                    int(self.has_below), int(self.has_above),
                                    buf.data_ptr() if buf is not None else None, self._stream(stream))
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def sum_local(self, w, stream=None):
        self._call(0, w, None, stream)

    def plane(self, op: int, which: str, w, buf, stream=None):
        if (which == "top" and not self.has_above) or (which == "bot" and not self.has_below):
            return
        self._call(1 + op, w, buf, stream)

    def new_plane_buffer(self):
        return self.torch.zeros(self.mesh.plane, dtype=self.torch.float64, device=self.device)

    def bytes_per_apply(self) -> int:
        """Algorithmic HBM bytes of the local DSSUM: each local copy of a
        shared node read and written once (16 B)."""
        m = self.mesh
        n1 = m.n1
        # local points whose node is shared: all except element-interior points
        # and the unshared points on the brick's outer faces
        inner = (m.lx - 2) ** 3
        return m.nel * (m.lx ** 3 - inner) * 16
