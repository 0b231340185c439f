"""The assembled SEM Helmholtz/Poisson operator on a (distributed) box mesh:
w = Q Q^T A_local u — ax_helm on every local element, then DSSUM.

This is the caller Neko builds around ax_helm (the reference's kernel is the
element-local part; gather-scatter and the mesh are reference non-goals,
SPEC.md:14).  Per apply on rank r of a z-slab partition:

  stream S0: ax on the slab's two boundary element layers
             -> PARTIAL top plane -> NCCL send up / recv from below
             -> FINISH bottom plane -> NCCL send down / recv from above
             -> WRITE top plane
  stream S1: ax on the interior element layers            (overlaps the exchange)
  S0 waits S1 -> local DSSUM of every other shared node

Interface nodes are only touched by the plane steps and local nodes only by
the local step, so the two streams never write the same point; the result
is bit-identical to the single-domain DSSUM (dist.py).
"""

from __future__ import annotations

import ctypes

from . import _lib, kernelrt
from .dist import SlabDSSUM
from .errors import DeviceError
from .gs import BoxGatherScatter
from .mesh import BoxMesh

FIELDS = ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")


class HelmholtzOperator:
    """w = DSSUM(A_local u) on this rank's slab; geometry resident in HBM."""

    def __init__(self, mesh: BoxMesh, torch, device, comm=None, mode: str = "fast",
                 geometry: dict | None = None, amp: float = 0.1, overlap: bool = True):
        self.mesh = mesh
        self.torch = torch
        self.device = device
        self.mode = kernelrt.MODES[mode]
        self.lib = _lib.load()
        self.geom = geometry if geometry is not None else mesh.geometry(torch, device, amp=amp)
        self.mats = mesh.matrices(torch, device)
        self.gs = BoxGatherScatter(mesh, torch, device)
        self.dssum = SlabDSSUM(self.gs, comm, rank=mesh.rank, world=mesh.world)
        self.comm = comm
        self.overlap = overlap and mesh.world > 1 and (mesh.ez1 - mesh.ez0) > 2
        self.side = torch.cuda.Stream(device) if self.overlap else None
        self.L3 = mesh.lx ** 3
        self._part = {}
        self._dots = torch.zeros(3, dtype=torch.float64, device=device)

    # ----------------------------------------------------------- pieces

    def ax(self, u, w, e0: int = 0, e1: int | None = None, stream=None, dot=None):
        """ax_helm on local elements [e0, e1) (stream-ordered).  dot: a device
        scalar receiving sum u*w over those elements (fused into the kernel
        for lx = 8 fast mode)."""
        m = self.mesh
        e1 = m.nel if e1 is None else e1
        n = e1 - e0
        if n <= 0:
            return
        off = e0 * self.L3 * 8

        def p(t, shifted=True):
            return t.data_ptr() + (off if shifted else 0)

        ptrs = [p(w), p(u), p(self.mats["dxd"], False), p(self.mats["dyd"], False),
                p(self.mats["dzd"], False), p(self.mats["dxtd"], False), p(self.mats["dytd"], False),
                p(self.mats["dztd"], False)] + [p(self.geom[f]) for f in FIELDS]
        if stream is None:
            stream = self.torch.cuda.current_stream(self.device)
        sp = ctypes.c_void_p(stream.cuda_stream)
        if dot is None:
            rc = self.lib.axhelm_apply(*ptrs, n, m.lx, self.mode, sp)
        else:
            part = self._partials(stream)
            rc = self.lib.axhelm_apply_dot(*ptrs, n, m.lx, self.mode, part.data_ptr(), dot.data_ptr(), sp)
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def _partials(self, stream):
        """Per-stream scratch for the fused dot's block partials."""
        key = stream.cuda_stream
        if key not in self._part:
            nb = self.lib.axhelm_reduce_blocks(self.mesh.nel * self.L3)
            self._part[key] = self.torch.empty(max(nb, 2048), dtype=self.torch.float64, device=self.device)
        return self._part[key]

    def apply(self, u, w, dot=None):
        """w = Q Q^T A u on this rank (with the interface exchange).  dot: an
        optional device scalar receiving the rank-local sum_p u_p (A u)_p
        before assembly (= <u, QQ^T A u> for continuous u; PCG's p.Ap)."""
        m = self.mesh
        torch = self.torch
        if not self.overlap:
            self.ax(u, w, dot=dot)
            self.dssum(w)
            return w
        s0 = torch.cuda.current_stream(self.device)
        lay = m.nx * m.ny
        d3 = self._dots if dot is not None else None
        # boundary element layers first (their results feed the exchange)
        self.ax(u, w, 0, lay, dot=d3[0:1] if d3 is not None else None)
        self.ax(u, w, m.nel - lay, m.nel, dot=d3[1:2] if d3 is not None else None)
        self.side.wait_stream(s0)
        with torch.cuda.stream(self.side):
            self.ax(u, w, lay, m.nel - lay, stream=self.side, dot=d3[2:3] if d3 is not None else None)
        d = self.dssum
        if d.has_top:
            self.gs.plane(0, "top", w, d.buf_top)
        if m.world > 1:
            d.comm.sendrecv(send=d.buf_top if d.has_top else None, dst=m.rank + 1,
                            recv=d.buf_bot if d.has_bot else None, src=m.rank - 1)
        d.phase_finish(w)
        if m.world > 1:
            d.comm.sendrecv(send=d.buf_bot if d.has_bot else None, dst=m.rank - 1,
                            recv=d.buf_top if d.has_top else None, src=m.rank + 1)
        d.phase_write(w)
        s0.wait_stream(self.side)
        self.gs.sum_local(w)
        if dot is not None:
            dot.copy_(d3.sum().reshape(dot.shape))
        return w

    def bytes_per_apply(self) -> int:
        return 72 * self.mesh.nel * self.L3 + self.gs.bytes_per_apply()
