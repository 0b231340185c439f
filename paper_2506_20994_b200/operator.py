"""The assembled SEM Helmholtz/Poisson operator on a (distributed) box mesh:
w = Q Q^T A_local u — ax_helm on every local element, then DSSUM.

This is the caller Neko builds around ax_helm (the reference's kernel is the
element-local part; gather-scatter and the mesh are reference non-goals,
SPEC.md:14).  Per apply on rank r of a z-slab partition:

  stream S0: ax on the slab's two boundary element layers
             -> PARTIAL top plane -> send up / recv from below
             -> FINISH bottom plane -> send down / recv from above
             -> WRITE top plane
             (exchange="peer": the three plane kernels write the neighbours'
             buffers and flags over NVLink themselves — dist.PeerExchange;
             exchange="nccl": plane buffers over NCCL send / recv)
  stream S1: ax on the interior element layers + the local DSSUM of every
             other shared node                              (overlaps the exchange)
  S0 waits S1

The local part is one axhelm_ax_gs_box call.  Its schedules: "sequential"
(default) — the apply streams w out, then one DSSUM pass; "follow" — a
concurrent follower kernel sums each element layer's node planes as soon as
the apply has finished that layer, while its w is still in L2; n — layer
blocks with kernel boundaries.  Measured at C2 the follower,
limited to the threads that fit beside the apply's persistent CTAs, cannot
hide its L2 latency and the sequential pass wins.
Interface nodes are only touched by the plane steps and local nodes only by
the local step, so the streams never write the same point; the result is
bit-identical to the single-domain DSSUM (dist.py) for every schedule.
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

    SCHEDULES = {"follow": -1, "sequential": 0}

    def __init__(self, mesh: BoxMesh, torch, device, comm=None, mode: str = "fast",
                 geometry: dict | None = None, amp: float = 0.1, overlap: bool = True,
                 schedule: str | int = "sequential", exchange: str = "nccl"):
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
        # apply(local_dssum=False) through the x-folding kernel (class-2 DSSUM
        # nodes summed by the apply; axhelm_apply_box).  Off by default: the
        # PCG update's gathers of those copies hit L2 anyway, and the fold
        # measured 2% slower per PCG iteration (3.40 -> 3.47 ms, same box);
        # the assembled apply (local_dssum=True) always folds.
        self.fold_unassembled = False
        self.xfolded = False  # last apply(local_dssum=False): class-2 nodes summed by the apply
        self.side = torch.cuda.Stream(device) if self.overlap else None
        self.L3 = mesh.lx ** 3
        self._part = {}
        self._dots = torch.zeros(3, dtype=torch.float64, device=device)
        # ax + local DSSUM schedule (axhelm_ax_gs_box): "sequential" = apply
        # then a separate DSSUM pass (default: fastest measured);
        # "follow" = the DSSUM runs concurrently, layer by layer behind the
        # apply, on w still in L2; n > 0 = blocks of n element layers separated
        # by kernel boundaries
        self.schedule = self.SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
        n1 = mesh.n1
        nl = mesh.ez1 - mesh.ez0
        self.zlo = mesh.ez0 * n1 + (1 if mesh.rank > 0 else 0)
        self.zhi = mesh.ez1 * n1 - (1 if mesh.rank < mesh.world - 1 else 0)
        self._progress = torch.zeros(max(nl, 1), dtype=torch.int32, device=device)
        # interface-plane transport: "nccl" (TorchComm send/recv of plane
        # buffers) or "peer" (dist.PeerExchange: the plane kernels write the
        # neighbour's buffers over NVLink themselves)
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', not {exchange!r}")
        self.peer = None
        if exchange == "peer" and comm is not None and mesh.world > 1:
            from .dist import PeerExchange

            self.peer = PeerExchange(mesh, comm, self.lib)

    # ----------------------------------------------------------- pieces

    def ax(self, u, w, e0: int = 0, e1: int | None = None, stream=None, dot=None, xfold: bool = False):
        """ax_helm on local elements [e0, e1) (stream-ordered).  dot: a device
        scalar receiving sum u*w over those elements (fused into the kernel
        for lx = 8 fast mode).  xfold: [e0, e1) are whole x-runs and the
        x-folding apply may sum the class-2 DSSUM nodes (axhelm_apply_box);
        returns whether it did."""
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
        if xfold:
            flag = ctypes.c_int(0)
            part = self._partials(stream) if dot is not None else None
            rc = self.lib.axhelm_apply_box(*ptrs, m.nx, n, m.lx, self.mode,
                                           part.data_ptr() if part is not None else None,
                                           dot.data_ptr() if dot is not None else None, ctypes.byref(flag), sp)
            if rc:
                raise DeviceError(_lib.last_error(self.lib))
            return bool(flag.value)
        if dot is None:
            rc = self.lib.axhelm_apply(*ptrs, n, m.lx, self.mode, sp)
        else:
            part = self._partials(stream)
            rc = self.lib.axhelm_apply_dot(*ptrs, n, m.lx, self.mode, part.data_ptr(), dot.data_ptr(), sp)
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def ax_gs(self, u, w, l0: int, l1: int, stream=None, dot=None):
        """ax on local element layers [l0, l1) and the local DSSUM of every
        owned node plane, per self.schedule (layers outside [l0, l1) must
        already be applied on this stream's timeline)."""
        m = self.mesh
        ptrs = [w.data_ptr(), u.data_ptr()] + [self.mats[k].data_ptr() for k in
                                               ("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd")]
        ptrs += [self.geom[f].data_ptr() for f in FIELDS]
        if stream is None:
            stream = self.torch.cuda.current_stream(self.device)
        part = self._partials(stream) if dot is not None else None
        rc = self.lib.axhelm_ax_gs_box(*ptrs, m.nx, m.ny, m.lx, m.ez0, m.ez1, l0, l1, self.zlo, self.zhi,
                                       self.mode, self.schedule, self._progress.data_ptr(),
                                       part.data_ptr() if part is not None else None,
                                       dot.data_ptr() if dot is not None else None,
                                       ctypes.c_void_p(stream.cuda_stream))
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def _partials(self, stream):
        """Per-stream scratch for the fused dot's block partials."""
        key = stream.cuda_stream
        if key not in self._part:
            nb = max(self.lib.axhelm_reduce_blocks(self.mesh.nel * self.L3),
                     self.lib.axhelm_ax_gs_scratch(self.mesh.ez1 - self.mesh.ez0))
            self._part[key] = self.torch.empty(max(nb, 2048), dtype=self.torch.float64, device=self.device)
        return self._part[key]

    def apply(self, u, w, dot=None, local_dssum: bool = True):
        """w = Q Q^T A u on this rank (with the interface exchange).  dot: an
        optional device scalar receiving the rank-local sum_p u_p (A u)_p
        before assembly (= <u, QQ^T A u> for continuous u; PCG's p.Ap).
        local_dssum=False leaves the local shared nodes unassembled (only the
        interface planes are summed) for a consumer that gathers them itself
        (axhelm_cg_update_box); self.xfolded then says whether the class-2
        nodes came out summed already (x-folding apply)."""
        m = self.mesh
        torch = self.torch
        nl = m.ez1 - m.ez0
        if not self.overlap:
            if local_dssum:
                self.ax_gs(u, w, 0, nl, dot=dot)
            else:
                self.xfolded = bool(self.ax(u, w, dot=dot, xfold=self.fold_unassembled))
            self._exchange(w)
            return w
        s0 = torch.cuda.current_stream(self.device)
        lay = m.nx * m.ny
        d3 = self._dots if dot is not None else None
        # boundary element layers first (their results feed the exchange)
        xf = not local_dssum and self.fold_unassembled
        f0 = self.ax(u, w, 0, lay, dot=d3[0:1] if d3 is not None else None, xfold=xf)
        f1 = self.ax(u, w, m.nel - lay, m.nel, dot=d3[1:2] if d3 is not None else None, xfold=xf)
        self.side.wait_stream(s0)
        with torch.cuda.stream(self.side):
            # interior layers + every local DSSUM plane
            dd = d3[2:3] if d3 is not None else None
            if local_dssum:
                self.ax_gs(u, w, 1, nl - 1, stream=self.side, dot=dd)
            else:
                f2 = self.ax(u, w, lay, m.nel - lay, stream=self.side, dot=dd, xfold=xf)
                if not (bool(f0) == bool(f1) == bool(f2)):
                    raise DeviceError("x-folding chosen for some element ranges only")
                self.xfolded = bool(f0)
        self._exchange(w)
        s0.wait_stream(self.side)
        if dot is not None:
            dot.copy_(d3.sum().reshape(dot.shape))
        return w

    def _exchange(self, w):
        """Interface planes: PARTIAL (top) -> send up -> FINISH (bottom) ->
        send down -> WRITE (top).  Touches only interface-plane points."""
        m = self.mesh
        d = self.dssum
        if self.peer is not None:
            self.peer.exchange(w, self.torch.cuda.current_stream(self.device))
            return
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

    def bytes_per_apply(self) -> int:
        return 72 * self.mesh.nel * self.L3 + self.gs.bytes_per_apply()
