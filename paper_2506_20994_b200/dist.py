"""Multi-GPU DSSUM over z-slabs: the interface-plane exchange.

Ranks own contiguous z-slabs of element layers (mesh.slab_range), so the
only nodes shared across ranks lie on the planes between neighbouring
slabs, and each such node is shared by exactly two ranks.  One apply's
exchange:

  1. every rank: local DSSUM of its own shared nodes (not on an interface);
     PARTIAL sums of its copies of the top-plane nodes -> send up
  2. every rank: FINISH its bottom plane — continue the received partial
     with its own copies, write the sums to its copies -> send them down
  3. every rank: WRITE the received final sums into its top-plane copies

Slabs are contiguous in the global z-major element order, so the lower
rank's copies precede the upper rank's: the running sum of 1+2 is exactly
the single-GPU ascending-order sum — DSSUM stays bit-exact at any rank
count.  Messages: two planes of NX*NY doubles per interface per apply
(6.4 MB at 128^3 elements, lx=8) over NCCL (NVLink) — or any `Comm`.

The protocol only needs `ops` with sum_local / plane / new_plane_buffer
(gs.GatherScatter on the GPU) and a `Comm`; the gloo CPU tests drive it with
oracle-backed ops (tests/test_dist_cpu.py).
"""

from __future__ import annotations

import ctypes

from .gs import FINISH, PARTIAL, WRITE


class TorchComm:
    """Point-to-point and all-reduce over torch.distributed (NCCL on GPUs,
    gloo on CPUs).  Stream-ordered on NCCL: wait() makes the current stream
    wait for the transfer, the host does not block."""

    def __init__(self, dist=None):
        if dist is None:
            import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        # gloo moves CPU tensors only: stage device buffers through the host
        # (used to exercise multi-rank runs on a single GPU / CPU-only boxes)
        self.host_staged = dist.get_backend() == "gloo"

    def sendrecv(self, send=None, dst=None, recv=None, src=None):
        d = self.dist
        s_t, r_t = send, recv
        if self.host_staged:
            s_t = send.cpu() if send is not None else None
            r_t = recv.new_empty(recv.shape, device="cpu") if recv is not None else None
        ops = []
        if s_t is not None:
            ops.append(d.P2POp(d.isend, s_t, dst))
        if r_t is not None:
            ops.append(d.P2POp(d.irecv, r_t, src))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        if self.host_staged and recv is not None and r_t is not recv:
            recv.copy_(r_t)

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def allreduce_sum(self, t):
        if self.host_staged and t.device.type != "cpu":
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t


class PeerExchange:
    """The interface-plane exchange over PEER memory: each rank
    exports one IPC-shareable device region (receive buffers for the planes
    from below / above and the flags its neighbours signal) and opens its
    neighbours' regions; the plane kernels (axhelm_gs_box_peer) write the
    partial / final sums straight into the neighbour's buffer over NVLink and
    signal with a system-scope release store.  No NCCL, no host round trip:
    one apply's exchange is three kernel launches on the caller's stream.

      rank r:  PARTIAL top plane  -> recv_bot of r+1, flag_bot(r+1) = seq
               FINISH bottom plane (waits flag_bot(r) >= seq)
                                  -> recv_top of r-1, flag_top(r-1) = seq
               WRITE top plane     (waits flag_top(r) >= seq)

    Summation order = the NCCL path's (bit-identical).  Works between
    processes on different GPUs (NVLink peer mappings) and on one GPU.

    The same regions carry the PCG's small all-reduces (`allreduce_sum`):
    each rank writes its values into every rank's region and sums the slots
    in rank order (axhelm_peer_allreduce) — identical bits on every rank."""

    # region head: flags (0: from below, 8: from above), CTA counters at 256 /
    # 260, device sequence numbers at 384 (exchange) / 392 (all-reduce)
    HEAD = 512

    def __init__(self, mesh, comm, lib, torch=None):
        import torch as _torch

        self.mesh = mesh
        self.lib = lib
        self.rank, self.world = comm.rank, comm.world
        self.has_top = self.rank < self.world - 1
        self.has_bot = self.rank > 0
        self.plane_bytes = ((mesh.plane * 8 + 255) // 256) * 256
        self.ar_off = self.HEAD + 2 * self.plane_bytes
        size = self.ar_off + lib.axhelm_peer_allreduce_bytes()
        self.base = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        self._check(lib.axhelm_peer_alloc(size, ctypes.byref(self.base), handle))
        handles = comm.allgather_object(bytes(handle))
        self.peers = {q: (self._open(h) if q != self.rank else self.base.value) for q, h in enumerate(handles)}
        self.peer_bot = self.peers[self.rank - 1] if self.has_bot else None
        self.peer_top = self.peers[self.rank + 1] if self.has_top else None
        dev = _torch.device("cuda", _torch.cuda.current_device())
        self.bases = _torch.tensor([self.peers[q] for q in range(self.world)], dtype=_torch.int64, device=dev)
        self.seq = 0
        self.ar_seq = 0

    def allreduce_sum(self, t):
        """In-place sum of a small float64 device tensor (<= 4 values) over all
        ranks, on the current stream."""
        import torch as _torch

        assert t.dtype == _torch.float64 and t.is_contiguous() and t.numel() <= 4
        self.ar_seq += 1
        stream = _torch.cuda.current_stream()
        self._check(self.lib.axhelm_peer_allreduce(t.data_ptr(), t.numel(), t.data_ptr(), self.bases.data_ptr(),
                                                   self.ar_off, self.world, self.rank, 0, self.base.value + 392,
                                                   ctypes.c_void_p(stream.cuda_stream)))
        return t

    def _check(self, rc):
        if rc:
            from . import _lib
            from .errors import DeviceError

            raise DeviceError(_lib.last_error(self.lib))

    def _open(self, handle: bytes):
        p = ctypes.c_void_p()
        buf = (ctypes.c_char * 64).from_buffer_copy(handle)
        self._check(self.lib.axhelm_peer_open(buf, ctypes.byref(p)))
        return p.value

    # region layout
    @staticmethod
    def _flag_bot(b):
        return b
    @staticmethod
    def _flag_top(b):
        return b + 8

    def _recv_bot(self, b):
        return b + self.HEAD

    def _recv_top(self, b):
        return b + self.HEAD + self.plane_bytes

    def exchange(self, w, stream):
        """Interface planes of w (this rank's slab), stream-ordered."""
        m = self.mesh
        self.seq += 1
        b = self.base.value
        sp = ctypes.c_void_p(stream.cuda_stream)
        args = (m.nx, m.ny, m.lx, m.ez0, m.ez1)
        sq = b + 384  # the sequence lives in device memory: CUDA-graph replays advance it
        if self.has_top:
            self._check(self.lib.axhelm_gs_box_peer(PARTIAL, w.data_ptr(), *args, None,
                                                    self._recv_bot(self.peer_top), None,
                                                    self._flag_bot(self.peer_top), 0, b + 256, sq, sp))
        if self.has_bot:
            self._check(self.lib.axhelm_gs_box_peer(FINISH, w.data_ptr(), *args, self._recv_bot(b),
                                                    self._recv_top(self.peer_bot), self._flag_bot(b),
                                                    self._flag_top(self.peer_bot), 0, b + 260, sq, sp))
        if self.has_top:
            self._check(self.lib.axhelm_gs_box_peer(WRITE, w.data_ptr(), *args, self._recv_top(b), None,
                                                    self._flag_top(b), None, 0, None, sq, sp))
        self._check(self.lib.axhelm_peer_seq_bump(sq, sp))

    def close(self):
        for q, p in getattr(self, "peers", {}).items():
            if q != self.rank and p:
                self.lib.axhelm_peer_close(ctypes.c_void_p(p))
        self.peers = {}
        self.peer_bot = self.peer_top = None
        if self.base:
            self.lib.axhelm_peer_free(self.base)
            self.base = ctypes.c_void_p()


class SlabDSSUM:
    """DSSUM of one rank's slab, including the interface exchange."""

    def __init__(self, ops, comm=None, rank=0, world=1):
        self.ops = ops
        self.comm = comm
        self.rank = comm.rank if comm is not None else rank
        self.world = comm.world if comm is not None else world
        self.has_top = self.rank < self.world - 1
        self.has_bot = self.rank > 0
        self.buf_top = ops.new_plane_buffer() if self.has_top else None
        self.buf_bot = ops.new_plane_buffer() if self.has_bot else None

    # phases (also driven directly by the single-process loopback below)
    def phase_local_partial(self, w):
        self.ops.sum_local(w)
        if self.has_top:
            self.ops.plane(PARTIAL, "top", w, self.buf_top)

    def phase_finish(self, w):
        if self.has_bot:
            self.ops.plane(FINISH, "bot", w, self.buf_bot)

    def phase_write(self, w):
        if self.has_top:
            self.ops.plane(WRITE, "top", w, self.buf_top)

    def __call__(self, w):
        self.phase_local_partial(w)
        if self.world > 1:
            self.comm.sendrecv(send=self.buf_top if self.has_top else None, dst=self.rank + 1,
                               recv=self.buf_bot if self.has_bot else None, src=self.rank - 1)
        self.phase_finish(w)
        if self.world > 1:
            self.comm.sendrecv(send=self.buf_bot if self.has_bot else None, dst=self.rank - 1,
                               recv=self.buf_top if self.has_top else None, src=self.rank + 1)
        self.phase_write(w)
        return w


def loopback_dssum(slabs: list, ws: list) -> None:
    """Run the exchange for several slabs held by ONE process (e.g. on one
    GPU): the same phases, with the messages as device copies."""
    for s, w in zip(slabs, ws):
        s.phase_local_partial(w)
    for r in range(len(slabs) - 1):
        slabs[r + 1].buf_bot.copy_(slabs[r].buf_top)
    for s, w in zip(slabs, ws):
        s.phase_finish(w)
    for r in range(1, len(slabs)):
        slabs[r - 1].buf_top.copy_(slabs[r].buf_bot)
    for s, w in zip(slabs, ws):
        s.phase_write(w)
