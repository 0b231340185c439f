"""Jacobi-preconditioned conjugate gradients for the assembled SEM Poisson
problem  Q Q^T A x = f,  x = 0 on the brick's outer boundary (SURVEY §8f,
config C5: 100 iterations, lx=8, 2^21 elements).

No reference implementation (SPEC.md:14 — the Poisson solve is a non-goal);
the weak form is PAPER.md:126-130 and the operator is HelmholtzOperator
(ax_helm + DSSUM + interface exchange).  Vectors are local-point fields
[nel][lx][lx][lx], continuous across elements (equal on all copies of a
node); global inner products weight each copy by 1/multiplicity so every
node counts once:  <a, b> = sum_p a_p b_p / mult_p  (all-reduced over ranks).

One iteration (no host synchronisation; scalars live in device memory),
fused form (default; 152 B of HBM traffic per point):
  w  = A p (+ interface planes), pw = sum_p p (A p)   (DMMA ax with the dot)
  r -= a QQ^T w ; rz', rr                   (axhelm_cg_update_box: each point
                                             gathers its node's copies — the
                                             local DSSUM without its own pass —
                                             cwt from the position)
  x += a p ; p = dinv r + (rz'/rz) p         (axhelm_cg_xpupdate)
Separate-pass form (fused=False; 184 B/point):
  w  = Q Q^T A p,  pw = sum_p p (A p)       (operator.apply: the dot is fused
                                             into the lx=8 DMMA kernel and taken
                                             before assembly, = <p, mask QQ^T A p>
                                             since p is continuous and vanishes
                                             on the boundary; + all-reduce)
  x += a p ; r -= a w ; rz', rr             (axhelm_cg_update, weights
                                             cwt = mask/mult; + all-reduce)
  p  = dinv r + (rz'/rz) p                  (axhelm_cg_pupdate)
r is left unmasked on the boundary: only dinv*r and cwt-weighted sums read
it, and both vanish there.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .errors import DeviceError
from .operator import HelmholtzOperator


class JacobiPCG:
    def __init__(self, op: HelmholtzOperator, fused: bool = True):
        """fused: fold the local DSSUM into the residual update
        (axhelm_cg_update_box gathers each point's copies; cwt from the
        position) and advance x in the p update — 152 instead of 184 B of HBM
        traffic per point per iteration.  False: the separate-pass kernels."""
        self.op = op
        self.fused = fused
        m = op.mesh
        torch = op.torch
        dev = op.device
        self.torch = torch
        self.lib = _lib.load()
        self.n = m.nel * m.lx ** 3
        f64 = dict(dtype=torch.float64, device=dev)
        # Dirichlet mask on the brick's outer boundary
        gid = m.gid(torch, dev)
        gx = gid % m.NX
        gy = (gid // m.NX) % m.NY
        gz = gid // m.plane
        nz_nodes = m.nz * m.n1 + 1
        on = (gx == 0) | (gx == m.NX - 1) | (gy == 0) | (gy == m.NY - 1) | (gz == 0) | (gz == nz_nodes - 1)
        self.mask = (~on).to(torch.float64)
        del gid, gx, gy, gz, on
        # multiplicity (DSSUM of ones, across ranks) and the Jacobi diagonal
        mult = torch.ones(m.shape, **f64)
        op.dssum(mult)
        self.cwt = (self.mask / mult).contiguous()
        del mult
        diag = torch.empty(m.shape, **f64)
        g = op.geom
        mt = op.mats
        rc = self.lib.axhelm_diag(diag.data_ptr(), *[mt[k].data_ptr() for k in
                                                     ("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd")],
                                  *[g[k].data_ptr() for k in ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")],
                                  m.nel, m.lx, self._s())
        if rc:
            raise DeviceError(_lib.last_error(self.lib))
        op.dssum(diag)
        self.dinv = torch.where(self.mask > 0, 1.0 / diag, torch.zeros_like(diag)).contiguous()
        del diag
        self.x = torch.zeros(m.shape, **f64)
        self.r = torch.empty(m.shape, **f64)
        self.p = torch.empty(m.shape, **f64)
        self.w = torch.empty(m.shape, **f64)
        nb = self.lib.axhelm_reduce_blocks(self.n)
        self.partial = torch.empty(2 * nb, **f64)

    def _s(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.op.device).cuda_stream)

    def _check(self, rc):
        if rc:
            raise DeviceError(_lib.last_error(self.lib))

    def _allreduce(self, t):
        if self.op.comm is not None and self.op.mesh.world > 1:
            if self.op.peer is not None:  # through peer memory, no NCCL
                self.op.peer.allreduce_sum(t)
            else:
                self.op.comm.allreduce_sum(t)

    def solve(self, f, iters: int = 100, graph: bool = False):
        """Run `iters` PCG iterations from x = 0.  Returns (x, rr_history)
        where rr_history[i] = <r_i, r_i> (device tensor, i = 0..iters).

        graph=True: the whole solve — init and `iters` iterations, ~10
        kernels each — is captured once into a CUDA graph (per f and iters)
        and replayed: one launch instead of ~10 iters, for problems small
        enough to be launch-bound.  Same kernels, same results bit for bit.
        Several ranks: only with the peer-memory exchange, whose sequence
        numbers live in device memory so every replay advances them."""
        if graph:
            return self._solve_graph(f, iters)
        return self._solve(f, iters)

    def _solve_graph(self, f, iters):
        torch = self.torch
        if self.op.mesh.world > 1 and self.op.peer is None:
            raise ValueError("graph=True with several ranks needs the peer-memory exchange "
                             "(NCCL / gloo calls are not captured)")
        key = (f.data_ptr(), iters)
        cache = self.__dict__.setdefault("_graphs", {})
        if key not in cache:
            self._solve(f, 1)  # warm-up: one-time library setup (attributes, matrix caches)
            torch.cuda.synchronize(self.op.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                out = self._solve(f, iters)
            cache[key] = (g, out)
        g, out = cache[key]
        g.replay()
        return out

    def _solve(self, f, iters):
        torch = self.torch
        dev = self.op.device
        n = self.n
        # per-iteration scalar slots: sc[i] = (rz_i, rr_i), pw[i]
        sc = torch.zeros(iters + 1, 2, dtype=torch.float64, device=dev)
        s = self._s()
        x, r, p, w = self.x, self.r, self.p, self.w
        P = self.partial.data_ptr()
        self._check(self.lib.axhelm_cg_init(f.data_ptr(), self.mask.data_ptr(), self.dinv.data_ptr(),
                                            self.cwt.data_ptr(), r.data_ptr(), p.data_ptr(),
                                            x.data_ptr(), n, P, sc[0].data_ptr(), s))
        self._allreduce(sc[0])
        # (rz_i, pw_i) side by side for the update kernel
        a = torch.zeros(iters, 2, dtype=torch.float64, device=dev)
        if self.fused:
            m = self.op.mesh
            for it in range(iters):
                a[it, 0:1].copy_(sc[it, 0:1])
                self.op.apply(p, w, dot=a[it, 1:2], local_dssum=False)
                self._allreduce(a[it, 1:2])
                self._check(self.lib.axhelm_cg_update_box(r.data_ptr(), w.data_ptr(), self.dinv.data_ptr(),
                                                          a[it].data_ptr(), m.nx, m.ny, m.nz, m.lx, m.ez0,
                                                          m.ez1, int(m.rank > 0), int(m.rank < m.world - 1),
                                                          int(self.op.xfolded), P, sc[it + 1].data_ptr(), s))
                self._allreduce(sc[it + 1])
                self._check(self.lib.axhelm_cg_xpupdate(x.data_ptr(), p.data_ptr(), r.data_ptr(),
                                                        self.dinv.data_ptr(), a[it].data_ptr(),
                                                        sc[it + 1].data_ptr(), n, s))
            return x, sc[:, 1]
        for it in range(iters):
            a[it, 0:1].copy_(sc[it, 0:1])
            self.op.apply(p, w, dot=a[it, 1:2])
            self._allreduce(a[it, 1:2])
            self._check(self.lib.axhelm_cg_update(x.data_ptr(), r.data_ptr(), p.data_ptr(), w.data_ptr(),
                                                  self.dinv.data_ptr(), self.cwt.data_ptr(),
                                                  a[it].data_ptr(), n, P, sc[it + 1].data_ptr(), s))
            self._allreduce(sc[it + 1])
            self._check(self.lib.axhelm_cg_pupdate(p.data_ptr(), r.data_ptr(), self.dinv.data_ptr(),
                                                   sc[it + 1].data_ptr(), sc[it].data_ptr(), n, s))
        return x, sc[:, 1]
