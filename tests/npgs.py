"""TEST HELPER: a NumPy implementation of the gather-scatter ops interface
(sum_local / plane / new_plane_buffer) used to drive the product's
multi-rank DSSUM protocol (paper_2506_20994_b200/dist.py) on CPUs with the
gloo backend.  Checker-side code: the product's ops are the CUDA kernels."""

import numpy as np
import torch

PARTIAL, FINISH, WRITE = 0, 1, 2


class NumpyGSOps:
    def __init__(self, gid_local, plane, n1, ez0, ez1, rank, world):
        flat = gid_local.reshape(-1)
        order = np.argsort(flat, kind="stable")
        sg = flat[order]
        uniq, starts, counts = np.unique(sg, return_index=True, return_counts=True)
        gz = uniq // plane
        top = (gz == ez1 * n1) & (rank < world - 1)
        bot = (gz == ez0 * n1) & (rank > 0)
        local = (counts > 1) & ~top & ~bot
        self.plane_n = plane

        def csr(sel):
            return [(int(uniq[q] % plane), order[starts[q]:starts[q] + counts[q]]) for q in np.flatnonzero(sel)]

        self.local = csr(local)
        self.top = csr(top)
        self.bot = csr(bot)

    def new_plane_buffer(self):
        return torch.zeros(self.plane_n, dtype=torch.float64)

    def sum_local(self, w):
        a = w.numpy().reshape(-1)
        for _, copies in self.local:
            s = 0.0
            for c in copies:
                s = s + a[c]
            a[copies] = s

    def plane(self, op, which, w, buf):
        a = w.numpy().reshape(-1)
        b = buf.numpy()
        for slot, copies in (self.top if which == "top" else self.bot):
            if op == PARTIAL:
                s = 0.0
                for c in copies:
                    s = s + a[c]
                b[slot] = s
            elif op == FINISH:
                s = b[slot]
                for c in copies:
                    s = s + a[c]
                a[copies] = s
                b[slot] = s
            else:
                a[copies] = b[slot]
