"""Golden vectors for the ASSEMBLED operator and the PCG, derived from the
reference's own arithmetic.  Run in the build container:

    python tests/golden/make_assembled_golden.py

The reference has no gather-scatter or solver, but it does
have the element operator as a dense matrix: mdg.sem.dense_assemble
(/root/reference/pkg/src/mdg/sem.py:340-364) applies ax_reference to every
unit vector of one element.  For small bricks (element order
e = (ez ny + ey) nx + ex, global node id (gz NY + gy) NX + gx with
NX = nx (lx-1) + 1 — the numbering contract of include/axhelm.h) this
script assembles the global stiffness K = sum_e Q_e^T K_e Q_e from those
element matrices, with per-element geometry from
mdg.sem.random_spd_geometry, and stores per case:

  h1d, g11d .. g23d   [nel, lx, lx, lx]  the geometry fed to the GPU
  u                   [nel, lx, lx, lx]  a continuous field: u_g[gid]
  w                   [nel, lx, lx, lx]  (K u_g)[gid]   = QQ^T A u
  f                   [nel, lx, lx, lx]  a continuous right-hand side
  x                   [nel, lx, lx, lx]  the dense solve of the Dirichlet
                                         problem: x_I = K_II^-1 f_I, x_B = 0

into assembled_cases.npz.  Tests: tests/test_operator_gpu.py
(HelmholtzOperator.apply vs w, <= 1e-12 normwise) and tests/test_cg_gpu.py
(JacobiPCG's converged x vs x, <= 1e-9).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
CASES = ((3, 2, 2, 4, 11), (2, 3, 2, 5, 12), (2, 2, 3, 6, 13), (2, 2, 2, 8, 14), (4, 1, 1, 3, 15))
FIELDS = ("h1", "g11", "g22", "g33", "g12", "g13", "g23")


def box_gid(nx, ny, nz, lx):
    n1 = lx - 1
    NX, NY = nx * n1 + 1, ny * n1 + 1
    e = np.arange(nx * ny * nz)
    ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
    k, j, i = np.meshgrid(np.arange(lx), np.arange(lx), np.arange(lx), indexing="ij")
    gx = ex[:, None, None, None] * n1 + i[None]
    gy = ey[:, None, None, None] * n1 + j[None]
    gz = ez[:, None, None, None] * n1 + k[None]
    return (gz * NY + gy) * NX + gx, (NX, NY, nz * n1 + 1)


def main() -> None:
    sys.path.insert(0, str(REF))
    from mdg import sem

    out = {}
    for nx, ny, nz, lx, seed in CASES:
        nel = nx * ny * nz
        basis = sem.gll_basis(lx)
        geom = sem.random_spd_geometry(nel, lx, seed)
        gid, (NX, NY, NZ) = box_gid(nx, ny, nz, lx)
        ng = NX * NY * NZ
        K = np.zeros((ng, ng))
        for e in range(nel):
            ge = sem.GeomFactors(**{f: getattr(geom, f)[e:e + 1] for f in FIELDS})
            Ke = sem.dense_assemble(basis, ge)
            idx = gid[e].ravel()
            K[np.ix_(idx, idx)] += Ke
        rng = np.random.default_rng(seed)
        u_g = rng.standard_normal(ng)
        f_g = rng.standard_normal(ng)
        gx, gy, gz = np.arange(ng) % NX, (np.arange(ng) // NX) % NY, np.arange(ng) // (NX * NY)
        inner = ~((gx == 0) | (gx == NX - 1) | (gy == 0) | (gy == NY - 1) | (gz == 0) | (gz == NZ - 1))
        x_g = np.zeros(ng)
        if inner.any():
            x_g[inner] = np.linalg.solve(K[np.ix_(inner, inner)], f_g[inner])
        tag = f"{nx}x{ny}x{nz}_lx{lx}"
        for f in FIELDS:
            out[f"{tag}/{f}d"] = np.ascontiguousarray(getattr(geom, f))
        out[f"{tag}/u"] = u_g[gid]
        out[f"{tag}/w"] = (K @ u_g)[gid]
        out[f"{tag}/f"] = f_g[gid]
        out[f"{tag}/x"] = x_g[gid]
        print(tag, "nodes", ng, "interior", int(inner.sum()))
    np.savez_compressed(OUT / "assembled_cases.npz", **out)


if __name__ == "__main__":
    main()
