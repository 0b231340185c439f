"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the checker for the B200 ax_helm path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2506_20994_b200``) never imports, links or executes anything under
``oracle/``; a product path that fell back to this file would void every
parity claim.

It restates, in NumPy, the reference's algorithm for the path (reference =
``/root/reference/pkg/src/mdg``, "mdg").  Each function cites the reference
``file:line`` it follows.  Parity is PINNED: ``tests/test_oracle_pins.py``
checks every function here against golden vectors produced by importing the
reference itself (``tests/golden/make_golden.py``; committed fixtures under
``tests/golden/``).

Scalar arithmetic contract (the reason this oracle can be bit-exact): the
reference apply uses separate NumPy ufunc multiplies and adds in a fixed
association, with no fused multiply-add (sem.py:319-335).  Every restated
expression below performs the same IEEE-754 binary64 operations on the same
operands in the same order, so results are bit-identical, not just close.

The gather-scatter (DSSUM), box-mesh numbering and Jacobi-PCG restatements
at the end have no reference implementation (SPEC.md:14 puts them out of the
reference's scope); they are marked "parity unpinned" and are validated by
exact integer-valued sums and algebraic identities instead (tests/).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
from pathlib import Path

import numpy as np

LX_MIN, LX_MAX = 2, 16  # sem.py:36-37

# mdg/axprogram.py:32-48 — the 15-pointer ABI parameter order.
ABI_ORDER = (
    "wd", "ud", "dxd", "dyd", "dzd", "dxtd", "dytd", "dztd",
    "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d",
)
FIELDS = ("ud", "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")
MATRICES = ("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd")


# --------------------------------------------------------------- GLL basis


def legendre(n: int, x):
    """L_n(x) and L_n'(x) by the three-term recurrence (sem.py:143-173)."""
    x = np.asarray(x, dtype=np.float64)
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1, d1 = x.copy(), np.ones_like(x)
    for k in range(2, n + 1):
        p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        d1 = x * d1 + k * p1
        p0, p1 = p1, p2
    return p1, d1


def gll(lx: int):
    """GLL points, weights and D[i][j] = l_j'(x_i) (sem.py:182-236).

    Same construction as the reference: damped Newton from Chebyshev-Lobatto
    guesses on the left half, mirrored; weights 2/(N(N+1)L_N^2); closed-form
    D with corners -+N(N+1)/4.  Returns (points, weights, deriv).
    """
    if not (LX_MIN <= lx <= LX_MAX):
        raise ValueError(f"lx must be in [{LX_MIN}, {LX_MAX}]")
    n = lx - 1
    x = np.empty(lx)
    x[0], x[-1] = -1.0, 1.0
    if lx % 2 == 1:
        x[lx // 2] = 0.0
    h = np.pi / n
    for idx in range(1, (lx - 2) // 2 + 1):
        t = -np.cos(np.pi * idx / n)
        for _ in range(100):
            p, d = legendre(n, t)
            d2 = (2.0 * t * d - n * (n + 1) * p) / (1.0 - t * t)
            step = float(np.clip(d / d2, -0.5 * h, 0.5 * h))
            t -= step
            if abs(step) < 1e-16:
                break
        x[idx], x[lx - 1 - idx] = t, -t
    ln, _ = legendre(n, x)
    w = 2.0 / (n * (n + 1) * ln * ln)
    dm = np.zeros((lx, lx))
    for i in range(lx):
        for j in range(lx):
            if i != j:
                dm[i, j] = (ln[i] / ln[j]) / (x[i] - x[j])
    dm[0, 0] = -n * (n + 1) / 4.0
    dm[-1, -1] = n * (n + 1) / 4.0
    return x, w, dm


def operator_matrices(deriv: np.ndarray):
    """(stage-1 matrix, stage-2 matrix) = (D^T, D) (sem.py:288-297)."""
    return np.ascontiguousarray(deriv.T), np.ascontiguousarray(deriv)


# ------------------------------------------------------------- geometry


def random_spd_geometry(nel: int, lx: int, seed: int) -> dict[str, np.ndarray]:
    """Seeded SPD metric blocks M M^T + 0.1 I and h1 ~ U(0.5,1.5) (sem.py:265-285).

    Same generator stream as the reference: one uniform draw of the
    (nel,lx,lx,lx,3,3) M tensor, then the h1 draw.
    """
    rng = np.random.default_rng(seed)
    m = rng.uniform(-1.0, 1.0, size=(nel, lx, lx, lx, 3, 3))
    g = np.einsum("...ab,...cb->...ac", m, m) + 0.1 * np.eye(3)
    h1 = rng.uniform(0.5, 1.5, size=(nel, lx, lx, lx))
    c = np.ascontiguousarray
    return {
        "g11d": c(g[..., 0, 0]), "g22d": c(g[..., 1, 1]), "g33d": c(g[..., 2, 2]),
        "g12d": c(g[..., 0, 1]), "g13d": c(g[..., 0, 2]), "g23d": c(g[..., 1, 2]),
        "h1d": c(h1),
    }


def box_geometry(nel: int, lx: int, h: float) -> dict[str, np.ndarray]:
    """Axis-aligned cubes: g11=g22=g33=w_i w_j w_k h/2, rest 0, h1=1 (sem.py:239-262)."""
    _, w, _ = gll(lx)
    diag = (h / 2.0) * (w[:, None, None] * w[None, :, None] * w[None, None, :])
    diag = np.ascontiguousarray(np.broadcast_to(diag, (nel, lx, lx, lx)))
    z = np.zeros((nel, lx, lx, lx))
    return {
        "g11d": diag.copy(), "g22d": diag.copy(), "g33d": diag.copy(),
        "g12d": z.copy(), "g13d": z.copy(), "g23d": z.copy(),
        "h1d": np.ones((nel, lx, lx, lx)),
    }


def problem(lx: int, nel: int, seed: int | None = None) -> dict[str, np.ndarray]:
    """The benchmark problem bench._problem builds (bench.py:41-47) as the
    15-array ABI dict ax_arrays returns (axprogram.py:74-101).

    seed defaults to the bench seed 7919*lx + nel (bench.py:42).
    """
    if seed is None:
        seed = 7919 * lx + nel
    _, _, deriv = gll(lx)
    geom = random_spd_geometry(nel, lx, seed)
    u = np.random.default_rng(seed).standard_normal((nel, lx, lx, lx))
    a, b = operator_matrices(deriv)
    arrays = {"wd": np.zeros_like(u), "ud": u}
    for name in ("dxd", "dyd", "dzd"):
        arrays[name] = a.copy()
    for name in ("dxtd", "dytd", "dztd"):
        arrays[name] = b.copy()
    arrays.update(geom)
    return {k: arrays[k] for k in ABI_ORDER}


# ---------------------------------------------------------------- the apply


def ax(arrays: dict[str, np.ndarray]) -> np.ndarray:
    """w = A u with the reference's exact per-point operation order.

    Restates sem.ax_reference (sem.py:300-337) and the IR tasklets
    (axprogram.py:159-163 stage 1, :188-192 combine, :229 stage 2), honouring
    all six matrix slots separately (dxd/dyd/dzd stage 1, dxtd/dytd/dztd
    stage 2) like the compiled ABI does:

      r[e,k,j,i] = (((0 + dx[0,i] u[e,k,j,0]) + dx[1,i] u[e,k,j,1]) + ...)
      s[e,k,j,i] = same over dy[l,j] u[e,k,l,i];  t: dz[l,k] u[e,l,j,i]
      ur = h1 ((g11 r + g12 s) + g13 t); us, ut likewise
      w = (((w + dxt[l,i] ur[e,k,j,l]) + dyt[l,j] us[e,k,l,i]) + dzt[l,k] ut[e,l,j,i]) for l = 0..lx-1
    """
    u = arrays["ud"]
    dx, dy, dz = arrays["dxd"], arrays["dyd"], arrays["dzd"]
    dxt, dyt, dzt = arrays["dxtd"], arrays["dytd"], arrays["dztd"]
    lx = u.shape[1]
    r = np.zeros_like(u)
    s = np.zeros_like(u)
    t = np.zeros_like(u)
    for l in range(lx):
        r = r + u[:, :, :, l, None] * dx[l][None, None, None, :]
        s = s + u[:, :, l, None, :] * dy[l][None, None, :, None]
        t = t + u[:, l, None, :, :] * dz[l][None, :, None, None]
    h1 = arrays["h1d"]
    g11, g22, g33 = arrays["g11d"], arrays["g22d"], arrays["g33d"]
    g12, g13, g23 = arrays["g12d"], arrays["g13d"], arrays["g23d"]
    ur = h1 * ((g11 * r + g12 * s) + g13 * t)
    us = h1 * ((g12 * r + g22 * s) + g23 * t)
    ut = h1 * ((g13 * r + g23 * s) + g33 * t)
    w = np.zeros_like(u)
    for l in range(lx):
        w = w + ur[:, :, :, l, None] * dxt[l][None, None, None, :]
        w = w + us[:, :, l, None, :] * dyt[l][None, None, :, None]
        w = w + ut[:, l, None, :, :] * dzt[l][None, :, None, None]
    return w


def flops_model(lx: int, nel: int) -> int:
    """nel * lx^3 * (12 lx + 18) (sem.py:367-375)."""
    return int(nel) * int(lx) ** 3 * (12 * int(lx) + 18)


def normwise_rel(got: np.ndarray, want: np.ndarray) -> float:
    """max|got - want| / max|want| (cabi-harness compare.ts:10-27)."""
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    diff = float(np.max(np.abs(got - want))) if want.size else 0.0
    return diff / scale if scale > 0 else diff


def digest(a: np.ndarray) -> str:
    """sha256 of the little-endian float64 bytes (bit-exact fingerprint)."""
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


# --------------------------------------------------- MDGT tensor interchange


def mdgt_encode(a: np.ndarray) -> bytes:
    """MDGT v1: magic, version, rank, u32 dims, LE doubles (tensorfile.py:24-32)."""
    import struct

    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return (b"MDGT" + struct.pack("<BB", 1, a.ndim)
            + struct.pack(f"<{a.ndim}I", *a.shape) + a.astype("<f8").tobytes())


# -------------------------------------------------------- C restatement


_HERE = Path(__file__).resolve().parent
_LIB = None


def c_oracle():
    """ctypes handle of oracle/liboracle_ax.so (ax_oracle.c), built by
    ``make -C oracle`` / __graft_entry__.build().  None if not built."""
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle_ax.so"
        if not path.exists():
            return None
        lib = ctypes.CDLL(str(path))
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_ax_helm.argtypes = [dp] * 15 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        lib.oracle_ax_helm.restype = ctypes.c_int
        lib.oracle_dssum.argtypes = [dp, ctypes.POINTER(ctypes.c_int64), dp, ctypes.c_int64]
        lib.oracle_dssum.restype = None
        _LIB = lib
    return _LIB


def ax_c(arrays: dict[str, np.ndarray], nthreads: int = 0) -> np.ndarray:
    """Same arithmetic as ax(), in C (oracle/ax_oracle.c), OpenMP over elements."""
    lib = c_oracle()
    if lib is None:
        raise RuntimeError("oracle/liboracle_ax.so not built (run make -C oracle)")
    u = arrays["ud"]
    nel, lx = u.shape[0], u.shape[1]
    out = np.zeros_like(u)
    dp = ctypes.POINTER(ctypes.c_double)
    ptrs = []
    for name in ABI_ORDER:
        a = out if name == "wd" else np.ascontiguousarray(arrays[name], dtype=np.float64)
        if name != "wd":
            arrays = dict(arrays)
            arrays[name] = a
        ptrs.append(a.ctypes.data_as(dp))
    rc = lib.oracle_ax_helm(*ptrs, nel, lx, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_ax_helm rejected lx={lx}")
    return out


# ===================================================================
# Gather-scatter / box mesh / PCG — parity unpinned (no reference: SPEC.md:14)
# ===================================================================


def box_mesh_gid(nx: int, ny: int, nz: int, lx: int) -> np.ndarray:
    """Global node id of every local GLL point of an nx*ny*nz brick of hexes.

    Element order e = (ez*ny + ey)*nx + ex; local point order
    [e][k][j][i] (sem.py:68-100).  Global node (gx, gy, gz) with
    gx = ex*(lx-1) + i etc., numbered gz-major: ((gz*NY)+gy)*NX+gx with
    NX = nx*(lx-1)+1.  Returns int64 [nel, lx, lx, lx].
    """
    n1 = lx - 1
    NX, NY = nx * n1 + 1, ny * n1 + 1
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    k, j, i = np.meshgrid(np.arange(lx), np.arange(lx), np.arange(lx), indexing="ij")
    gx = ex.reshape(-1, 1, 1, 1) * n1 + i[None]
    gy = ey.reshape(-1, 1, 1, 1) * n1 + j[None]
    gz = ez.reshape(-1, 1, 1, 1) * n1 + k[None]
    return ((gz.astype(np.int64) * NY + gy) * NX + gx).astype(np.int64)


def dssum(w: np.ndarray, gid: np.ndarray) -> np.ndarray:
    """Direct stiffness summation: every local copy of a SHARED global node
    (multiplicity > 1) gets the sum of all copies, accumulated from 0.0 in
    ascending flat local index; unshared points are left untouched.

    The deterministic order is the contract the CUDA gather kernel follows,
    which is what makes the result bit-exact.  (np.add.at applies updates in
    index-array order, i.e. ascending local index here.)
    """
    flat = w.reshape(-1)
    g = gid.reshape(-1)
    nglob = int(g.max()) + 1 if g.size else 0
    acc = np.zeros(nglob)
    np.add.at(acc, g, flat)
    cnt = np.bincount(g, minlength=nglob)
    out = flat.copy()
    shared = cnt[g] > 1
    out[shared] = acc[g[shared]]
    return out.reshape(w.shape)


def multiplicity(gid: np.ndarray) -> np.ndarray:
    """Number of local copies of each point's global node (float64)."""
    g = gid.reshape(-1)
    return np.bincount(g)[g].astype(np.float64).reshape(gid.shape)


def gs_boundary_mask(nx: int, ny: int, nz: int, lx: int) -> np.ndarray:
    """1.0 on interior global nodes, 0.0 on the brick's outer boundary
    (homogeneous Dirichlet), as a local field [nel,lx,lx,lx]."""
    n1 = lx - 1
    NX, NY, NZ = nx * n1 + 1, ny * n1 + 1, nz * n1 + 1
    gid = box_mesh_gid(nx, ny, nz, lx)
    gx = gid % NX
    gy = (gid // NX) % NY
    gz = gid // (NX * NY)
    on = (gx == 0) | (gx == NX - 1) | (gy == 0) | (gy == NY - 1) | (gz == 0) | (gz == NZ - 1)
    return np.where(on, 0.0, 1.0)


def box_mesh_gid_slab(nx: int, ny: int, nz: int, lx: int, ez0: int, ez1: int) -> np.ndarray:
    """box_mesh_gid restricted to the element layers [ez0, ez1)."""
    g = box_mesh_gid(nx, ny, nz, lx)
    return g[ez0 * nx * ny: ez1 * nx * ny]


def box_deformed_geometry(nx: int, ny: int, nz: int, lx: int, amp: float,
                          ez0: int = 0, ez1: int | None = None) -> dict[str, np.ndarray]:
    """Geometric factors of the deformed brick (restates the device
    generator's formulas, csrc/mesh_gs.cu box_geom_kernel; parity unpinned:
    there is no reference mesh).  X = X0 + d (1,1,1), d = amp/c_min sin sin sin;
    G = w_i w_j w_k det J J^-1 J^-T, h1 = 1."""
    ez1 = nz if ez1 is None else ez1
    x, w, _ = gll(lx)
    ez, ey, ex = np.meshgrid(np.arange(ez0, ez1), np.arange(ny), np.arange(nx), indexing="ij")
    ex, ey, ez = (a.reshape(-1, 1, 1, 1).astype(np.float64) for a in (ex, ey, ez))
    X0 = ex + 0.5 * (x[None, None, None, :] + 1.0)
    Y0 = ey + 0.5 * (x[None, None, :, None] + 1.0)
    Z0 = ez + 0.5 * (x[None, :, None, None] + 1.0)
    cx, cy, cz = 2 * np.pi / nx, 2 * np.pi / ny, 2 * np.pi / nz
    cmin = min(cx, cy, cz)
    sx, csx = np.sin(cx * X0), np.cos(cx * X0)
    sy, csy = np.sin(cy * Y0), np.cos(cy * Y0)
    sz, csz = np.sin(cz * Z0), np.cos(cz * Z0)
    grad = [amp * (cx / cmin) * csx * sy * sz, amp * (cy / cmin) * sx * csy * sz,
            amp * (cz / cmin) * sx * sy * csz]
    shape = np.broadcast(X0, Y0, Z0).shape
    J = np.empty(shape + (3, 3))
    for a in range(3):
        for b in range(3):
            J[..., a, b] = 0.5 * ((1.0 if a == b else 0.0) + grad[b])
    Jinv = np.linalg.inv(J)
    det = np.linalg.det(J)
    W = w[None, :, None, None] * w[None, None, :, None] * w[None, None, None, :]
    G = np.einsum("...ba,...ca->...bc", Jinv, Jinv) * (W * det)[..., None, None]
    c = np.ascontiguousarray
    return {"h1d": np.ones(shape), "g11d": c(G[..., 0, 0]), "g22d": c(G[..., 1, 1]),
            "g33d": c(G[..., 2, 2]), "g12d": c(G[..., 0, 1]), "g13d": c(G[..., 0, 2]),
            "g23d": c(G[..., 1, 2])}


def local_diag(arrays: dict[str, np.ndarray]) -> np.ndarray:
    """Diagonal of each element's A_e by applying ax() to unit vectors
    (parity unpinned; restates sem.dense_assemble's column-by-column idea,
    sem.py:340-364, per element)."""
    u = arrays["ud"]
    nel, lx = u.shape[0], u.shape[1]
    n = lx ** 3
    out = np.empty_like(u)
    for e in range(nel):
        sub = {k: (np.broadcast_to(v[e:e + 1], (n, lx, lx, lx)).copy() if v.ndim == 4 else v)
               for k, v in arrays.items()}
        sub["ud"] = np.eye(n).reshape(n, lx, lx, lx)
        w = ax(sub).reshape(n, n)
        out[e] = np.diag(w).reshape(lx, lx, lx)
    return out


def pcg(arrays: dict[str, np.ndarray], gid: np.ndarray, mask: np.ndarray, f: np.ndarray,
        iters: int):
    """Jacobi-PCG for mask.Q Q^T A x = mask.f from x = 0, the algorithm of
    paper_2506_20994_b200/cg.py restated in NumPy (parity unpinned: the
    reference has no solver).  Returns (x, rr_history)."""
    mult = multiplicity(gid)
    minv = 1.0 / mult
    diag = dssum(local_diag(arrays), gid)
    dinv = np.where(mask > 0, 1.0 / diag, 0.0)

    def A(p):
        a = dict(arrays)
        a["ud"] = p
        return dssum(ax(a), gid)

    x = np.zeros_like(f)
    r = mask * f
    p = dinv * r
    rz = float(np.sum(minv * r * dinv * r))
    hist = [float(np.sum(minv * r * r))]
    for _ in range(iters):
        w = A(p)
        pw = float(np.sum(minv * p * w))
        alpha = rz / pw if pw != 0.0 else 0.0  # exact convergence: step 0 (cg.cu cg_ratio)
        x = x + alpha * p
        r = r - alpha * mask * w
        rz_new = float(np.sum(minv * r * dinv * r))
        hist.append(float(np.sum(minv * r * r)))
        p = dinv * r + (rz_new / rz if rz != 0.0 else 0.0) * p
        rz = rz_new
    return x, np.array(hist)
