"""The assembled operator w = QQ^T A u (operator.py) on the GPU: every
schedule of axhelm_ax_gs_box — the concurrent DSSUM follower, layer blocks
with kernel boundaries — against the sequential apply + DSSUM and the oracle
(oracle.ax + oracle.dssum), bit for bit in strict mode; and the multi-rank
overlapped apply with two ranks sharing one GPU over gloo (host-staged
interface planes)."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("CUDA device required")
    return t


def _oracle_assembled(op, u_np, nx, ny, nz, lx):
    arrays = {k: v.cpu().numpy() for k, v in {**op.geom, **op.mats}.items()}
    arrays["ud"] = u_np
    arrays["wd"] = np.zeros_like(u_np)
    return o.dssum(o.ax(arrays), o.box_mesh_gid(nx, ny, nz, lx))


@pytest.mark.parametrize("dims", [(3, 2, 7, 5), (2, 3, 5, 8), (2, 2, 4, 3), (1, 2, 3, 12), (4, 3, 5, 2), (1, 1, 3, 16)])
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_schedules_equal_sequential_and_oracle(torch, dims, mode):
    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    nx, ny, nz, lx = dims
    m = BoxMesh(nx, ny, nz, lx)
    ref = HelmholtzOperator(m, torch, "cuda", mode=mode, schedule="sequential")
    u_np = np.random.default_rng(nz * lx).standard_normal(m.shape)
    u = torch.from_numpy(u_np).cuda()
    w0 = torch.empty_like(u)
    d0 = torch.zeros(1, dtype=torch.float64, device="cuda")
    ref.apply(u, w0, dot=d0)
    want = _oracle_assembled(ref, u_np, nx, ny, nz, lx)
    if mode == "strict":
        assert o.digest(w0.cpu().numpy()) == o.digest(want)
    else:
        assert o.normwise_rel(w0.cpu().numpy(), want) <= 1e-12
    for block in ("follow", 1, 2, 3, nz + 1):
        op = HelmholtzOperator(m, torch, "cuda", mode=mode, schedule=block, geometry=ref.geom)
        w = torch.full_like(u, np.nan)
        d = torch.zeros(1, dtype=torch.float64, device="cuda")
        op.apply(u, w, dot=d)
        torch.cuda.synchronize()
        assert torch.equal(w, w0), (block, mode)
        # the dot is a sum of per-block sums: same value to reassociation
        assert abs(float(d) - float(d0)) <= 1e-12 * max(1.0, abs(float(d0))), block
    # <u, A u> before assembly, against the oracle's element-local apply
    arrays = {k: v.cpu().numpy() for k, v in {**ref.geom, **ref.mats}.items()}
    arrays["ud"] = u_np
    arrays["wd"] = np.zeros_like(u_np)
    dw = float(np.sum(u_np * o.ax(arrays)))
    assert abs(float(d0) - dw) <= 1e-11 * max(1.0, abs(dw))


@pytest.mark.parametrize("dims", [(17, 9, 33), (64, 4, 16), (2, 1, 700), (5, 7, 3), (1, 6, 40)])
@pytest.mark.parametrize("block", ["sequential", 3])
def test_xfold_apply_bit_identical(torch, dims, block, monkeypatch):
    """lx = 8 fast: the x-folding DMMA apply (class-2 DSSUM nodes summed in
    its epilogue, segment seams by xfold_seams) gives w bit-identical to the
    plain apply + full DSSUM pass (AXHELM_XFOLD=0), and matches the oracle.
    Sizes chosen so CTA segments end mid x-run (seams), at run ends, and
    with one element per CTA; nx = 1 has no x faces (xfold off)."""
    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    nx, ny, nz = dims
    lx = 8
    m = BoxMesh(nx, ny, nz, lx)
    op = HelmholtzOperator(m, torch, "cuda", mode="fast", schedule=block)
    u_np = np.random.default_rng(nx * ny + nz).standard_normal(m.shape)
    u = torch.from_numpy(u_np).cuda()
    w = torch.full_like(u, np.nan)
    d = torch.zeros(1, dtype=torch.float64, device="cuda")
    op.apply(u, w, dot=d)
    monkeypatch.setenv("AXHELM_XFOLD", "0")
    w0 = torch.full_like(u, np.nan)
    d0 = torch.zeros(1, dtype=torch.float64, device="cuda")
    op.apply(u, w0, dot=d0)
    torch.cuda.synchronize()
    assert torch.equal(w, w0)
    assert abs(float(d) - float(d0)) <= 1e-12 * max(1.0, abs(float(d0)))
    if m.nel <= 6000:
        want = _oracle_assembled(op, u_np, nx, ny, nz, lx)
        assert o.normwise_rel(w.cpu().numpy(), want) <= 1e-12


def test_ax_gs_box_rejects_bad_ranges(torch):
    import ctypes

    from paper_2506_20994_b200 import _lib

    lib = _lib.load()
    z = [None] * 15
    # planes outside the slab
    assert lib.axhelm_ax_gs_box(*z, 2, 2, 4, 0, 3, 0, 3, 0, 99, 0, 1, None, None, None, ctypes.c_void_p(0)) != 0
    assert "outside" in _lib.last_error(lib)
    # layer range beyond the slab
    assert lib.axhelm_ax_gs_box(*z, 2, 2, 4, 0, 3, 0, 4, 0, 9, 0, 1, None, None, None, ctypes.c_void_p(0)) != 0
    # dot without scratch
    assert lib.axhelm_ax_gs_box(*z, 2, 2, 4, 0, 3, 0, 3, 0, 9, 0, 1, None, None, ctypes.c_void_p(8),
                                ctypes.c_void_p(0)) != 0
    # follow schedule without progress scratch
    assert lib.axhelm_ax_gs_box(*z, 2, 2, 4, 0, 3, 0, 3, 0, 9, 0, -1, None, None, None,
                                ctypes.c_void_p(0)) != 0
    assert "progress" in _lib.last_error(lib)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, dims, mode, block, q, exchange="nccl", applies=1):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_20994_b200.dist import TorchComm
        from paper_2506_20994_b200.mesh import BoxMesh
        from paper_2506_20994_b200.operator import HelmholtzOperator

        nx, ny, nz, lx = dims
        m = BoxMesh(nx, ny, nz, lx, rank, world)
        op = HelmholtzOperator(m, torch, "cuda", comm=TorchComm(dist), mode=mode, schedule=block,
                               exchange=exchange)
        ug = np.random.default_rng(5).standard_normal((nx * ny * nz, lx, lx, lx))
        u = torch.from_numpy(ug[m.ez0 * nx * ny: m.ez1 * nx * ny].copy()).cuda()
        w = torch.empty_like(u)
        d = torch.zeros(1, dtype=torch.float64, device="cuda")
        for _ in range(applies):  # repeated applies: the peer flags' sequence numbers advance
            w.fill_(np.nan)
            op.apply(u, w, dot=d)
        torch.cuda.synchronize()
        q.put((rank, w.cpu().numpy(), float(d), op.overlap))
        if op.peer is not None:
            dist.barrier()  # nobody frees its region while a neighbour may still write it
            op.peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,dims,block,exchange,world", [("strict", (3, 2, 8, 5), "sequential", "nccl", 2),
                                                            ("strict", (3, 2, 8, 5), "follow", "nccl", 2),
                                                            ("strict", (3, 2, 8, 5), 2, "nccl", 2),
                                                            ("fast", (2, 3, 8, 8), "follow", "nccl", 2),
                                                            ("strict", (3, 2, 8, 5), "sequential", "peer", 2),
                                                            ("fast", (2, 3, 8, 8), "sequential", "peer", 2),
                                                            ("fast", (5, 3, 12, 8), "sequential", "nccl", 2),
                                                            ("fast", (4, 2, 12, 8), 2, "peer", 3),
                                                            ("strict", (2, 2, 9, 4), "sequential", "peer", 3)])
def test_ranks_on_one_gpu_bit_exact(torch, mode, dims, block, exchange, world):
    """z-slab ranks with the overlapped boundary/interior apply and the
    interface exchange — host-staged over gloo ("nccl" transport path) or
    through peer memory (CUDA IPC between the two processes, the kernels
    writing each other's buffers and flags) — the gathered result equals the
    single-domain sequential apply bit for bit (and, in strict mode, the
    oracle) for every schedule, over three consecutive applies."""
    import torch.multiprocessing as mp

    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    nx, ny, nz, lx = dims
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, dims, mode, block, q, exchange, 3))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, w, d, ov = q.get(timeout=300)
        res[r] = (w, d, ov)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res[r][2] for r in res), "expected the overlapped path (slabs of > 2 layers)"
    got = np.concatenate([res[r][0] for r in range(world)])
    ref = HelmholtzOperator(BoxMesh(nx, ny, nz, lx), torch, "cuda", mode=mode, schedule="sequential")
    ug = np.random.default_rng(5).standard_normal((nx * ny * nz, lx, lx, lx))
    u = torch.from_numpy(ug).cuda()
    w = torch.empty_like(u)
    ref.apply(u, w)
    assert o.digest(got) == o.digest(w.cpu().numpy())
    if mode == "strict":
        assert o.digest(got) == o.digest(_oracle_assembled(ref, ug, nx, ny, nz, lx))


GEOM = ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")


def assembled_cases(golden_dir):
    with np.load(golden_dir / "assembled_cases.npz") as z:
        tags = sorted({k.split("/")[0] for k in z.files})
        for tag in tags:
            dims, lx = tag.split("_lx")
            nx, ny, nz = (int(v) for v in dims.split("x"))
            yield (nx, ny, nz, int(lx)), {k.split("/")[1]: z[k] for k in z.files if k.startswith(tag + "/")}


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_assembled_operator_matches_reference_assembly(torch, golden_dir, mode):
    """f1 pinned to reference arithmetic: HelmholtzOperator.apply (ax_helm +
    DSSUM) on continuous fields equals K u with K assembled from the
    reference's own element matrices (mdg.sem.dense_assemble, sem.py:340-364;
    tests/golden/make_assembled_golden.py), <= 1e-12 normwise."""
    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    for (nx, ny, nz, lx), c in assembled_cases(golden_dir):
        m = BoxMesh(nx, ny, nz, lx)
        geom = {k: torch.from_numpy(c[k]).cuda() for k in GEOM}
        op = HelmholtzOperator(m, torch, "cuda", mode=mode, geometry=geom)
        u = torch.from_numpy(c["u"]).cuda()
        w = torch.full_like(u, float("nan"))
        op.apply(u, w)
        torch.cuda.synchronize()
        err = o.normwise_rel(w.cpu().numpy(), c["w"])
        assert err <= 1e-12, ((nx, ny, nz, lx), mode, err)
