"""GPU Jacobi-PCG (cg.py) against the NumPy restatement (oracle.pcg) and a
manufactured solution.  Parity unpinned (the reference has no solver,
SPEC.md:14): iterates agree to FP64 reassociation; the solve converges."""

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


def _setup(torch, nx, ny, nz, lx, mode="strict"):
    from paper_2506_20994_b200.cg import JacobiPCG
    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    m = BoxMesh(nx, ny, nz, lx)
    op = HelmholtzOperator(m, torch, "cuda", mode=mode, amp=0.1)
    return m, op, JacobiPCG(op)


def test_diagonal_matches_unit_vector_applies(torch):
    m, op, pcg = _setup(torch, 2, 2, 2, 4)
    arrays = {k: v.cpu().numpy() for k, v in {**op.geom, **op.mats}.items()}
    arrays["ud"] = np.zeros(m.shape)
    want = o.dssum(o.local_diag(arrays), o.box_mesh_gid(2, 2, 2, 4))
    mask = pcg.mask.cpu().numpy()
    dinv = pcg.dinv.cpu().numpy()
    got = np.divide(1.0, dinv, out=np.zeros_like(dinv), where=mask > 0)
    assert o.normwise_rel(got, np.where(mask > 0, want, 0.0)) <= 1e-13


@pytest.mark.parametrize("dims,mode", [((3, 2, 2, 4), "strict"), ((2, 2, 3, 5), "fast"), ((2, 2, 2, 8), "fast"),
                                       ((3, 3, 3, 2), "strict"), ((1, 2, 2, 16), "fast"), ((2, 1, 3, 11), "strict")])
def test_pcg_iterates_match_oracle(torch, dims, mode):
    nx, ny, nz, lx = dims
    m, op, pcg = _setup(torch, nx, ny, nz, lx, mode)
    gid = o.box_mesh_gid(nx, ny, nz, lx)
    rng = np.random.default_rng(1)
    # a continuous right-hand side: random per global node
    fg = rng.standard_normal(int(gid.max()) + 1)
    f = fg[gid]
    x, hist = pcg.solve(torch.from_numpy(f).cuda(), iters=25)
    arrays = {k: v.cpu().numpy() for k, v in {**op.geom, **op.mats}.items()}
    arrays["ud"] = np.zeros(m.shape)
    xw, hw = o.pcg(arrays, gid, pcg.mask.cpu().numpy(), f, 25)
    h = hist.cpu().numpy()
    live = hw > 1e-24 * hw[0]  # before the residual reaches rounding level (tiny meshes converge early)
    assert np.max(np.abs(h - hw)[live] / hw[live]) <= 1e-8
    assert o.normwise_rel(x.cpu().numpy(), xw) <= 1e-9


def test_pcg_converges_to_manufactured_solution(torch):
    nx, ny, nz, lx = 3, 3, 3, 6
    m, op, pcg = _setup(torch, nx, ny, nz, lx, "fast")
    gid = m.gid(torch, "cuda")
    xs = torch.randn(int(gid.max()) + 1, dtype=torch.float64, device="cuda")[gid] * pcg.mask
    f = torch.empty_like(xs)
    op.apply(xs, f)
    x, hist = pcg.solve(f, iters=300)
    h = hist.cpu().numpy()
    assert h[-1] <= 1e-20 * h[0]
    assert float((x - xs).abs().max() / xs.abs().max()) <= 1e-8


@pytest.mark.parametrize("dims,mode", [((3, 2, 4, 5), "strict"), ((2, 3, 3, 8), "fast"), ((2, 2, 2, 3), "strict")])
def test_fused_update_matches_separate_passes(torch, dims, mode):
    """axhelm_cg_update_box (local DSSUM gathered inside the residual update,
    cwt from the position) + axhelm_cg_xpupdate against the separate DSSUM
    pass + cg_update + cg_pupdate: the per-point arithmetic is identical
    (the gathered sum is the DSSUM's, bit for bit); only the fixed order of
    the block reductions differs (element-major vs point-major), so the
    iterates agree to reassociation."""
    from paper_2506_20994_b200.cg import JacobiPCG

    nx, ny, nz, lx = dims
    m, op, pcg = _setup(torch, nx, ny, nz, lx, mode)
    gid = m.gid(torch, "cuda")
    f = torch.randn(int(gid.max()) + 1, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(3))[gid]
    x1, h1 = pcg.solve(f, iters=12)
    x1, h1 = x1.clone(), h1.clone()
    x2, h2 = JacobiPCG(op, fused=False).solve(f, iters=12)
    torch.cuda.synchronize()
    assert float(((h1 - h2).abs() / h2).max()) <= 1e-10
    assert float((x1 - x2).abs().max() / x2.abs().max()) <= 1e-10


@pytest.mark.parametrize("dims", [(17, 5, 9), (3, 2, 4), (1, 3, 5)])
def test_xfold_update_bit_identical(torch, dims, monkeypatch):
    """lx = 8 fast: apply(local_dssum=False) with the x-folding kernel (class-2
    nodes summed by the apply, read once by the update) + axhelm_cg_update_box
    gives r and the two update sums bit-identical to the plain apply whose
    x copies the update gathers (AXHELM_XFOLD=0); nx = 1 never folds."""
    import ctypes

    nx, ny, nz = dims
    m, op, pcg = _setup(torch, nx, ny, nz, 8, "fast")
    op.fold_unassembled = True
    g = torch.Generator(device="cuda").manual_seed(11)
    p = torch.randn(m.shape, dtype=torch.float64, device="cuda", generator=g)
    r0 = torch.randn(m.shape, dtype=torch.float64, device="cuda", generator=g)
    a = torch.tensor([0.7, 1.3], dtype=torch.float64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = []
    for env in (None, "0"):
        if env is not None:
            monkeypatch.setenv("AXHELM_XFOLD", env)
        w = torch.full_like(p, np.nan)
        dot = torch.zeros(1, dtype=torch.float64, device="cuda")
        op.apply(p, w, dot=dot, local_dssum=False)
        r = r0.clone()
        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        assert pcg.lib.axhelm_cg_update_box(r.data_ptr(), w.data_ptr(), pcg.dinv.data_ptr(), a.data_ptr(),
                                            nx, ny, nz, 8, 0, nz, 0, 0, int(op.xfolded),
                                            pcg.partial.data_ptr(), out.data_ptr(), s) == 0
        torch.cuda.synchronize()
        res.append((op.xfolded, r, out, float(dot)))
    assert res[0][0] == (nx > 1) and res[1][0] is False
    assert torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][2], res[1][2])
    assert abs(res[0][3] - res[1][3]) <= 1e-12 * max(1.0, abs(res[1][3]))


def _pcg_rank_worker(rank, world, port, dims, exchange, q, mode="strict"):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_20994_b200.cg import JacobiPCG
        from paper_2506_20994_b200.dist import TorchComm
        from paper_2506_20994_b200.mesh import BoxMesh
        from paper_2506_20994_b200.operator import HelmholtzOperator

        nx, ny, nz, lx = dims
        m = BoxMesh(nx, ny, nz, lx, rank, world)
        op = HelmholtzOperator(m, torch, "cuda", comm=TorchComm(dist), mode=mode, exchange=exchange)
        op.fold_unassembled = mode == "fast"
        pcg = JacobiPCG(op)
        gid = m.gid(torch, "cuda")
        fg = torch.from_numpy(np.random.default_rng(2).standard_normal(
            (nx * (lx - 1) + 1) * (ny * (lx - 1) + 1) * (nz * (lx - 1) + 1))).cuda()
        f = fg[gid].contiguous()
        x, hist = pcg.solve(f, iters=15)
        torch.cuda.synchronize()
        x, hist = x.cpu().numpy(), hist.cpu().numpy()
        graph_ok = None
        if exchange == "peer":  # the whole multi-rank solve as a CUDA graph, replayed twice
            graph_ok = True
            for _ in range(2):
                xg, hg = pcg.solve(f, iters=15, graph=True)
                torch.cuda.synchronize()
                graph_ok &= bool(np.array_equal(hg.cpu().numpy(), hist) and np.array_equal(xg.cpu().numpy(), x))
        q.put((rank, x, hist, graph_ok))
        dist.barrier()
        if op.peer is not None:
            op.peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange,world,mode,dims", [("nccl", 2, "strict", (2, 3, 9, 4)),
                                                      ("peer", 2, "strict", (2, 3, 9, 4)),
                                                      ("peer", 3, "strict", (2, 3, 9, 4)),
                                                      ("nccl", 2, "fast", (3, 2, 9, 8)),
                                                      ("peer", 2, "fast", (3, 2, 9, 8))])
def test_pcg_ranks_on_one_gpu(torch, exchange, world, mode, dims):
    """Multi-rank PCG (z-slabs, ranks sharing one GPU): the interface exchange
    and the dot all-reduces through gloo ("nccl" transport path) or through
    peer memory (CUDA IPC; axhelm_gs_box_peer + axhelm_peer_allreduce).  The
    iterates match the single-domain solve to reassociation of the dots, and
    with the peer all-reduce every rank holds the same residual history bit
    for bit; with peer memory the whole multi-rank solve also runs as a
    captured CUDA graph (device-side sequence numbers), bit-identical."""
    import socket

    import torch.multiprocessing as mp

    from paper_2506_20994_b200.mesh import BoxMesh

    nx, ny, nz, lx = dims
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pcg_rank_worker, args=(r, world, port, dims, exchange, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, x, h, gok = q.get(timeout=300)
        res[r] = (x, h)
        assert gok is None or gok, f"rank {r}: graph replay differs from the eager solve"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, op, pcg = _setup(torch, nx, ny, nz, lx, mode)
    gid = m.gid(torch, "cuda")
    fg = torch.from_numpy(np.random.default_rng(2).standard_normal(
        (nx * (lx - 1) + 1) * (ny * (lx - 1) + 1) * (nz * (lx - 1) + 1))).cuda()
    xw, hw = pcg.solve(fg[gid], iters=15)
    hw = hw.cpu().numpy()
    for r in range(world):
        assert np.max(np.abs(res[r][1] - hw) / hw) <= 1e-10, r
    x = np.concatenate([res[r][0] for r in range(world)])
    assert o.normwise_rel(x, xw.cpu().numpy()) <= 1e-10
    if exchange == "peer":
        for r in range(1, world):
            assert np.array_equal(res[r][1], res[0][1])


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_graph_replay_equals_eager(torch, mode):
    """The CUDA-graph PCG (whole solve captured once, replayed) gives the
    eager solve's iterates bit for bit, on repeated replays."""
    m, op, pcg = _setup(torch, 3, 2, 2, 8, mode)
    gid = m.gid(torch, "cuda")
    f = torch.randn(int(gid.max()) + 1, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(9))[gid].contiguous()
    xe, he = pcg.solve(f, iters=20)
    xe, he = xe.clone(), he.clone()
    for _ in range(2):
        xg, hg = pcg.solve(f, iters=20, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(hg, he) and torch.equal(xg, xe)


def test_pcg_converges_to_reference_dense_solve(torch, golden_dir):
    """f2 pinned to reference arithmetic: JacobiPCG on the assembled operator
    converges to x = K_II^-1 f_I (K assembled from the reference's element
    matrices, mdg.sem.dense_assemble; tests/golden/make_assembled_golden.py)
    to 1e-9 of max|x| (800 iterations: the random SPD metric blocks make K
    ill-conditioned), in both the fused and the separate-pass form."""
    from paper_2506_20994_b200.cg import JacobiPCG
    from paper_2506_20994_b200.mesh import BoxMesh
    from paper_2506_20994_b200.operator import HelmholtzOperator

    with np.load(golden_dir / "assembled_cases.npz") as z:
        tags = sorted({k.split("/")[0] for k in z.files})
        cases = [(tag, {k.split("/")[1]: z[k] for k in z.files if k.startswith(tag + "/")}) for tag in tags]
    for tag, c in cases:
        if np.count_nonzero(np.abs(c["x"]) > 0) <= 50:
            continue  # tiny interior: CG terminates exactly (p.Ap = 0)
        dims, lx = tag.split("_lx")
        nx, ny, nz = (int(v) for v in dims.split("x"))
        m = BoxMesh(nx, ny, nz, int(lx))
        geom = {k: torch.from_numpy(c[k]).cuda() for k in ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")}
        for fused in (True, False):
            op = HelmholtzOperator(m, torch, "cuda", mode="fast", geometry=geom)
            pcg = JacobiPCG(op, fused=fused)
            f = torch.from_numpy(c["f"]).cuda()
            x, hist = pcg.solve(f, iters=800)  # random SPD metrics: ill-conditioned
            torch.cuda.synchronize()
            got = x.cpu().numpy()
            err = np.abs(got - c["x"]).max() / np.abs(c["x"]).max()
            assert err <= 1e-9, (tag, fused, err, float(hist[-1]))
