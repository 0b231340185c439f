"""PCG per-iteration time, eager vs CUDA-graph replay, across problem sizes
(the small ones are launch-bound): python tools/pcg_graph.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.cg import JacobiPCG  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

iters = 100
for n in (4, 8, 16, 32, 64):
    m = BoxMesh(n, n, n, 8)
    op = HelmholtzOperator(m, torch, "cuda", mode="fast")
    pcg = JacobiPCG(op)
    u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
    f = torch.empty_like(u)
    op.apply(u * pcg.mask, f)
    res = {}
    for graph in (False, True):
        pcg.solve(f, iters=iters, graph=graph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pcg.solve(f, iters=iters, graph=graph)
        e1.record()
        torch.cuda.synchronize()
        res[graph] = e0.elapsed_time(e1) / iters
    print(f"{n}^3 elements ({m.nel}): eager {res[False] * 1e3:8.1f} us/iter   graph {res[True] * 1e3:8.1f} us/iter"
          f"   {res[False] / res[True]:.2f}x", flush=True)
