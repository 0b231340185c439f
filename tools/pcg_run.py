"""A few Jacobi-PCG iterations on the C2 brick (64^3 elements, lx=8) for
profiling: python tools/pcg_run.py [--iters 3] [--fused 1] [--mode fast]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.cg import JacobiPCG  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--fused", type=int, default=1)
ap.add_argument("--mode", default="fast")
ap.add_argument("--n", type=int, default=64)
a = ap.parse_args()
m = BoxMesh(a.n, a.n, a.n, 8)
op = HelmholtzOperator(m, torch, "cuda", mode=a.mode)
pcg = JacobiPCG(op, fused=bool(a.fused))
u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
f = torch.empty_like(u)
op.apply(u * pcg.mask, f)
pcg.solve(f, iters=a.iters)
torch.cuda.synchronize()
print("done")
