"""Jacobi-PCG iterations on the C2 brick, mean ms per iteration (CUDA events),
for same-box A/B of library builds (AXHELM_LIB=...):
python tools/pcg_time.py [--iters 100] [--mode fast]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.cg import JacobiPCG  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--mode", default="fast")
ap.add_argument("--n", type=int, default=64)
a = ap.parse_args()
m = BoxMesh(a.n, a.n, a.n, 8)
op = HelmholtzOperator(m, torch, "cuda", mode=a.mode)
pcg = JacobiPCG(op)
g = torch.Generator(device="cuda").manual_seed(3)
u = torch.randn(m.shape, dtype=torch.float64, device="cuda", generator=g)
f = torch.empty_like(u)
op.apply(u * pcg.mask, f)
pcg.solve(f, iters=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_, hist = pcg.solve(f, iters=a.iters)
e1.record()
torch.cuda.synchronize()
h = hist.cpu()
print(json.dumps({"mode": a.mode, "ms_per_iter": round(e0.elapsed_time(e1) / a.iters, 4),
                  "rr_reduction": float(h[-1] / h[0])}))
