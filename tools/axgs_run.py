"""A few assembled applies w = QQ^T A u (sequential schedule: the x-folding
DMMA apply + the DSSUM pass) on the C2 brick, for profiling:
python tools/axgs_run.py [--reps 3] [--mode fast]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="fast")
ap.add_argument("--n", type=int, default=64)
a = ap.parse_args()
m = BoxMesh(a.n, a.n, a.n, 8)
op = HelmholtzOperator(m, torch, "cuda", mode=a.mode)
u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
for _ in range(a.reps):
    op.apply(u, w)
torch.cuda.synchronize()
print("done")
