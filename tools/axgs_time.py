"""Assembled operator w = QQ^T A u on the C2 brick (sequential schedule):
mean ms per apply over --reps (CUDA events), for same-box A/B of library
builds (AXHELM_LIB=...): python tools/axgs_time.py [--reps 50] [--mode fast]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--mode", default="fast")
ap.add_argument("--n", type=int, default=64)
a = ap.parse_args()
m = BoxMesh(a.n, a.n, a.n, 8)
op = HelmholtzOperator(m, torch, "cuda", mode=a.mode)
u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
for _ in range(5):
    op.apply(u, w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    op.apply(u, w)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"mode": a.mode, "ms": round(e0.elapsed_time(e1) / a.reps, 4),
                  "checksum": float(w.double().sum())}))
