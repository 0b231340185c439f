"""Assembled operator (ax + DSSUM) time vs L2 block size on one GPU:
python tools/gs_block_sweep.py [--lx 8] [--nel 262144] [--mode fast] [--blocks 0,1,2,3,4,6,8]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lx", type=int, default=8)
ap.add_argument("--nel", type=int, default=1 << 18)
ap.add_argument("--mode", default="fast")
ap.add_argument("--blocks", default="sequential,follow,2,4,8")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
dev = torch.device("cuda", 0)
nx, ny, nz = bench.mesh_dims(a.nel)
m = BoxMesh(nx, ny, nz, a.lx)
geom = None
u = torch.randn(m.shape, dtype=torch.float64, device=dev)
w = torch.empty_like(u)
ref = None
for b in (x if not x.isdigit() else int(x) for x in a.blocks.split(",")):
    op = HelmholtzOperator(m, torch, dev, mode=a.mode, geometry=geom, schedule=b)
    geom = op.geom
    for _ in range(3):
        op.apply(u, w)
    torch.cuda.synchronize()
    if ref is None:
        ref = w.clone()
    same = bool(torch.equal(w, ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        op.apply(u, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    pts = m.nel * a.lx ** 3
    print(json.dumps({"lx": a.lx, "nel": m.nel, "mesh": [nx, ny, nz], "mode": a.mode, "schedule": b,
                      "ms": round(ms, 4), "gdof_s": round(pts / ms / 1e6, 2), "bit_equal_sequential": same}),
          flush=True)
