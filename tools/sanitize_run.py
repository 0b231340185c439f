"""Small workload touching every kernel family once, for compute-sanitizer:
python tools/sanitize_run.py  (run as: compute-sanitizer --tool memcheck python tools/sanitize_run.py)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_20994_b200 import load_kernel  # noqa: E402
from paper_2506_20994_b200.cg import JacobiPCG  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

rng = np.random.default_rng(0)
for lx in (3, 5, 7, 8, 9, 12, 16):
    for mode in ("strict", "fast"):
        nel = 5
        arr = {n: torch.from_numpy(rng.standard_normal((lx, lx))).cuda() for n in
               ("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd")}
        for n in ("ud", "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d"):
            arr[n] = torch.from_numpy(rng.standard_normal((nel, lx, lx, lx))).cuda()
        arr["wd"] = torch.zeros(nel, lx, lx, lx, dtype=torch.float64, device="cuda")
        load_kernel(mode=mode)(arr, nel, lx)
# persistent line kernels (v11; v12 for fast lx 9 / 10) with more groups than
# resident CTAs: the u buffer
# re-armed by TMA, the mbarrier parity flipping, the geometry pipeline and
# prefetches crossing elements (lx 7: three elements per CTA, partial group)
for lx, nel in ((7, 1801), (9, 701), (10, 601), (16, 321)):
    arr = {n: torch.from_numpy(rng.standard_normal((lx, lx))).cuda() for n in
           ("dxd", "dyd", "dzd", "dxtd", "dytd", "dztd")}
    for n in ("ud", "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d"):
        arr[n] = torch.from_numpy(rng.standard_normal((nel, lx, lx, lx))).cuda()
    arr["wd"] = torch.zeros(nel, lx, lx, lx, dtype=torch.float64, device="cuda")
    for mode in ("strict", "fast"):
        load_kernel(mode=mode)(arr, nel, lx)
torch.cuda.synchronize()
for sched in ("sequential", "follow", 1):
    m = BoxMesh(3, 2, 4, 8)
    op = HelmholtzOperator(m, torch, "cuda", mode="fast", schedule=sched)
    u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
    w = torch.empty_like(u)
    d = torch.zeros(1, dtype=torch.float64, device="cuda")
    op.apply(u, w, dot=d)
pcg = JacobiPCG(op)
pcg.solve(u * pcg.mask, iters=3)
# x-folding apply with multi-element CTA segments (folds inside segments and
# at seams), assembled and unassembled (PCG update reading folded nodes once)
m = BoxMesh(16, 8, 8, 8)
op = HelmholtzOperator(m, torch, "cuda", mode="fast")
u = torch.randn(m.shape, dtype=torch.float64, device="cuda")
w = torch.empty_like(u)
op.apply(u, w)
op.fold_unassembled = True
pcg = JacobiPCG(op)
pcg.solve(u * pcg.mask, iters=2)
torch.cuda.synchronize()
print("sanitize workload done")
