"""e2e host path timing: __dace_ax_helm body with pinned host buffers at C2.
python tools/e2e.py [--reps 3] [--mode fast]"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="fast")
ap.add_argument("--pageable", action="store_true", help="ordinary (pageable) host memory, as a numpy caller passes")
a = ap.parse_args()
lib = _lib.load()
nel, lx = 1 << 18, 8
arr = bench.device_problem(torch, nel, lx, torch.device("cuda", 0))
host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=not a.pageable) for k, v in arr.items()}
for k, v in arr.items():
    host[k].copy_(v)
del arr
torch.cuda.synchronize()
ptrs = [host[n].data_ptr() for n in bench.ABI]
m = 0 if a.mode == "strict" else 1
assert lib.axhelm_apply_sync(*ptrs, nel, lx, m) == 0
ts = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    assert lib.axhelm_apply_sync(*ptrs, nel, lx, m) == 0
    ts.append(time.perf_counter() - t0)
t = min(ts)
h2d = sum(host[n].numel() * 8 for n in bench.ABI if n != "wd")
print(f"e2e ({'pageable' if a.pageable else 'pinned'}) {t * 1e3:.1f} ms  {nel * lx ** 3 / t / 1e9:.3f} GDOF/s  H2D {h2d / t / 1e9:.1f} GB/s", flush=True)
