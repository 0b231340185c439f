"""Minimal driver for profiling: N applies of ax_helm on device-generated
inputs (python tools/run_ax.py --lx 8 --nel 262144 --mode strict --reps 3)."""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200 import _lib, kernelrt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lx", type=int, default=8)
ap.add_argument("--nel", type=int, default=1 << 18)
ap.add_argument("--mode", default="strict")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
lib = _lib.load()
arr = bench.device_problem(torch, a.nel, a.lx, torch.device("cuda", 0))
ptrs = [arr[n].data_ptr() for n in bench.ABI]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(a.reps):
    assert lib.axhelm_apply(*ptrs, a.nel, a.lx, kernelrt.MODES[a.mode], s) == 0
torch.cuda.synchronize()
print("done")
