"""Polynomial-order sweep (BASELINE config C3): lx = 2..16 at ~1e8 GLL
points, both modes; prints one JSON line per (lx, mode).
python tools/sweep.py [--lx 2-12] [--points 1e8] [--reps 20]"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200 import _lib, kernelrt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lx", default="2-12")
ap.add_argument("--points", type=float, default=1e8)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--modes", default="fast,strict")
a = ap.parse_args()
lo, hi = (int(x) for x in a.lx.split("-")) if "-" in a.lx else (int(a.lx), int(a.lx))
lib = _lib.load()
dev = torch.device("cuda", 0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for lx in range(lo, hi + 1):
    nel = int(round(a.points / lx ** 3))
    arr = bench.device_problem(torch, nel, lx, dev)
    ptrs = [arr[n].data_ptr() for n in bench.ABI]
    for mode in a.modes.split(","):
        m = kernelrt.MODES[mode]
        for _ in range(3):
            assert lib.axhelm_apply(*ptrs, nel, lx, m, s) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            lib.axhelm_apply(*ptrs, nel, lx, m, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        pts = nel * lx ** 3
        print(json.dumps({"lx": lx, "nel": nel, "mode": mode, "ms": round(ms, 4),
                          "gdof_s": round(pts / ms / 1e6, 2), "hbm_gbs": round(72 * pts / ms / 1e6, 1),
                          "gflops": round(nel * lx ** 3 * (12 * lx + 18) / ms / 1e6, 1),
                          "kernel": bench.kernel_name(lx, mode)}), flush=True)
    del arr
    torch.cuda.empty_cache()
