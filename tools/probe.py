"""Timing experiments on the GPU box: the stream probe (memory ceiling of
the ring design) vs the apply, over a few step counts, with clocks.
python tools/probe.py"""
import ctypes
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200 import _lib  # noqa: E402

lib = _lib.load()
nel, lx = 1 << 18, 8
arr = bench.device_problem(torch, nel, lx, torch.device("cuda", 0))
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ptrs = [arr[n].data_ptr() for n in bench.ABI]
probe_ptrs = [arr[n].data_ptr() for n in ("wd", "ud", "h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")]


def timeit(fn, steps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    clk = bench.ClockSampler(0)
    time.sleep(0.1)
    t0w = time.time()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    c = clk.stop(t0w, time.time())
    return a.elapsed_time(b) / steps, c


import os
which = os.environ.get("PROBE_ONLY", "probe,strict,fast").split(",")
for name, fn in [
    ("probe", lambda: lib.axhelm_probe_stream(*probe_ptrs, nel, s)),
    ("strict", lambda: lib.axhelm_apply(*ptrs, nel, lx, 0, s)),
    ("fast", lambda: lib.axhelm_apply(*ptrs, nel, lx, 1, s)),
]:
    if name not in which:
        continue
    for steps in (5, 50, 300):
        ms, c = timeit(fn, steps)
        print(f"{name:7s} steps={steps:4d} {ms:.4f} ms  {72 * nel * 512 / ms / 1e6:.0f} GB/s  clk={c['sm_mhz']} {c['reasons']}")
