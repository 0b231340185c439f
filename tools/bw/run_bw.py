"""python tools/bw/run_bw.py : TMA-ring bandwidth vs ring depth / CTAs per SM."""
import ctypes
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
lib = ctypes.CDLL(str(HERE / "libprobe_bw.so"))
nel = 1 << 18
fields = [torch.randn(nel * 512, dtype=torch.float64, device="cuda") for _ in range(8)]
w = torch.empty(nel * 512, dtype=torch.float64, device="cuda")
fp = torch.tensor([f.data_ptr() for f in fields], dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for write in (1, 0):
    for depth in (2, 3, 4, 6):
        for cps in (1, 2, 3, 4, 6):
            if (depth * 32 + 0.2) * cps > 226:
                continue
            grid = 148 * cps
            args = (ctypes.c_void_p(fp.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_int64(nel),
                    depth, write, grid, 128, ctypes.c_void_p(s))
            for _ in range(3):
                assert lib.probe_bw(*args) == 0
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                lib.probe_bw(*args)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 20
            byts = nel * 4096 * (8 + write)
            print(f"write={write} depth={depth} ctas/sm={cps}: {ms:.4f} ms {byts / ms / 1e6:.0f} GB/s", flush=True)
