"""Host<->device bandwidth on the GPU box: raw pinned copies vs the
__dace_ax_helm host path (e2e) at several chunk sizes / stream counts.
python tools/pcie.py"""
import ctypes
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

GB = 1 << 30
h = torch.empty(GB // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(GB // 8, dtype=torch.float64, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name} pinned 1 GiB: {5 * GB / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
s2 = torch.cuda.Stream()
h2 = torch.empty_like(h)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D+D2H concurrent: {10 * GB / (time.perf_counter() - t0) / 1e9:.1f} GB/s total", flush=True)
