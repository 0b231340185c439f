"""DSSUM timing on the GPU box: structured (box) vs CSR gather-scatter on the
C2-sized mesh (64^3 elements, lx=8) and the ax + DSSUM step.
python tools/bench_gs.py [--n 64] [--lx 8] [--reps 20]"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200 import _lib, kernelrt  # noqa: E402
from paper_2506_20994_b200.dist import SlabDSSUM  # noqa: E402
from paper_2506_20994_b200.gs import BoxGatherScatter, GatherScatter  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--lx", type=int, default=8)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--csr", action="store_true")
a = ap.parse_args()
m = BoxMesh(a.n, a.n, a.n, a.lx)
dev = torch.device("cuda", 0)
arr = {**m.geometry(torch, dev), **m.matrices(torch, dev)}
arr["ud"] = torch.randn(m.shape, dtype=torch.float64, device=dev)
arr["wd"] = torch.empty_like(arr["ud"])
lib = _lib.load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ptrs = [arr[n].data_ptr() for n in kernelrt.ABI_CONTAINER_ORDER]


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


box = BoxGatherScatter(m, torch, dev)
dbox = SlabDSSUM(box)
pts = m.nel * a.lx ** 3
t = timeit(lambda: dbox(arr["wd"]), a.reps)
print(f"gs box : {t:.4f} ms  {box.bytes_per_apply() / t / 1e6:.0f} GB/s (algorithmic {box.bytes_per_apply()/1e9:.3f} GB)")
if a.csr:
    csr = GatherScatter(m, torch, dev)
    dcsr = SlabDSSUM(csr)
    t = timeit(lambda: dcsr(arr["wd"]), a.reps)
    print(f"gs csr : {t:.4f} ms  {csr.bytes_per_apply() / t / 1e6:.0f} GB/s (algorithmic {csr.bytes_per_apply()/1e9:.3f} GB)")
for mode in ("fast", "strict"):
    ax = lambda: lib.axhelm_apply(*ptrs, m.nel, a.lx, kernelrt.MODES[mode], s)  # noqa: E731
    t_ax = timeit(ax, a.reps)

    def step():
        ax()
        dbox(arr["wd"])

    t_st = timeit(step, a.reps)
    print(f"{mode:6s} ax {t_ax:.4f} ms ({pts / t_ax / 1e6:.1f} GDOF/s)   ax+gs {t_st:.4f} ms ({pts / t_st / 1e6:.1f} GDOF/s)")
