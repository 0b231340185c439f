"""Timeline of one follow-schedule apply (ax + concurrent DSSUM follower):
when each element layer became available to the follower, relative to the
follower's start, next to the apply's own duration.
python tools/follow_trace.py [--mode fast] [--nel 262144]"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20994_b200 import _lib  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--nel", type=int, default=1 << 18)
ap.add_argument("--lx", type=int, default=8)
a = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
nx, ny, nz = bench.mesh_dims(a.nel)
m = BoxMesh(nx, ny, nz, a.lx)
op = HelmholtzOperator(m, torch, dev, mode=a.mode, schedule="follow")
u = torch.randn(m.shape, dtype=torch.float64, device=dev)
w = torch.empty_like(u)
for _ in range(3):
    op.apply(u, w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
op.apply(u, w)
e1.record()
torch.cuda.synchronize()
n = nz + 2
buf = (ctypes.c_ulonglong * n)()
assert lib.axhelm_debug_follow_trace(buf, n) == 0
t = [x - buf[0] for x in buf]
print(json.dumps({"apply_ms": round(e0.elapsed_time(e1), 4),
                  "follower_total_us": round(t[-1] / 1e3, 1),
                  "layer_ready_us": [round(x / 1e3, 1) for x in t[1:-1]]}))

# the follower alone after a finished apply (no waiting): its own throughput
op_seq = HelmholtzOperator(m, torch, dev, mode=a.mode, schedule="sequential", geometry=op.geom)
op_seq.ax(u, w)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
f = lib.axhelm_debug_follow_only
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int] + [ctypes.c_int64] * 4 + [ctypes.c_void_p]
for _ in range(2):
    op_seq.ax(u, w)
    torch.cuda.synchronize()
    e0.record()
    assert f(w.data_ptr(), m.nx, m.ny, m.lx, m.ez0, m.ez1, op.zlo, op.zhi, sp) == 0
    e1.record()
    torch.cuda.synchronize()
t_f = e0.elapsed_time(e1)
op_seq.ax(u, w)
torch.cuda.synchronize()
e0.record()
op_seq.gs.sum_local(w)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"follower_alone_ms": round(t_f, 4), "gs_pass_ms": round(e0.elapsed_time(e1), 4)}))
