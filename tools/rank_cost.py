"""Per-rank device cost of one rank of the strong-scaled C4 / C5 problem on
ONE GPU, for a scaling projection where only one GPU is available:
an interior z-slab (both interfaces) of the 128^3-element brick split over
N ranks, with a loopback communicator whose messages are local device copies
(the plane kernels, the boundary-first split and the interior / exchange
overlap all run; only the NVLink transfer itself is missing, ~2 x 6.4 MB
per apply).  Values are numerically meaningless (no neighbour data); the
timing is the rank's.

python tools/rank_cost.py [--world 8] [--steps 50] [--cg-iters 100]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2506_20994_b200.cg import JacobiPCG  # noqa: E402
from paper_2506_20994_b200.mesh import BoxMesh  # noqa: E402
from paper_2506_20994_b200.operator import HelmholtzOperator  # noqa: E402


class LoopbackComm:
    """rank r of `world`: sends land in the matching receive buffer of the
    same process (stream-ordered device copies); all-reduces are identity."""

    host_staged = False

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def sendrecv(self, send=None, dst=None, recv=None, src=None):
        if send is not None and recv is not None and send.shape == recv.shape:
            recv.copy_(send)
        elif recv is not None:
            recv.zero_()

    def allgather_object(self, obj):
        return [obj] * self.world

    def allreduce_sum(self, t):
        return t


ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--cg-iters", type=int, default=100)
a = ap.parse_args()
rank = a.world // 2 if a.world > 1 else 0
mesh = BoxMesh(128, 128, 128, 8, rank, a.world)
comm = LoopbackComm(rank, a.world) if a.world > 1 else None
op = HelmholtzOperator(mesh, torch, "cuda", comm=comm, mode="fast", exchange="nccl")
g = torch.Generator(device="cuda").manual_seed(5)
u = torch.randn(mesh.shape, dtype=torch.float64, device="cuda", generator=g)
w = torch.empty_like(u)
for _ in range(5):
    op.apply(u, w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    op.apply(u, w)
e1.record()
torch.cuda.synchronize()
apply_ms = e0.elapsed_time(e1) / a.steps
pcg = JacobiPCG(op)
f = torch.empty_like(u)
op.apply(u * pcg.mask, f)
pcg.solve(f, iters=3)
torch.cuda.synchronize()
e0.record()
pcg.solve(f, iters=a.cg_iters)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"world": a.world, "rank": rank, "elements": mesh.nel, "overlap": op.overlap,
                  "apply_ms": round(apply_ms, 4), "pcg_ms_per_iter": round(e0.elapsed_time(e1) / a.cg_iters, 4)}))
