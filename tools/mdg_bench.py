"""`mdg bench` for the B200 kernel: the reference's sweep and CSV format
(mdg/bench.py:23-27 FULL_MESH_SIZES / CSV_HEADER, :69-174 run_bench) with
"gpu-strict" and "gpu-fast" variants, so the reference's own `read_csv` and
`plotsvg.render_records` (plotsvg.py:101-135) consume the output unchanged
(SURVEY §8f row 3).

Protocol as run_bench: per (lx, nel) one warm-up run that doubles as the
checksum run, then `reps` timed runs, median; Gflop/s from the flop model
nel*lx^3*(12 lx + 18) (sem.py:367-375); unknowns = nel*(lx-1)^3
(bench.py:162).  Timing: CUDA events around each apply on the launching
stream (device-resident inputs, synthetic device-generated data of the
reference's distribution, bench.device_problem).  Gate: gpu-fast is held to
the reference's relaxed-fp bar (1e-12 normwise vs gpu-strict,
tests/test_codegen.py:180-187) — its checksum cannot meet the bit-exactness
the 1e-10 relative checksum gate implies (SURVEY §7 hard part 3).

python tools/mdg_bench.py [--lx 3-8] [--max-nel 32768] [--reps 9] [--out gpu_bench.csv]
"""
from __future__ import annotations

import argparse
import ctypes
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

FULL_MESH_SIZES = (128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768)  # bench.py:23
CSV_HEADER = "lx,nel,unknowns,variant,seconds_median,gflops,checksum"  # bench.py:25
VARIANTS = ("gpu-strict", "gpu-fast")
FAST_TOL = 1e-12


def flops_model(lx: int, nel: int) -> int:
    return nel * lx ** 3 * (12 * lx + 18)


def render_csv(records) -> str:
    """Same text as mdg.bench.render_csv (repr floats)."""
    lines = [CSV_HEADER]
    for r in records:
        lines.append(f"{r['lx']},{r['nel']},{r['unknowns']},{r['variant']},"
                     f"{r['seconds_median']!r},{r['gflops']!r},{r['checksum']!r}")
    return "\n".join(lines) + "\n"


def run(lx_range=(3, 8), meshes=FULL_MESH_SIZES, max_nel=32768, reps=9, log=print):
    import torch

    import bench
    from paper_2506_20994_b200 import _lib, kernelrt

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(st.cuda_stream)
    records = []
    for lx in range(lx_range[0], lx_range[1] + 1):
        for nel in (n for n in meshes if n <= max_nel):
            arr = bench.device_problem(torch, nel, lx, dev, seed=7919 * lx + nel)
            ptrs = [arr[n].data_ptr() for n in bench.ABI]
            ref = None
            for variant in VARIANTS:
                mode = kernelrt.MODES[variant.split("-")[1]]

                def apply():
                    rc = lib.axhelm_apply(*ptrs, nel, lx, mode, sp)
                    if rc:
                        raise RuntimeError(_lib.last_error(lib))

                apply()  # warm-up = checksum run (bench.py:139-152)
                torch.cuda.synchronize()
                wd = arr["wd"].clone()
                checksum = float(wd.sum())
                if ref is None:
                    ref = wd
                else:
                    err = float((wd - ref).abs().max() / ref.abs().max())
                    if err > FAST_TOL:
                        raise RuntimeError(f"lx={lx} nel={nel} {variant}: {err:.3e} > {FAST_TOL} vs gpu-strict")
                times = []
                for _ in range(reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    apply()
                    e1.record(st)
                    e1.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e-3)
                sec = statistics.median(times)
                rec = {"lx": lx, "nel": nel, "unknowns": nel * (lx - 1) ** 3, "variant": variant,
                       "seconds_median": sec, "gflops": flops_model(lx, nel) / sec / 1e9, "checksum": checksum}
                records.append(rec)
                if log:
                    log(f"lx={lx} nel={nel} {variant}: {sec:.6f} s, {rec['gflops']:.3f} Gflops/s")
            del arr
    return records


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lx", default="3-8")
    ap.add_argument("--max-nel", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--out", default="gpu_bench.csv")
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.lx.split("-")) if "-" in a.lx else (int(a.lx), int(a.lx))
    recs = run((lo, hi), max_nel=a.max_nel, reps=a.reps, log=lambda s: print(s, file=sys.stderr))
    Path(a.out).write_text(render_csv(recs), encoding="ascii")
    print(a.out)


if __name__ == "__main__":
    main()
