"""Build oracle/_ref: the REFERENCE's own compiled CPU kernel (gen-opt).

TEST/BASELINE INFRASTRUCTURE ONLY.  Runs the reference pipeline exactly as
its benchmark does (mdg/bench.py:50-66): build_ax_program ->
ax_optimization_recipe -> generate_source (strict fp) -> kernelrt.compile_shared
(-O2 -std=c99 -shared -fPIC -ffp-contract=off -fopenmp, kernelrt.py:61-71).
Outputs go only to oracle/_ref/lx<L>/{kernel.c,libkernel.so} (git-ignored;
the .so travels to the GPU box where bench.py --impl reference and the
cpu_baseline leg load it through the reference ABI).

Needs /root/reference (this container only); a no-op elsewhere.
"""

from __future__ import annotations

import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "_ref"
LXS = tuple(range(2, 13))


def main(lxs=LXS) -> int:
    if not REF.exists():
        print("build_ref: /root/reference absent; keeping prebuilt oracle/_ref")
        return 0
    sys.path.insert(0, str(REF))
    from mdg import axprogram, codegen, kernelrt, transforms

    for lx in lxs:
        d = OUT / f"lx{lx}"
        so = d / "libkernel.so"
        if so.exists():
            continue
        g = transforms.ax_optimization_recipe(axprogram.build_ax_program(lx, "nel"), lx)
        src = codegen.generate_source(g, codegen.EmitConfig(strict_fp=True))
        kernelrt.compile_shared(src, out_dir=d, strict_fp=True, compiler="gcc")
    print(f"build_ref: reference gen-opt kernels in {OUT}")
    return 0


if __name__ == "__main__":
    import warnings

    warnings.simplefilter("ignore")
    sys.exit(main())
