"""Generate the golden fixtures by importing the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``mdg`` from /root/reference/pkg/src (read-only, in place) and
writes small committed fixtures next to this file.  Nothing at test/bench
time reads /root/reference; the fixtures are what travel.

  gll.json        GLL points/weights/deriv for lx 2..16 as float.hex
                  (mdg.sem.gll_basis, sem.py:182-236)
  ax_cases.npz    full inputs + expected wd for a handful of small cases
                  (mdg.bench._problem inputs, mdg.sem.ax_reference output)
  ax_digests.json sha256 of inputs and of ax_reference's wd for the
                  conformance grid lx 2..16 x nel {1,8,64} (bench seeds),
                  the acceptance grid lx 2..8 x nel {1,8,64} x seeds 0..4
                  (test_acceptance.py:104-114), and config C1 (lx 8, 512
                  elements); plus the reference checksum wd.sum()
  genopt_digests.json  sha256 of wd from the reference's own compiled
                  gen-opt kernel (codegen + kernelrt, strict fp) — proves the
                  compiled reference path agrees bit-for-bit too
  mdgt_2x2.t      MDGT bytes written by mdg.tensorfile.write_tensor
  dump_lx*_nel*/  `mdg run --dump` directories (15 tensors, sizes.txt,
                  expected_wd.t) written by the reference CLI
  lx2_box_stiffness.npy  8x8 dense operator of one lx=2 unit box
                  (mdg.sem.dense_assemble; hand-derived in test_oracle.py:137-158)
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, str(REF))
    import mdg
    from mdg import bench, sem, tensorfile
    from mdg.axprogram import ABI_CONTAINER_ORDER

    # ---- GLL
    gll = {}
    for lx in range(2, 17):
        b = sem.gll_basis(lx)
        gll[str(lx)] = {
            "points": [float(v).hex() for v in b.points],
            "weights": [float(v).hex() for v in b.weights],
            "deriv": [[float(v).hex() for v in row] for row in b.deriv],
        }
    (OUT / "gll.json").write_text(json.dumps(gll, indent=0))

    def ref_apply(arrays, nel, lx):
        basis = sem.gll_basis(lx)
        u = sem.ElementField(nel, lx, arrays["ud"])
        g = sem.GeomFactors(
            g11=arrays["g11d"], g22=arrays["g22d"], g33=arrays["g33d"],
            g12=arrays["g12d"], g13=arrays["g13d"], g23=arrays["g23d"],
            h1=arrays["h1d"],
        )
        return sem.ax_reference(u, basis, g).data

    def seeded(lx, nel, seed):
        # test_acceptance.py:35-40 seeded_inputs
        basis = sem.gll_basis(lx)
        geom = sem.random_spd_geometry(nel, lx, seed)
        rng = np.random.default_rng(seed)
        u = sem.ElementField(nel, lx, rng.standard_normal((nel, lx, lx, lx)))
        return mdg.ax_arrays(u, basis, geom)

    # ---- full small cases
    cases = {}
    for lx, nel in ((2, 3), (3, 2), (4, 2), (5, 2), (6, 1), (7, 1), (8, 2), (12, 1), (16, 1)):
        _, arrays = bench._problem(lx, nel)
        wd = ref_apply(arrays, nel, lx)
        tag = f"lx{lx}_nel{nel}"
        for name in ABI_CONTAINER_ORDER:
            if name != "wd":
                cases[f"{tag}/{name}"] = np.asarray(arrays[name])
        cases[f"{tag}/expected_wd"] = wd
    # box geometry case (sem.py:239-262), lx 4, 2 elements, h = 0.5
    basis = sem.gll_basis(4)
    geom = sem.box_geometry(2, 4, 0.5)
    u = sem.ElementField(2, 4, np.random.default_rng(99).standard_normal((2, 4, 4, 4)))
    arrays = mdg.ax_arrays(u, basis, geom)
    for name in ABI_CONTAINER_ORDER:
        if name != "wd":
            cases[f"box_lx4_nel2/{name}"] = np.asarray(arrays[name])
    cases["box_lx4_nel2/expected_wd"] = sem.ax_reference(u, basis, geom).data
    np.savez_compressed(OUT / "ax_cases.npz", **cases)

    # ---- digests
    digests = {"bench": {}, "acceptance": {}, "C1": {}}
    for lx in range(2, 17):
        for nel in (1, 8, 64):
            _, arrays = bench._problem(lx, nel)
            wd = ref_apply(arrays, nel, lx)
            digests["bench"][f"{lx},{nel}"] = {
                "inputs": {k: sha(arrays[k]) for k in ABI_CONTAINER_ORDER if k != "wd"},
                "wd": sha(wd),
                "checksum": float(wd.sum()).hex(),
                "maxabs": float(np.max(np.abs(wd))).hex(),
            }
    for lx in range(2, 9):
        for nel in (1, 8, 64):
            for seed in range(5):
                arrays = seeded(lx, nel, seed)
                wd = ref_apply(arrays, nel, lx)
                digests["acceptance"][f"{lx},{nel},{seed}"] = {
                    "ud": sha(arrays["ud"]), "g11d": sha(arrays["g11d"]),
                    "h1d": sha(arrays["h1d"]), "wd": sha(wd),
                }
    _, arrays = bench._problem(8, 512)
    wd = ref_apply(arrays, 512, 8)
    digests["C1"] = {
        "lx": 8, "nel": 512,
        "inputs": {k: sha(arrays[k]) for k in ABI_CONTAINER_ORDER if k != "wd"},
        "wd": sha(wd), "checksum": float(wd.sum()).hex(),
        "maxabs": float(np.max(np.abs(wd))).hex(),
        "flops": mdg.flops_model(8, 512),
    }
    (OUT / "ax_digests.json").write_text(json.dumps(digests, indent=1))

    # ---- the reference's own compiled gen-opt kernel agrees bit-for-bit
    from mdg import axprogram, codegen, kernelrt, transforms

    gd = {}
    for lx in (3, 5, 8):
        g = transforms.ax_optimization_recipe(axprogram.build_ax_program(lx, "nel"), lx)
        so = kernelrt.compile_shared(codegen.generate_source(g, codegen.EmitConfig()))
        fn = kernelrt.load_kernel(so)
        for nel in (1, 8, 64):
            _, arrays = bench._problem(lx, nel)
            arrays = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
            arrays["wd"] = np.zeros_like(arrays["wd"])
            fn(arrays, nel, lx)
            gd[f"{lx},{nel}"] = sha(arrays["wd"])
    (OUT / "genopt_digests.json").write_text(json.dumps(gd, indent=1))

    # ---- an `mdg run --dump` directory made by the reference CLI itself
    #      (cli.py:115-153), the cabi-harness conformance input format
    import subprocess
    import tempfile

    for lx, nel in ((4, 8), (8, 2)):
        dump = OUT / f"dump_lx{lx}_nel{nel}"
        with tempfile.TemporaryDirectory() as td:
            env = dict(__import__("os").environ, PYTHONPATH=str(REF))
            graph = Path(td) / "ax.mdg"
            subprocess.run([sys.executable, "-m", "mdg", "build", "--lx", str(lx), "-o", str(graph)],
                           check=True, env=env, capture_output=True)
            subprocess.run([sys.executable, "-m", "mdg", "run", "-i", str(graph), "--nel", str(nel),
                            "--seed", "1", "--dump", str(dump)], check=True, env=env, capture_output=True)

    # ---- MDGT bytes and the lx=2 stiffness
    tensorfile.write_tensor(OUT / "mdgt_2x2.t", np.array([[1.0, 2.0], [3.0, -0.5]]))
    np.save(OUT / "lx2_box_stiffness.npy",
            sem.dense_assemble(sem.gll_basis(2), sem.box_geometry(1, 2, 2.0)))
    print("fixtures written to", OUT)


if __name__ == "__main__":
    main()
