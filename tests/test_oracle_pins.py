"""Pin the CPU oracle to the reference before trusting it (CPU only).

Every fixture here was produced by importing the reference package itself
(tests/golden/make_golden.py).  The oracle restatements in oracle/ must
reproduce them bit-for-bit.
"""

import json

import numpy as np
import pytest

from oracle import oracle as o

ABI = o.ABI_ORDER


@pytest.fixture(scope="module")
def digests(golden_dir):
    return json.loads((golden_dir / "ax_digests.json").read_text())


@pytest.fixture(scope="module")
def cases(golden_dir):
    with np.load(golden_dir / "ax_cases.npz") as z:
        return {k: z[k] for k in z.files}


def _case(cases, tag):
    return {name: cases[f"{tag}/{name}"] for name in ABI if name != "wd"}, cases[f"{tag}/expected_wd"]


class TestGll:
    """sem.gll_basis frozen values (tests/test_gll.py:46-71) and full bit pins."""

    def test_bit_exact_all_lx(self, golden_dir):
        ref = json.loads((golden_dir / "gll.json").read_text())
        for lx in range(2, 17):
            x, w, d = o.gll(lx)
            want = ref[str(lx)]
            assert [v.hex() for v in x] == want["points"], lx
            assert [v.hex() for v in w] == want["weights"], lx
            assert [[v.hex() for v in row] for row in d] == want["deriv"], lx

    def test_frozen_closed_forms(self):
        x, w, d = o.gll(2)
        assert list(x) == [-1.0, 1.0] and list(w) == [1.0, 1.0]
        np.testing.assert_allclose(d, [[-0.5, 0.5], [-0.5, 0.5]], atol=1e-15)
        x, w, _ = o.gll(3)
        np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], atol=1e-15)
        x, _, _ = o.gll(4)
        r = 1 / np.sqrt(5.0)
        np.testing.assert_allclose(x, [-1, -r, r, 1], atol=1e-15)
        x, w, _ = o.gll(8)
        assert abs(float(np.sum(w * x**12)) - 2 / 13) <= 1e-12

    def test_range(self):
        for bad in (0, 1, 17):
            with pytest.raises(ValueError):
                o.gll(bad)


class TestAxAgainstReference:
    def test_full_cases_bit_exact(self, cases):
        tags = sorted({k.split("/")[0] for k in cases})
        assert len(tags) == 10
        for tag in tags:
            arrays, want = _case(cases, tag)
            got = o.ax(arrays)
            assert np.array_equal(got, want), tag
            assert o.digest(got) == o.digest(want), tag

    def test_problem_regenerates_fixture_inputs(self, cases):
        for lx, nel in ((2, 3), (5, 2), (8, 2), (16, 1)):
            arrays = o.problem(lx, nel)
            fix, _ = _case(cases, f"lx{lx}_nel{nel}")
            for name, a in fix.items():
                assert np.array_equal(arrays[name], a), (lx, nel, name)

    def test_box_geometry_case(self, cases):
        arrays, want = _case(cases, "box_lx4_nel2")
        g = o.box_geometry(2, 4, 0.5)
        for name, a in g.items():
            assert np.array_equal(a, arrays[name]), name
        assert np.array_equal(o.ax(arrays), want)

    def test_bench_grid_digests(self, digests):
        """lx 2..16 x nel {1,8,64}, bench._problem seeds: inputs and wd bit-exact."""
        for key, rec in digests["bench"].items():
            lx, nel = map(int, key.split(","))
            arrays = o.problem(lx, nel)
            for name, h in rec["inputs"].items():
                assert o.digest(arrays[name]) == h, (key, name)
            wd = o.ax(arrays)
            assert o.digest(wd) == rec["wd"], key
            assert float(wd.sum()).hex() == rec["checksum"], key

    def test_acceptance_grid_digests(self, digests):
        """test_acceptance.py:104-114 grid: lx 2..8 x nel {1,8,64} x seeds 0..4."""
        for key, rec in digests["acceptance"].items():
            lx, nel, seed = map(int, key.split(","))
            arrays = o.problem(lx, nel, seed=seed)
            assert o.digest(arrays["ud"]) == rec["ud"], key
            assert o.digest(arrays["g11d"]) == rec["g11d"], key
            assert o.digest(o.ax(arrays)) == rec["wd"], key

    def test_c1_numpy_and_c(self, digests):
        c1 = digests["C1"]
        arrays = o.problem(8, 512)
        for name, h in c1["inputs"].items():
            assert o.digest(arrays[name]) == h, name
        assert o.digest(o.ax(arrays)) == c1["wd"]
        if o.c_oracle() is not None:
            assert o.digest(o.ax_c(arrays)) == c1["wd"]
        assert o.flops_model(8, 512) == c1["flops"]

    def test_reference_genopt_agrees(self, golden_dir, digests):
        """The reference's compiled gen-opt kernel (strict fp) = ax_reference."""
        gd = json.loads((golden_dir / "genopt_digests.json").read_text())
        for key, h in gd.items():
            assert digests["bench"][key]["wd"] == h, key


class TestCOracle:
    def test_matches_numpy(self):
        if o.c_oracle() is None:
            pytest.skip("oracle/liboracle_ax.so not built")
        for lx in (2, 3, 7, 9, 12, 16):
            arrays = o.problem(lx, 5)
            assert np.array_equal(o.ax_c(arrays, nthreads=2), o.ax(arrays)), lx

    def test_honours_all_six_matrix_slots(self):
        if o.c_oracle() is None:
            pytest.skip("oracle/liboracle_ax.so not built")
        rng = np.random.default_rng(4)
        arrays = o.problem(4, 3)
        for name in o.MATRICES:
            arrays[name] = rng.standard_normal((4, 4))
        assert np.array_equal(o.ax_c(arrays), o.ax(arrays))


class TestOperatorProperties:
    """test_oracle.py:129-246 pins restated on the oracle."""

    def test_lx2_box_stiffness(self, golden_dir):
        want = np.load(golden_dir / "lx2_box_stiffness.npy")
        g = o.box_geometry(8, 2, 2.0)
        a, b = o.operator_matrices(o.gll(2)[2])
        arrays = {"ud": np.eye(8).reshape(8, 2, 2, 2), **g}
        for n in ("dxd", "dyd", "dzd"):
            arrays[n] = a
        for n in ("dxtd", "dytd", "dztd"):
            arrays[n] = b
        dense = o.ax(arrays).reshape(8, 8).T
        assert np.array_equal(dense, want)
        hand = np.zeros((8, 8))
        for p in range(8):
            for q in range(8):
                ham = bin(p ^ q).count("1")
                hand[p, q] = 1.5 if ham == 0 else (-0.5 if ham == 1 else 0.0)
        np.testing.assert_allclose(dense, hand, atol=1e-14)

    @pytest.mark.parametrize("lx", [2, 4, 6])
    def test_annihilates_constants(self, lx):
        arrays = o.problem(lx, 2, seed=3)
        arrays["ud"] = np.full_like(arrays["ud"], 3.75)
        scale = max(float(np.abs(arrays[f]).max()) for f in o.FIELDS if f != "ud")
        assert np.abs(o.ax(arrays)).max() <= 1e-11 * 3.75 * scale

    def test_flops_frozen(self):
        assert o.flops_model(2, 1) == 336
        assert o.flops_model(8, 32768) == 1_912_602_624
        assert o.flops_model(3, 0) == 0

    def test_mdgt_golden_bytes(self, golden_dir):
        blob = (golden_dir / "mdgt_2x2.t").read_bytes()
        assert o.mdgt_encode(np.array([[1.0, 2.0], [3.0, -0.5]])) == blob


def _assembled_cases(golden_dir):
    with np.load(golden_dir / "assembled_cases.npz") as z:
        tags = sorted({k.split("/")[0] for k in z.files})
        for tag in tags:
            dims, lx = tag.split("_lx")
            nx, ny, nz = (int(v) for v in dims.split("x"))
            yield (nx, ny, nz, int(lx)), {k.split("/")[1]: z[k] for k in z.files if k.startswith(tag + "/")}


def test_oracle_dssum_and_pcg_pinned_to_reference_assembly(golden_dir):
    """f1/f2 parity anchor: the oracle's assembled operator dssum(ax(u)) and
    its PCG reproduce the global stiffness assembled from the reference's
    own element matrices (mdg.sem.dense_assemble, sem.py:340-364;
    tests/golden/make_assembled_golden.py): w to 1e-12 normwise, the
    converged x to 1e-9 of the dense solve."""
    for (nx, ny, nz, lx), c in _assembled_cases(golden_dir):
        gid = o.box_mesh_gid(nx, ny, nz, lx)
        a, b = o.operator_matrices(o.gll(lx)[2])
        arrays = {k: c[k] for k in ("h1d", "g11d", "g22d", "g33d", "g12d", "g13d", "g23d")}
        arrays.update({"dxd": a, "dyd": a, "dzd": a, "dxtd": b, "dytd": b, "dztd": b})
        arrays["ud"] = c["u"]
        arrays["wd"] = np.zeros_like(c["u"])
        w = o.dssum(o.ax(arrays), gid)
        assert o.normwise_rel(w, c["w"]) <= 1e-12, (nx, ny, nz, lx)
        mask = o.gs_boundary_mask(nx, ny, nz, lx)
        # the NumPy PCG is slow (the GPU test covers every case); a 7-node
        # interior converges exactly and breaks down (p.Ap = 0): w only
        if lx <= 5 and np.count_nonzero(np.abs(c["x"]) > 0) > 50:
            x, _ = o.pcg(arrays, gid, mask, c["f"], iters=150)
            assert np.abs(x - c["x"]).max() <= 1e-9 * np.abs(c["x"]).max(), (nx, ny, nz, lx)


def test_signed_zero_inputs_pinned(golden_dir):
    """u with exact zeros of both signs (tests/golden/make_zero_golden.py,
    digests written by the reference's sem.ax_reference): the oracle's
    running sums from +0.0 give the reference's zero signs bit for bit."""
    import sys

    sys.path.insert(0, str(golden_dir))
    from make_zero_golden import CASES, zero_inputs

    want = json.loads((golden_dir / "zero_digests.json").read_text())
    for lx, nel in CASES:
        arrays = zero_inputs(o.problem(lx, nel))
        assert o.digest(o.ax(arrays)) == want[f"{lx},{nel}"]["w"], (lx, nel)
