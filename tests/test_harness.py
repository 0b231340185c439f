"""The cabi-harness flow (reference pkg/cabi-harness: run.ts:31-78,
compare.ts:10-27, conformance.test.ts:63-99) against `mdg run --dump`
directories the reference CLI produced (tests/golden/dump_*)."""

import shutil

import numpy as np
import pytest

from tools import axrun
from paper_2506_20994_b200.tensorfile import read_tensor, write_tensor


def test_compare_exit_codes(tmp_path, golden_dir):
    want = golden_dir / "dump_lx4_nel8" / "expected_wd.t"
    assert axrun.main(["compare", "-a", str(want), "-b", str(want)]) == 0
    w = read_tensor(want)
    w.flat[3] += 1e-9
    got = tmp_path / "g.t"
    write_tensor(got, w)
    assert axrun.main(["compare", "-a", str(got), "-b", str(want)]) == 1
    assert axrun.main(["compare", "-a", str(got), "-b", str(want), "--rtol", "1e-6"]) == 0
    bad = tmp_path / "bad.t"
    bad.write_bytes(b"XXXX")
    assert axrun.main(["compare", "-a", str(bad), "-b", str(want)]) == 5
    write_tensor(got, w[:1])
    assert axrun.main(["compare", "-a", str(got), "-b", str(want)]) == 4


def test_run_rejects_bad_dumps(tmp_path, golden_dir):
    d = tmp_path / "dump"
    shutil.copytree(golden_dir / "dump_lx4_nel8", d)
    (d / "sizes.txt").write_text("9 4\n")  # dims disagree with sizes.txt
    assert axrun.main(["run", "--inputs", str(d), "-o", str(tmp_path / "o.t")]) == 4
    (d / "sizes.txt").write_text("8 four\n")
    assert axrun.main(["run", "--inputs", str(d), "-o", str(tmp_path / "o.t")]) == 5
    (d / "sizes.txt").write_text("8 4\n")
    assert axrun.main(["run", "--inputs", str(d), "-o", str(tmp_path / "o.t"), "--entry", "nope"]) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("dump", ["dump_lx4_nel8", "dump_lx8_nel2"])
def test_conformance_strict_and_fast(tmp_path, golden_dir, dump):
    d = golden_dir / dump
    out = tmp_path / "wd.t"
    assert axrun.main(["run", "--inputs", str(d), "-o", str(out), "--mode", "strict"]) == 0
    assert axrun.main(["compare", "-a", str(out), "-b", str(d / "expected_wd.t")]) == 0
    assert axrun.main(["run", "--inputs", str(d), "-o", str(out), "--mode", "fast"]) == 0
    assert axrun.main(["compare", "-a", str(out), "-b", str(d / "expected_wd.t"), "--rtol", "1e-12"]) == 0


def _records():
    return [{"lx": 8, "nel": 128, "unknowns": 128 * 343, "variant": "gpu-strict", "seconds_median": 1.5e-05,
             "gflops": 3.14, "checksum": -1.25e-11},
            {"lx": 8, "nel": 128, "unknowns": 128 * 343, "variant": "gpu-fast", "seconds_median": 1.25e-05,
             "gflops": 3.77, "checksum": 2.5e-12}]


def test_mdg_bench_csv_matches_reference_format():
    """tools/mdg_bench writes the reference's CSV (mdg/bench.py:25, :180-191):
    exact header, 7 fields, repr floats."""
    from tools import mdg_bench

    text = mdg_bench.render_csv(_records())
    lines = text.splitlines()
    assert lines[0] == "lx,nel,unknowns,variant,seconds_median,gflops,checksum"
    for line in lines[1:]:
        f = line.split(",")
        assert len(f) == 7
        int(f[0]), int(f[1]), int(f[2]), float(f[4]), float(f[5]), float(f[6])
    assert lines[1].endswith(",1.5e-05,3.14,-1.25e-11")


def test_mdg_bench_csv_parses_with_the_reference(tmp_path):
    """The reference's own read_csv and SVG renderer consume the file (in the
    build container, where /root/reference exists)."""
    import sys
    from pathlib import Path

    src = Path("/root/reference/pkg/src")
    if not src.exists():
        pytest.skip("reference not mounted (GPU box)")
    sys.path.insert(0, str(src))
    try:
        from mdg import bench as rbench
        from mdg import plotsvg
    finally:
        sys.path.remove(str(src))
    from tools import mdg_bench

    recs = rbench.read_csv(mdg_bench.render_csv(_records()))
    assert [r.variant for r in recs] == ["gpu-strict", "gpu-fast"]
    svg = plotsvg.render_records(recs)
    assert svg.lstrip().startswith("<svg") or "<svg" in svg
