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
