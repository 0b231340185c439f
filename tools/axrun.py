"""Mirror of the reference cabi-harness `run` / `compare` commands over MDGT
dumps (cabi-harness/src/run.ts:31-78, compare.ts:10-27, exit codes
errors.ts:1-7), driving this package's __dace_ax_helm.

  python tools/axrun.py run --inputs DIR -o out.t [--entry SYMBOL] [--lib PATH]
  python tools/axrun.py compare -a got.t -b want.t [--rtol X]

DIR holds wd.t ... g23d.t plus sizes.txt, e.g. made by `mdg run --dump`
(cli.py:145-152).
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2506_20994_b200 import ABI_CONTAINER_ORDER, expected_shape, load_kernel  # noqa: E402
from paper_2506_20994_b200.errors import CodegenError, ParseError, VersionError  # noqa: E402
from paper_2506_20994_b200.tensorfile import read_sizes, read_tensor, write_tensor  # noqa: E402

EXIT_OK, EXIT_MISMATCH, EXIT_USAGE, EXIT_MISSING_SYMBOL, EXIT_SHAPE_MISMATCH, EXIT_FORMAT_ERROR = 0, 1, 2, 3, 4, 5


def cmd_run(a) -> int:
    d = Path(a.inputs)
    try:
        nelv, lx = read_sizes(d / "sizes.txt")
        arrays = {n: np.ascontiguousarray(read_tensor(d / f"{n}.t")) for n in ABI_CONTAINER_ORDER}
    except (ParseError, VersionError, FileNotFoundError) as exc:
        print(exc, file=sys.stderr)
        return EXIT_FORMAT_ERROR
    for n in ABI_CONTAINER_ORDER:
        want = expected_shape(n, nelv, lx)
        if arrays[n].shape != want:
            print(f"{n}.t: dims {list(arrays[n].shape)} do not match sizes.txt "
                  f"(nelv={nelv}, lx={lx}), expected {list(want)}", file=sys.stderr)
            return EXIT_SHAPE_MISMATCH
    try:
        fn = load_kernel(a.lib, entry=a.entry, mode=a.mode)
    except CodegenError as exc:
        print(exc, file=sys.stderr)
        return EXIT_MISSING_SYMBOL
    fn(arrays, nelv, lx)
    write_tensor(a.o, arrays["wd"])
    return EXIT_OK


def cmd_compare(a) -> int:
    try:
        got, want = read_tensor(a.a), read_tensor(a.b)
    except (ParseError, VersionError, FileNotFoundError) as exc:
        print(exc, file=sys.stderr)
        return EXIT_FORMAT_ERROR
    if got.shape != want.shape:
        print(f"dims {list(got.shape)} vs {list(want.shape)}", file=sys.stderr)
        return EXIT_SHAPE_MISMATCH
    diff = float(np.max(np.abs(got - want))) if want.size else 0.0
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    rel = diff / scale if scale > 0 else diff
    print(f"max abs diff {diff!r}\nmax rel diff {rel!r}")
    if a.rtol is None:
        return EXIT_OK if diff == 0.0 else EXIT_MISMATCH
    return EXIT_OK if rel <= a.rtol else EXIT_MISMATCH


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="axrun")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--inputs", required=True)
    r.add_argument("-o", required=True)
    r.add_argument("--entry", default="__dace_ax_helm")
    r.add_argument("--lib", default=None)
    r.add_argument("--mode", choices=("strict", "fast"), default=None)
    c = sub.add_parser("compare")
    c.add_argument("-a", required=True)
    c.add_argument("-b", required=True)
    c.add_argument("--rtol", type=float, default=None)
    try:
        a = ap.parse_args(argv)
    except SystemExit as exc:
        return EXIT_USAGE if exc.code else EXIT_OK
    return cmd_run(a) if a.cmd == "run" else cmd_compare(a)


if __name__ == "__main__":
    sys.exit(main())
