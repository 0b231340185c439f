"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/axhelm.h declares, the operator API validates its
arguments exactly like the reference's kernelrt (kernelrt.py:98-104,
tests/test_codegen.py:189-214), the product GLL basis is bit-exact with the
reference, and the MDGT format matches the reference's golden bytes."""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as o
from paper_2506_20994_b200 import (
    ABI_CONTAINER_ORDER, BindingError, CodegenError, RangeError, gll_basis, load_kernel,
)
from paper_2506_20994_b200 import _lib, tensorfile

ROOT = Path(__file__).resolve().parents[1]
HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared_functions():
    names = []
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if n not in {"if", "while", "defined"}))


def test_header_declares_reference_signature():
    text = (ROOT / "include" / "axhelm.h").read_text()
    sig = re.search(r"void __dace_ax_helm\((.*?)\);", text, flags=re.S).group(1)
    params = re.findall(r"(\w+)\s*(?:,|$)", " ".join(sig.split()))
    assert tuple(params[:15]) == ABI_CONTAINER_ORDER  # codegen.py:183-194
    assert params[15:] == ["nelv", "lx"]
    assert "int nelv" in sig and "int lx" in sig
    assert sig.count("const double*") == 14  # only wd is mutable (test_codegen.py:64-67)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.lib_path()))
    names = declared_functions()
    assert "__dace_ax_helm" in names and "axhelm_apply" in names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/ but not exported"
    for n in _lib.PROTOTYPES:
        assert n in names, f"{n} bound in _lib but not declared in include/"


def test_models_and_version_without_gpu():
    lib = _lib.load()
    assert lib.axhelm_bytes_model(262144, 8) == 9_663_676_416
    assert lib.axhelm_flops_model(32768, 8) == 1_912_602_624  # test_oracle.py:245
    assert lib.axhelm_flops_model(1, 2) == 336
    assert b"sm_100a" in lib.axhelm_version()
    assert lib.axhelm_get_mode() in (0, 1)


def _arrays(lx=4, nel=2):
    a = o.problem(lx, nel)
    return {k: np.ascontiguousarray(v) for k, v in a.items()}


class TestBindingErrors:
    """Mirrors tests/test_codegen.py:189-214 of the reference."""

    def test_rejects_f32(self):
        fn = load_kernel()
        a = _arrays()
        a["ud"] = a["ud"].astype(np.float32)
        with pytest.raises(BindingError, match="ud"):
            fn(a, 2, 4)

    def test_rejects_non_contiguous(self):
        fn = load_kernel()
        a = _arrays()
        a["ud"] = np.asfortranarray(a["ud"])
        with pytest.raises(BindingError, match="contiguous"):
            fn(a, 2, 4)

    def test_rejects_missing(self):
        fn = load_kernel()
        a = _arrays()
        del a["g23d"]
        with pytest.raises(BindingError, match="g23d"):
            fn(a, 2, 4)

    def test_rejects_wrong_shape(self):
        fn = load_kernel()
        a = _arrays()
        with pytest.raises(BindingError, match="h1d"):
            a["h1d"] = a["h1d"][:1].copy()
            fn(a, 2, 4)

    def test_missing_symbol(self):
        with pytest.raises(CodegenError, match="zz_nope"):
            load_kernel(entry="zz_nope")

    def test_missing_library(self, tmp_path):
        with pytest.raises(CodegenError):
            load_kernel(tmp_path / "nope.so")

    def test_bad_mode(self):
        with pytest.raises(RangeError):
            load_kernel(mode="turbo")


def test_product_basis_bit_exact(golden_dir):
    ref = json.loads((golden_dir / "gll.json").read_text())
    for lx in range(2, 17):
        b = gll_basis(lx)
        assert [v.hex() for v in b.points] == ref[str(lx)]["points"]
        assert [v.hex() for v in b.weights] == ref[str(lx)]["weights"]
        assert [[v.hex() for v in r] for r in b.deriv] == ref[str(lx)]["deriv"]
    with pytest.raises(RangeError):
        gll_basis(17)


def test_tensorfile_golden_and_roundtrip(golden_dir, tmp_path):
    blob = (golden_dir / "mdgt_2x2.t").read_bytes()
    p = tmp_path / "g.t"
    tensorfile.write_tensor(p, np.array([[1.0, 2.0], [3.0, -0.5]]))
    assert p.read_bytes() == blob
    assert np.array_equal(tensorfile.read_tensor(p), [[1.0, 2.0], [3.0, -0.5]])
    from paper_2506_20994_b200.errors import ParseError, VersionError

    bad = tmp_path / "b.t"
    bad.write_bytes(b"NOPE" + blob[4:])
    with pytest.raises(ParseError):
        tensorfile.read_tensor(bad)
    v = bytearray(blob)
    v[4] = 9
    bad.write_bytes(bytes(v))
    with pytest.raises(VersionError):
        tensorfile.read_tensor(bad)
    bad.write_bytes(blob[:-8])
    with pytest.raises(ParseError, match="3 of 4"):
        tensorfile.read_tensor(bad)
    # a scalar is written as rank 1 (the reference's np.ascontiguousarray promotes 0-d)
    tensorfile.write_tensor(p, np.float64(2.5))
    assert p.read_bytes()[4:6] == bytes([1, 1]) and tensorfile.read_tensor(p).shape == (1,)
    s = tmp_path / "sizes.txt"
    tensorfile.write_sizes(s, 64, 8)
    assert s.read_text() == "64 8\n" and tensorfile.read_sizes(s) == (64, 8)


def test_product_never_imports_oracle():
    """The product package must not reference oracle/ (no CPU fallback)."""
    pkg = ROOT / "paper_2506_20994_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "liboracle" not in text and "oracle/_ref" not in text, f
