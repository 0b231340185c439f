"""The operator API raises the reference's own exception classes.

A caller written against mdg catches ``mdg.errors.BindingError`` /
``CodegenError`` (/root/reference/pkg/src/mdg/kernelrt.py:85-104); with mdg
importable, this package's errors ARE those classes (errors.py).  Runs in a
subprocess so mdg is on sys.path before the package is first imported.  No
kernel is launched: every failure here is raised before the C call.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")

CHECK = r'''
import numpy as np, pytest
import mdg.errors
from paper_2506_20994_b200 import errors, load_kernel, RangeError
assert errors.FROM_REFERENCE and errors.BindingError is mdg.errors.BindingError
lx, nel = 4, 3
arrays = {n: np.zeros((lx, lx)) if n[:2] in ("dx", "dy", "dz") else np.zeros((nel, lx, lx, lx))
          for n in ("wd", "ud", "dxd", "dyd", "dzd", "dxtd", "dytd", "dztd", "h1d", "g11d", "g22d",
                    "g33d", "g12d", "g13d", "g23d")}
fn = load_kernel()
with pytest.raises(mdg.errors.BindingError, match="g23d"):
    fn({k: v for k, v in arrays.items() if k != "g23d"}, nel, lx)
with pytest.raises(mdg.errors.BindingError, match="h1d"):
    fn({**arrays, "h1d": arrays["h1d"].astype(np.float32)}, nel, lx)
with pytest.raises(mdg.errors.BindingError, match="ud"):
    fn({**arrays, "ud": arrays["ud"][..., ::-1]}, nel, lx)  # not C-contiguous
with pytest.raises(mdg.errors.CodegenError):
    load_kernel(entry="__no_such_symbol")
with pytest.raises(mdg.errors.RangeError):
    load_kernel(mode="approximate")
assert issubclass(errors.DeviceError, mdg.errors.MdgError)
print("ok")
'''


@pytest.mark.skipif(not REF.exists(), reason="reference sources not present (GPU box)")
def test_reference_exception_classes_are_raised():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT), str(REF)]))
    out = subprocess.run([sys.executable, "-c", CHECK], env=env, capture_output=True, text=True,
                         timeout=300, cwd=str(ROOT))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_local_classes_without_reference():
    """Without mdg the package still raises classes with the reference's names and bases."""
    code = ("import sys; sys.modules['mdg'] = None\n"
            "from paper_2506_20994_b200 import errors\n"
            "assert not errors.FROM_REFERENCE\n"
            "assert issubclass(errors.BindingError, ValueError) and issubclass(errors.BindingError, errors.MdgError)\n"
            "print('ok')")
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
