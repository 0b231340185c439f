"""compute-sanitizer (memcheck, racecheck) over a small workload that runs
every kernel family once (tools/sanitize_run.py: the ax kernels for lx 3..16
in both modes, the three assembled-operator schedules with the fused dot,
DSSUM, PCG).  SURVEY §5: race detection / sanitizers."""

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer_clean(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(exe).exists():
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        str(ROOT / "tools" / "sanitize_run.py")],
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize workload done" in out
