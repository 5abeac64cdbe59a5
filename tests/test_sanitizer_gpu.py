"""compute-sanitizer memcheck and racecheck over every kernel family
(tools/sanitize_case.py): out-of-bounds / misaligned global accesses,
and shared-memory hazards in the per-warp flux scratch, the staged tables
and the in-place RK update (complements the static race
certificate, sweeps.py:89-105)."""

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer(cuda, tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(exe).exists():
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "99", sys.executable,
                        str(ROOT / "tools" / "sanitize_case.py")],
                       capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case ok" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
