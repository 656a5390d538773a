"""compute-sanitizer over every device kernel family (SURVEY.md section 5:
race detection / memory checking on the GPU box): memcheck and racecheck of
tools/sanitize_run.py (3D p = 1..4 x-line and work-item kernels, the x-line
diagonal, 2D, size-field targets, limiting, overlapped apply + fused
MINRES steps) must report no error and no shared-memory hazard."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not found")
    return exe


@pytest.mark.parametrize("tool", [["--tool", "memcheck", "--leak-check", "no"],
                                  ["--tool", "racecheck", "--racecheck-report", "hazard"]])
def test_sanitizer_clean(tool):
    env = dict(os.environ, TMOP_OVERLAP_MIN="0")
    r = subprocess.run([_sanitizer()] + tool + ["--error-exitcode", "9", sys.executable,
                                                os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize run ok" in out
    assert ("0 errors" in out) or ("0 hazards" in out), out[-2000:]
