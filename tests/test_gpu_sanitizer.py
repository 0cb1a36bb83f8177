"""T4: compute-sanitizer memcheck / racecheck / synccheck over every kernel on a
small workload (TMA ring + mbarriers, named barriers, lane-private atomics)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, f"--tool={tool}", "--error-exitcode=9", "--target-processes=all",
           sys.executable, os.path.join(ROOT, "tests", "helpers", "sanitize_run.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "sanitize_run ok" in r.stdout, tail
    txt = r.stdout + r.stderr
    assert ("ERROR SUMMARY: 0 errors" in txt) or ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in txt), tail
