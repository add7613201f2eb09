"""compute-sanitizer over small invocations of every kernel family (SURVEY.md
section 5: the kernels use named barriers, cp.async, bulk copies with
mbarriers and atomic tickets): memcheck, racecheck and synccheck must report
no errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(cuda, tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(REPO, "tools", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=REPO)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:  # the GPU pool's wrapper refuses sanitizer runs
        pytest.skip(out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case ok" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
