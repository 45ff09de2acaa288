"""compute-sanitizer tiers: memcheck, racecheck, synccheck and initcheck over every kernel
variant on tiny ragged inputs (scripts/sanitize_check.py) report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_check.py")],
                       capture_output=True, text=True, timeout=540, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-3000:]
    if r.returncode != 0 and "compute-sanitizer is closed" in tail:
        # the GPU pool disables the tool (a wrapper refuses it); the committed sanitizer runs
        # of the round are profiles/r01_sanitizers.txt and profiles/r02_sanitizers.txt
        pytest.skip("compute-sanitizer disabled on this GPU pool: " + tail.strip().splitlines()[-1][:200])
    assert r.returncode == 0, tail
    assert "sanitize_check ok" in r.stdout, tail
