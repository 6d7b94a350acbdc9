"""compute-sanitizer memcheck + racecheck over every kernel path (TMA row-block
kernel with all row classes, warp-per-row, pack, exchange, unpack, combine).

The GPU pool can close compute-sanitizer (it then exits 86 with a notice and
never starts the program); the test is skipped in that case, and the
round-1/2 clean runs stay in profiles/r*_compute_sanitizer.txt."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    r = subprocess.run(["compute-sanitizer", "--tool", tool, "--error-exitcode", "9",
                        sys.executable, os.path.join(ROOT, "scripts", "sanitize.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    if r.returncode == 86 and "compute-sanitizer is closed" in (r.stdout + r.stderr):
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize run complete" in r.stdout
