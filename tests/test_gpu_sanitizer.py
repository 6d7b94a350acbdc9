"""compute-sanitizer memcheck + racecheck over every kernel path (TMA row-block
kernel with all row classes, warp-per-row, pack, exchange, unpack, combine)."""
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
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize run complete" in r.stdout
