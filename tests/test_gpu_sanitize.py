"""compute-sanitizer memcheck over small runs of the benchmark paths (``-m gpu``).

The full sweep (memcheck, racecheck, synccheck on reduced c2 / c3 / c4) is
``tools/sanitize.sh``; its logs are summarised in ``profiles/``.  This test
keeps the two paths that had a finding in round 1 under memcheck on every
GPU test run.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("args", [["c3small", "--queries", "24", "--graphs", "1200"], ["c2", "--graphs", "40"]])
def test_memcheck_clean(gpu, args):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not present")
    r = subprocess.run([CS, "--tool", "memcheck", "--error-exitcode", "99", "--print-limit", "20", sys.executable,
                        str(REPO / "tools" / "sanitize_run.py"), *args], capture_output=True, text=True, timeout=900,
                       cwd=REPO)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr
