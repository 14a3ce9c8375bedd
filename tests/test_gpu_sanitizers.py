"""compute-sanitizer over every product kernel on small ragged problems (scripts/sanitize.py: norms,
pyramid, skip map, order kernels, BF16 dual multiply, FP32 SIMT, FP32X3, the two-rank emulation,
per-C-tile list expansion): memcheck, racecheck and synccheck must report no error (SURVEY.md 5,
sanitizers row).  Each run also checks its results against the float64 oracle."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    out = subprocess.run([SAN, "--tool", tool, "--print-limit", "20", sys.executable,
                          os.path.join(ROOT, "scripts", "sanitize.py")], capture_output=True, text=True, timeout=1200)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    summary = re.findall(r"(ERROR SUMMARY|RACECHECK SUMMARY): (\d+) (error|hazard)", log)
    assert summary, log[-3000:]
    assert all(int(n) == 0 for _, n, _ in summary), log[-3000:]
