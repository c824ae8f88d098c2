"""compute-sanitizer over every kernel family:
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards) and synccheck (barrier misuse) on tools/sanitize_driver.py — each
corpus kernel, bitonic / PCM / MS sorts in every form and shape, NQU, LUD,
SRAD (IEEE and fast) and the GPU interpreter at small sizes."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-6000:]
    assert "sanitize driver ok" in out
    # memcheck / synccheck end with "ERROR SUMMARY: 0 errors", racecheck with
    # "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" \
        else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-3000:]
