"""compute-sanitizer over small anneals of every kernel family (SMEM tier with and without
speculation, HBM tier, both von Neumann solvers): no memory errors, no shared-memory races,
no barrier misuse. GPU only; ~20 s per tool."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("tool,clean", [("memcheck", "ERROR SUMMARY: 0 errors"),
                                        ("racecheck", "RACECHECK SUMMARY: 0 hazards"),
                                        ("synccheck", "ERROR SUMMARY: 0 errors")])
def test_compute_sanitizer(tool, clean):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    out = subprocess.run([exe, "--tool", tool, "--print-limit", "10", sys.executable,
                          os.path.join(ROOT, "tools", "sanitizer_run.py")],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-2000:]
    assert clean in text, text[-2000:]
