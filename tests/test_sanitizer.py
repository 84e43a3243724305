"""compute-sanitizer over small anneals of every kernel family (SMEM tier with and without
speculation, HBM tier on both schedules, all von Neumann solvers, the batched GEMM's
variants): no memory errors, no barrier misuse, no shared-memory races other than the work
queue's mbarrier-ordered metadata handoff (which racecheck cannot see). GPU only."""
import os
import re
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
    limit = "100000" if tool == "racecheck" else "10"  # racecheck: every report is inspected below
    out = subprocess.run([exe, "--tool", tool, "--print-limit", limit, sys.executable,
                          os.path.join(ROOT, "tools", "sanitizer_run.py")],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:
        # the GPU pool's compute-sanitizer wrapper refuses every run (it has left GPUs needing a
        # reset elsewhere); earlier clean runs of this test are described in DESIGN.md §4
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    if tool == "racecheck":
        # The work queue's stage metadata is written by the producer and read by the consumers
        # across an mbarrier (arrive = release, try_wait = acquire); racecheck does not model
        # mbarrier ordering and reports exactly that pair. Any other hazard fails.
        blocks = re.findall(r"Error: Race reported between (\w+) access at (.*?)\n=+\s+and (\w+) access at (.*?)\n",
                            text)
        assert len(blocks) == text.count("Error: Race reported"), text[-3000:]  # every report parsed
        other = [b for b in blocks if "put_meta" not in b[1] and "put_meta" not in b[3]]
        assert not other, other[:5]
        assert "RACECHECK SUMMARY" in text, text[-2000:]
        assert out.returncode in (0, 1), text[-2000:]  # 1: the accepted reports above
        assert "12 renyi-2" in text and "queue 16 von-neumann" in text, text[-2000:]  # every family ran
        return
    assert out.returncode == 0, text[-2000:]
    assert clean in text, text[-2000:]
