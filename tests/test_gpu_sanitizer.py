"""compute-sanitizer over the pass kernels.

One tool per GPU call: B200_PROFILING.md reports that several
compute-sanitizer tools in one call have left a B200 unusable until a reset,
so this test only runs when LATTDSE_SANITIZE names ONE tool

    LATTDSE_SANITIZE=racecheck python -m pytest tests/test_gpu_sanitizer.py -m gpu -q

(scripts/sanitize.sh runs it under gpurun, one call per tool) and is skipped
in the plain `-m gpu` run. Round 2: the pool's wrapper answers
"compute-sanitizer is closed on this pool" (profiles/r2/sanitizer_closed.log),
so the race evidence of this round is tests/test_gpu_pass4.py instead: the
lean kernels against the generic ones, and bit-identical repeated runs.
"""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
TOOL = os.environ.get("LATTDSE_SANITIZE", "")


@pytest.mark.gpu
@pytest.mark.skipif(TOOL not in ("memcheck", "racecheck", "synccheck", "initcheck"),
                    reason="set LATTDSE_SANITIZE to one compute-sanitizer tool (one tool per GPU call)")
def test_compute_sanitizer_one_tool():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    out = subprocess.run([exe, "--tool", TOOL, "--error-exitcode", "9", "--print-limit", "20", sys.executable,
                          os.path.join(ROOT, "tests", "sanitize_case.py"), "--quick"],
                         capture_output=True, text=True, timeout=3000)
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{TOOL}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as f:
        f.write(out.stdout[-20000:] + "\n--- stderr ---\n" + out.stderr[-5000:] + f"\nrc={out.returncode}\n")
    if "closed on this pool" in out.stderr or "closed on this pool" in out.stdout:
        pytest.skip("compute-sanitizer is closed on this GPU pool (the box's wrapper refuses to run it)")
    assert out.returncode == 0, out.stdout[-3000:]
    assert "sanitize_case: ok" in out.stdout
    assert "ERROR SUMMARY: 0 errors" in out.stdout or "RACECHECK SUMMARY: 0 hazards" in out.stdout, out.stdout[-2000:]
