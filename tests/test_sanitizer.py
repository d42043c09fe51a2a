"""compute-sanitizer tier (SURVEY.md sections 4-5): the library's kernels under
memcheck / racecheck / synccheck / initcheck on small workloads
(scripts/sanitize_workload.py).  One tool per process, selected by
RBM_SANITIZER=<tool> (the tools are run one per GPU call: several tools in one
call have hung GPUs of this pool); skipped otherwise, so neither the CPU suite
nor the default -m gpu suite runs them.  Logs: profiles/r2_sanitizer_<tool>.log.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.environ.get("RBM_SANITIZER", "")


@pytest.mark.sanitizer
@pytest.mark.skipif(TOOL not in ("memcheck", "racecheck", "synccheck", "initcheck"),
                    reason="set RBM_SANITIZER=memcheck|racecheck|synccheck|initcheck (one tool per run)")
def test_kernels_clean_under_sanitizer():
    cmd = ["compute-sanitizer", "--tool", TOOL, "--error-exitcode", "9", "--print-limit", "50",
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_workload.py")]
    if TOOL == "racecheck":
        cmd[3:3] = ["--racecheck-report", "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    log = r.stdout + r.stderr
    if "closed on this pool" in log:
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + log.strip()[:200])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{TOOL}.log"), "w") as f:
        f.write(log)
    assert r.returncode == 0, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]
    assert "sanitize workload done" in log
