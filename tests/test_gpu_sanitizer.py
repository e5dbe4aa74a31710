"""compute-sanitizer over the product kernels: memcheck
(out-of-bounds / misaligned global accesses — every gradient tensor ends at
the end of its own allocation, so a load past a tensor's last element is
caught), racecheck (shared-memory hazards) and synccheck (barrier misuse),
through both step APIs, aligned and unaligned slots, and the operator
drop-ins (tools/sanitize_step.py).

Opt-in: BO_SANITIZER_TOOLS=memcheck (comma list). B200_PROFILING.md reports
that several compute-sanitizer tools in one GPU session once left a B200
unusable until a reset, so the default `-m gpu` run does not start the tool;
each tool is run in its own GPU session and its report kept under profiles/
(profiles/r02_sanitizer_*.txt)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not installed")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    wanted = [t for t in os.environ.get("BO_SANITIZER_TOOLS", "").split(",") if t]
    if tool not in wanted:
        pytest.skip("opt-in: BO_SANITIZER_TOOLS=" + tool + " (one tool per GPU session)")
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_step.py")]
    if tool == "memcheck":
        cmd[1:1] = ["--leak-check", "no"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    log = os.environ.get("BO_SANITIZER_LOG")
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd[:-2] + ["python", "tools/sanitize_step.py"]) + "\n" + out)
    assert r.returncode == 0, out[-6000:]
    assert "SANITIZE_STEP_OK" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
