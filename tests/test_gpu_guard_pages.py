"""Bounds check of the product kernels without compute-sanitizer (closed on
this pool): tools/guard_pages.py places every caller-owned tensor so that it
ends at the end of a mapped 2 MiB granule followed by an UNMAPPED one, runs
both step APIs (aligned and unaligned gradient slots) and the operator
drop-ins, and must finish without a fault (a load or store past a tensor's
end into the guard granule would raise an illegal-address error)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_pages_clean():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pytest.importorskip("cuda.bindings.driver")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_pages.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "GUARD_PAGES_OK" in out, out[-4000:]
