"""The C++ adapter over the C ABI, compiled against the reference's headers and
objects (oracle/_ref/adapter_test), run next to the reference's own
lamb_step / unscale_gradients / DistributedTrainer::train_step and — for
worlds 2, 3 and 4 in lockstep on one GPU — the reference's own
ring_allreduce<float> / ring_allreduce_f16_wire over InProcHub, on the same
inputs (bits equal on every rank)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


def test_cpp_adapter_against_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("adapter_test not built (needs the reference sources at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ADAPTER OK" in r.stdout, r.stdout + r.stderr
