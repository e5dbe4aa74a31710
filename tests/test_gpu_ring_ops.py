"""The reference's collective API as operator drop-ins (SURVEY §8(a) a7/a8,
§8(b)): bo_ring_allreduce_f32 = ring_allreduce<float> (collective.hpp:53-99,
104-107) and bo_ring_allreduce_f16_wire = ring_allreduce_f16_wire
(collective.cpp:37-86, collective.hpp:113-114) on caller device data, over
the library's own NVLink ring (push form, no NCCL), bit for bit against the
oracle's ring — itself pinned to the compiled reference
(tests/test_oracle_vs_reference.py) — on every rank. Sizes: the reference's
ring tests (test_collective.cpp:403-436: n in {1, 5, 64, 1537}), a chunk
that is not a multiple of 4, and one larger than the ring staging buffers
(the chunks run in slices). Worlds 2, 3, 4 and 8 in lockstep on one GPU
(bo_world_init_local), and one process per GPU on a multi-GPU box."""
import json
import os
import socket
import subprocess
import sys
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SIZES = [1, 5, 64, 1537, 300001, 1 << 20]


def case_data(world, n, kind):
    """Per-rank inputs; for the binary16 wire, values whose sums stay in range."""
    rng = np.random.default_rng(1000 * world + n + kind)
    x = rng.standard_normal((world, n)).astype(np.float32)
    return x * np.float32(0.25 if kind else 1.0)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_ring_allreduce_operators_lockstep(torch_cuda, oracle, world):
    torch = torch_cuda
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import (REDUCE_RING, GradPipeline, LambConfig, ScalerConfig,
                                                TrainerConfig, ring_allreduce, ring_allreduce_f16_wire)

    spec = bert_spec(BERT_TINY)
    cfg = TrainerConfig(LambConfig(), 1, 16 << 10, True, REDUCE_RING, ScalerConfig())
    pipes = [GradPipeline(spec, cfg, device=0, rank=r, world=world) for r in range(world)]
    GradPipeline.world_init_local(pipes)
    # the largest size runs in slices: its chunk exceeds the staging buffers
    assert (SIZES[-1] + world - 1) // world > pipes[0].shard_elems() // 2
    try:
        for n in SIZES:
            for kind in (0, 1):
                data = case_data(world, n, kind)
                ref = oracle.ring_allreduce(data, kind)
                xs = [torch.from_numpy(data[r].copy()).cuda() for r in range(world)]
                op = ring_allreduce if kind == 0 else ring_allreduce_f16_wire
                errors = []

                def rank_thread(r):
                    try:
                        torch.cuda.set_device(0)
                        op(pipes[r], xs[r])
                    except BaseException as e:  # noqa: BLE001
                        errors.append(e)

                threads = [threading.Thread(target=rank_thread, args=(r,)) for r in range(world)]
                for t in threads:
                    t.start()
                for t in threads:
                    t.join()
                assert not errors, errors
                for r in range(world):
                    got = xs[r].cpu().numpy()
                    assert np.array_equal(got.view(np.uint32), ref[r].view(np.uint32)), (n, kind, r)
                assert np.array_equal(ref[0], ref[-1])  # identical on every rank
    finally:
        for p in pipes:
            p.close()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.multigpu
@pytest.mark.parametrize("n", [2, 3, 4])
def test_ring_allreduce_operators_one_process_per_gpu(torch_cuda, n):
    if torch_cuda.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs (one per rank); the lockstep test covers one GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "ring_ops_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and len(lines) == n, r.stdout[-3000:] + r.stderr[-3000:]
    assert all(x["ok"] for x in lines), lines
