"""World-size-2 host-side logic of the N>1 path on CPU (gloo over 127.0.0.1):
NCCL-id exchange, bucket-layout agreement (BucketLayoutMismatch), shard
ownership, the ring's fold order across ranks, and the bench's reference arm
under torchrun."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, ("error", type(e).__name__, str(e))))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _exchange_id(rank, world):
    from paper_2008_00177_b200.pipeline import broadcast_unique_id

    return broadcast_unique_id(0)


def _layout_agree(rank, world):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import BucketLayout, agree_layout

    spec = bert_spec(BERT_TINY)
    L = BucketLayout.build(spec, 4096, True, 2)
    agree_layout(L.hash)  # same config: passes
    bb = 4096 if rank == 0 else 256  # trainer test "different bucket thresholds"
    agree_layout(BucketLayout.build(spec, bb, True, 2).hash)
    return "no error"


def _layout_wire_mismatch(rank, world):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import BucketLayout, agree_layout

    agree_layout(BucketLayout.build(bert_spec(BERT_TINY), 4096, rank == 1, 1).hash)
    return "no error"


def _shard_cover(rank, world):
    import torch
    import torch.distributed as dist

    from paper_2008_00177_b200.model_spec import BERT_BASE, bert_spec
    from paper_2008_00177_b200.pipeline import BucketLayout

    L = BucketLayout.build(bert_spec(BERT_BASE), 4 << 20)
    lo, hi = L.shard_ranges(world, rank)
    mine = torch.from_numpy(np.stack([lo, hi]))
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    owned = sum(int((a[1] - a[0]).sum()) for a in allr)
    return owned == int(L.bucket_elems.sum())


def _ring_fold(rank, world):
    """Each rank holds its own vector; the emulated ring (oracle) gives every
    rank the same bits, and the fold for chunk k starts at rank k."""
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle

    n = 1537
    rng = np.random.default_rng(rank)
    mine = torch.from_numpy(rng.uniform(-2, 2, n).astype(np.float32))
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    data = torch.stack(allv).numpy()
    o = Oracle()
    res = o.ring_allreduce(data, 1)[rank]
    c = -(-n // world)
    k = 0
    p = data[k, :c].copy()
    for j in range(1, world):
        p = o.f16_to_f32(o.f32_to_f16(p)) + data[(k + j) % world, :c]
    p = o.f16_to_f32(o.f32_to_f16(p))
    return bool(np.array_equal(res[:c], p)), res.tobytes()


def test_nccl_id_broadcast():
    try:
        ids = run_world(_exchange_id)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"spawn unavailable: {e}")
    if isinstance(ids[0], tuple):
        pytest.skip(f"ncclGetUniqueId unavailable here: {ids[0]}")
    assert len(ids[0]) == 128 and ids[0] == ids[1]


def test_layout_mismatch_detected():
    out = run_world(_layout_agree)
    assert all(o[0] == "error" and o[1] == "BucketLayoutMismatch" for o in out)
    out = run_world(_layout_wire_mismatch)
    assert all(o[0] == "error" and o[1] == "BucketLayoutMismatch" for o in out)


def test_shard_ownership_partitions_buckets():
    assert run_world(_shard_cover) == [True, True]
    assert run_world(_shard_cover, world=3) == [True, True, True]


def test_ring_identical_on_every_rank():
    out = run_world(_ring_fold)
    assert out[0][0] and out[1][0] and out[0][1] == out[1][1]


def test_bench_reference_arm_under_torchrun():
    """bench.py --impl reference: rank 0 prints one JSON line, rank 1 exits 0."""
    from oracle.oracle import reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--model", "bert-tiny"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
