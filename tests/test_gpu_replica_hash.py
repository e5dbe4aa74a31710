"""bo_replica_hash: the device-side replica hash behind the reference's
per-step divergence check (trainer.cpp:136-142 param_hash, checked across
ranks at trainer.cpp:442-453), against a numpy restatement of its
definition, on one rank and across the ranks of a lockstep world."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M1, M2, M3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _mix64(x):
    x = x + M1
    x = (x ^ (x >> np.uint64(30))) * M2
    x = (x ^ (x >> np.uint64(27))) * M3
    return x ^ (x >> np.uint64(31))


def replica_hash_np(spec, params):
    """sum mod 2^64 of mix64(mix64(t << 40 | i) ^ bits(w[t][i])) (bertopt_b200.h)."""
    h = np.uint64(0)
    off = 0
    with np.errstate(over="ignore"):
        for t, n in enumerate(spec.numels()):
            i = np.arange(n, dtype=np.uint64)
            key = (np.uint64(t) << np.uint64(40)) | i
            bits = np.asarray(params[off:off + n], np.float32).view(np.uint32).astype(np.uint64)
            h = h + np.sum(_mix64(_mix64(key) ^ bits), dtype=np.uint64)
            off += n
    return int(h)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_replica_hash_one_rank(torch_cuda, oracle):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 4)
    cfg = TrainerConfig(LambConfig(lr=1e-2), 2, 8192, False, 0, ScalerConfig(init_scale=1024.0))
    pipe, _, _ = run_pipeline(spec, cfg, p0, steps=2, resident=True)
    w = pipe.read_params()
    h = pipe.replica_hash()
    assert h == replica_hash_np(spec, w)
    assert h != replica_hash_np(spec, p0)  # the steps changed the parameters
    # one flipped low bit in one element changes it
    other = GradPipeline(spec, cfg)
    w2 = w.copy()
    w2.view(np.uint32)[len(w2) // 2] ^= 1
    other.load_params(w2)
    assert other.replica_hash() == replica_hash_np(spec, w2) != h
    other.load_params(w)
    assert other.replica_hash() == h  # same bits, other context
    pipe.close()
    other.close()


@pytest.mark.parametrize("world", [2, 4])
def test_replica_hash_equal_across_ranks(torch_cuda, oracle, world):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import REDUCE_RING, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_world_lockstep

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 6)
    cfg = TrainerConfig(LambConfig(lr=5e-3), 2, 8192, True, REDUCE_RING, ScalerConfig(init_scale=4096.0))
    pipes, _, _ = run_world_lockstep(spec, cfg, p0, world, 2, grad_seed=3, resident=True)
    hs = [p.replica_hash() for p in pipes]
    assert len(set(hs)) == 1
    assert hs[0] == replica_hash_np(spec, pipes[0].read_params())
    for p in pipes:
        p.close()
