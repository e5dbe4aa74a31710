"""The step's event timeline in the reference's EventLog schema
(trainer.cpp:43-71: {"ts","rank","event","bytes"} JSON lines; events
trainer.hpp:30-35), device-timed: bo_trace_enable / bo_trace_write."""
import json
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LINE = re.compile(r'^\{"ts":\d+\.\d{9},"rank":\d+,"event":"[a-z_]+","bytes":\d+\}$')


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _read(path):
    lines = open(path).read().splitlines()
    assert lines and all(LINE.match(ln) for ln in lines), lines[:3]
    evs = [json.loads(ln) for ln in lines]
    ts = [e["ts"] for e in evs]
    assert ts == sorted(ts) and ts[0] >= 0.0
    return evs


def test_trace_one_rank(torch_cuda, oracle, tmp_path):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    K = 2
    cfg = TrainerConfig(LambConfig(), K, 8192, False, 0, ScalerConfig(init_scale=1024.0))
    pipe = GradPipeline(spec, cfg)
    pipe.load_params(oracle.build_params(spec, 3))
    pipe.trace_enable()
    run_pipeline(spec, cfg, None, 2, pipe=pipe)                             # per-micro API
    run_pipeline(spec, cfg, None, 1, pipe=pipe, first_step=2, resident=True)  # bo_train_step
    path = str(tmp_path / "events.jsonl")
    pipe.trace_write(path)
    evs = _read(path)
    names = [e["event"] for e in evs]
    assert names.count("micro_ready") == 3 * K and names.count("step_end") == 3
    assert names.count("lamb_start") == 3
    assert all(e["rank"] == 0 for e in evs)
    P = spec.param_count()
    assert all(e["bytes"] == 2 * P for e in evs if e["event"] == "micro_ready")
    # per step: its micros, then LAMB, then the end
    order = [n for n in names if n in ("micro_ready", "lamb_start", "step_end")]
    assert order == (["micro_ready"] * K + ["lamb_start", "step_end"]) * 3
    pipe.trace_enable(False)
    pipe.close()


def test_trace_world_lockstep_with_overlap(torch_cuda, oracle, tmp_path, monkeypatch):
    """World 2 (lockstep on one GPU), the sync micro delivered bucket by
    bucket: bucket_ready per communication group, then that group's
    comm_start / comm_end with the bytes this rank sends."""
    import threading

    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import (REDUCE_RING, GradPipeline, LambConfig, ScalerConfig,
                                                TrainerConfig)
    from tests.harness import run_pipeline

    monkeypatch.setenv("BO_COMM_GROUP_ELEMS", "20000")
    spec = bert_spec(BERT_TINY)
    cfg = TrainerConfig(LambConfig(), 2, 8192, True, REDUCE_RING, ScalerConfig(init_scale=1024.0))
    p0 = oracle.build_params(spec, 3)
    pipes = [GradPipeline(spec, cfg, rank=r, world=2) for r in range(2)]
    for p in pipes:
        p.load_params(p0)
    GradPipeline.world_init_local(pipes)
    for p in pipes:
        p.trace_enable()
    errs = []

    def rank(r):
        try:
            run_pipeline(spec, cfg, None, 2, rank=r, world=2, pipe=pipes[r], overlap=[3, 7])
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r, p in enumerate(pipes):
        path = str(tmp_path / f"events{r}.jsonl")
        p.trace_write(path)
        evs = _read(path)
        assert all(e["rank"] == r for e in evs)
        names = [e["event"] for e in evs]
        groups = names.count("bucket_ready")
        assert groups >= 2 * 2  # several communication groups per step, 2 steps
        assert names.count("comm_start") == groups and names.count("comm_end") == groups
        sent = sum(e["bytes"] for e in evs if e["event"] == "comm_start")
        # binary16 wire: (N - 1) hops of one chunk of every bucket per step
        _, _, _, be = p.layout()
        chunk = np.ceil(np.asarray(be, np.int64) / 2).astype(np.int64).sum()
        assert sent == 2 * (1 * chunk * 2)
    for p in pipes:
        p.close()
