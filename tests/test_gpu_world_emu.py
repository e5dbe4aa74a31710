"""Worlds 2, 3, 4, 6 and 8 on ONE GPU, bit for bit: all ranks in this process
(bo_world_init_local), one host thread per rank, every rank's kernels on one
shared stream in lockstep — the step's cross-rank waits become rendezvous of
the host threads between launches, so no kernel ever waits for another
(ranks must not spin on each other as separate launches on one device:
B200_PROFILING.md). The kernels, buffers, ring fold order, partials exchange
and parameter push are the multi-GPU path's own; only the barriers differ.
Checked against the oracle's emulation of the same world (oracle.train):
found_inf and the loss-scale sequence bit-exact, moments bit-exact (summed
over the ranks' shards), replicas identical, parameters within 1e-5."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _check(pipes, su, fi, ref, exact=True):
    from tests.harness import max_rel_or_abs

    world = len(pipes)
    assert fi.tolist() == ref.found_inf.tolist(), (fi, ref.found_inf)
    assert np.array_equal(su.view(np.uint32), ref.scale_used.view(np.uint32))
    P = pipes[0].P
    m = np.zeros(P, np.float32)
    v = np.zeros(P, np.float32)
    ws = []
    for p in pipes:
        mi, vi = p.read_moments()
        m += mi  # every element is owned by exactly one rank (the others read 0)
        v += vi
        ws.append(p.read_params())
        st = p.status()
        assert st.loss_scale == ref.final_scale and st.lamb_step == ref.lamb_step
    for w in ws[1:]:
        assert np.array_equal(w.view(np.uint32), ws[0].view(np.uint32))  # replicas identical
    if exact:
        assert np.array_equal(m.view(np.uint32), ref.m.view(np.uint32))
        assert np.array_equal(v.view(np.uint32), ref.v.view(np.uint32))
    assert max_rel_or_abs(ws[0], ref.params) <= TOL
    assert max_rel_or_abs(m, ref.m, 1e-12) <= TOL
    return ws[0]


CASES = {
    # name: (f16 wire, K, bucket bytes, scaler, spike ppm, resident, overlap)
    "ring16": (True, 2, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, False, None),
    "ring16_resident": (True, 2, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, True, None),
    "ring32_resident": (False, 3, 4096, dict(init_scale=1024.0), 0, True, None),
    "ring16_k4_resident": (True, 4, 1 << 20, dict(init_scale=4096.0), 0, True, None),
    "ring16_overlap": (True, 2, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, False, [1, 5, 2, 17]),
    # grouped speculative LAMB (push of group g overlapping phase 1 of g+1),
    # skipped steps included (the rollback path)
    "ring16_grouped": (True, 2, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, False, None),
    "ring16_grouped_resident": (True, 4, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, True, None),
    # the serial LAMB (one group) at every world size (the default below 4)
    "ring16_serial_resident": (True, 4, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, True, None),
}


# 3 and 6: non-power-of-two worlds, where the reference's 1/world scaling
# (trainer.cpp:212-213) is inexact and chunks are zero-padded to c * N
# (collective.hpp:44-60); the reference's own ring tests run N in {2,3,4,8}
# (test_collective.cpp:403-436)
@pytest.mark.parametrize("world", [2, 3, 4, 6, 8])
@pytest.mark.parametrize("case", sorted(CASES))
def test_world_lockstep_matches_oracle(torch_cuda, oracle, world, case, monkeypatch):
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import REDUCE_RING, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_world_lockstep

    f16, K, bb, sc, ppm, resident, overlap = CASES[case]
    if overlap:
        monkeypatch.setenv("BO_COMM_GROUP_ELEMS", "20000")  # several communication groups
    if "grouped" in case:
        monkeypatch.setenv("BO_LAMB_GROUP_ELEMS", "30000")  # ~6 LAMB groups of BERT_TINY
    if "serial" in case:
        monkeypatch.setenv("BO_LAMB_GROUP_ELEMS", "0")
    spec = bert_spec(BERT_TINY)
    P = spec.param_count()
    p0 = oracle.build_params(spec, 21)
    steps = 5
    inj = [(1, world - 1, K - 1, P // 3, 0x7C00), (3, 0, 0, 7, 0x7E00)] if ppm else []
    cfg = TrainerConfig(LambConfig(lr=5e-3), K, bb, f16, REDUCE_RING, ScalerConfig(**sc))
    pipes, su, fi = run_world_lockstep(spec, cfg, p0, world, steps, grad_seed=9, spike_ppm=ppm,
                                       spike_exp=3, injections=inj, resident=resident,
                                       overlap=overlap)
    ref = oracle.train(spec, p0, world, K, bb, f16, OL(lr=5e-3), OS(**sc), steps, grad_seed=9,
                       spike_ppm=ppm, spike_exp=3, injections=inj)
    _check(pipes, su, fi, ref)
    path = pipes[0].path()
    assert "ring_p2p" in path and "ring_push" in path
    # grouped LAMB: requested by the case; the default at world >= 4 unless
    # more than 10 % of the elements sit in phase-mismatched chunks
    if "grouped" in case:
        assert "lamb_grouped" in path
    if "serial" in case or (world < 4 and "grouped" not in case):
        assert "lamb_grouped" not in path
    assert ("resident_micros" in path) == resident
    assert ("overlap" in path) == bool(overlap)
    if ppm:
        assert 1 <= int(ref.found_inf.sum()) < steps
    for p in pipes:
        p.close()


@pytest.mark.slow
def test_world8_bert_large_full_size(torch_cuda, oracle):
    """The north star's 8-rank world at full size: BERT-large (336M), K = 4
    resident micros, binary16 ring, 2 steps, 8 ranks on one B200."""
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_LARGE, bert_spec
    from paper_2008_00177_b200.pipeline import REDUCE_RING, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_world_lockstep

    spec = bert_spec(BERT_LARGE)
    p0 = oracle.build_params(spec, 3)
    sc = dict(init_scale=2.0 ** 15)
    cfg = TrainerConfig(LambConfig(lr=1e-4), 4, 4 << 20, True, REDUCE_RING, ScalerConfig(**sc))
    pipes, su, fi = run_world_lockstep(spec, cfg, p0, 8, 2, grad_seed=5, resident=True)
    ref = oracle.train(spec, p0, 8, 4, 4 << 20, True, OL(lr=1e-4), OS(**sc), 2, grad_seed=5)
    _check(pipes, su, fi, ref)
    for p in pipes:
        p.close()
