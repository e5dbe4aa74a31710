"""GPU parity of the single-rank pipeline against the CPU oracle.

Contract (BASELINE.json north_star): overflow flags, skipped steps and the
loss-scale sequence bit-exact; parameters and LAMB moments within 1e-5
relative after N steps. In practice the moments are bit-exact (their math has
no reduction) and parameters differ at most by the ulp an fp64 norm summed in
a different order can move the trust ratio.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5  # north-star tolerance for fp32 parameter / moment state


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _compare(pipe, ref, scale_used, found, exact_moments=True):
    from tests.harness import max_rel_or_abs

    assert np.array_equal(found, ref.found_inf), (found, ref.found_inf)
    assert np.array_equal(scale_used.view(np.uint32), ref.scale_used.view(np.uint32))
    st = pipe.status()
    assert st.loss_scale == ref.final_scale
    assert st.lamb_step == ref.lamb_step
    assert st.skipped_steps == int(ref.found_inf.sum())
    w = pipe.read_params()
    m, v = pipe.read_moments()
    assert max_rel_or_abs(w, ref.params) <= TOL
    if exact_moments:
        assert np.array_equal(m.view(np.uint32), ref.m.view(np.uint32))
        assert np.array_equal(v.view(np.uint32), ref.v.view(np.uint32))
    else:
        assert max_rel_or_abs(m, ref.m, 1e-12) <= TOL
        assert max_rel_or_abs(v, ref.v, 1e-20) <= TOL
    return w


@pytest.mark.parametrize("K", [1, 3, 4])
@pytest.mark.parametrize("aligned", [True, False])
def test_tiny_bert_matches_oracle(torch_cuda, oracle, K, aligned):
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 7)
    cfg = TrainerConfig(LambConfig(), K, 8192, False, 0, ScalerConfig(init_scale=4096.0))
    pipe, su, fi = run_pipeline(spec, cfg, p0, steps=4, aligned=aligned)
    ref = oracle.train(spec, p0, 1, K, 8192, False, OL(), OS(init_scale=4096.0), 4)
    w = _compare(pipe, ref, su, fi)
    # bit-exact in practice; record how close
    assert np.mean(w.view(np.uint32) == ref.params.view(np.uint32)) > 0.999
    # 16-byte aligned gradient slots take the fused one-rank kernels
    assert pipe.path() == (["one_rank_fused"] if aligned else ["one_rank_staged"])


@pytest.mark.parametrize("resident", [False, True])
def test_empty_and_ragged_tensors_match_oracle(torch_cuda, oracle, resident):
    """Zero-element and ragged tensors (sizes 0, 1, primes, one past a tile)
    through both step APIs, overflow injected: scale sequence and moments
    bit-exact, params within the north-star tolerance."""
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import flat_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = flat_spec([0, 5, 4097, 0, 3, 1, 8191], first_use=[2, 0, 1, 4, 3, 6, 5])
    P = spec.param_count()
    p0 = oracle.build_params(spec, 5)
    inj = [(1, 0, 2, P - 1, 0x7C00)]
    cfg = TrainerConfig(LambConfig(), 3, 4096, False, 0, ScalerConfig(init_scale=4096.0, growth_interval=2))
    pipe, su, fi = run_pipeline(spec, cfg, p0, steps=4, injections=inj, resident=resident)
    ref = oracle.train(spec, p0, 1, 3, 4096, False, OL(), OS(init_scale=4096.0, growth_interval=2), 4,
                       injections=inj)
    _compare(pipe, ref, su, fi)
    assert fi.tolist() == [0, 1, 0, 0]
    assert ("resident_micros" in pipe.path()) == resident


@pytest.mark.parametrize("resident", [False, True])
def test_dynamic_scaler_overflow_sequence(torch_cuda, oracle, resident):
    """Config 4 at desk scale: injected inf/NaN plus natural spikes, growth
    every 4, 24 steps, through the per-micro API and bo_train_step."""
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    P = spec.param_count()
    p0 = oracle.build_params(spec, 3)
    sc = dict(init_scale=2.0 ** 14, growth_interval=4, min_scale=1.0, max_scale=2.0 ** 20)
    inj = [(2, 0, 1, 17, 0x7C00), (5, 0, 0, P - 1, 0xFC00), (9, 0, 2, 12345, 0x7E00),
           (9, 0, 0, 5, 0x7C00)]
    cfg = TrainerConfig(LambConfig(lr=1e-2), 3, 4096, False, 0, ScalerConfig(**sc))
    # spike exponent 3: |g| = 8..16, overflows binary16 whenever S >= 2^13
    pipe, su, fi = run_pipeline(spec, cfg, p0, steps=24, spike_ppm=3, spike_exp=3,
                                injections=inj, resident=resident)
    assert ("resident_micros" in pipe.path()) == resident
    ref = oracle.train(spec, p0, 1, 3, 4096, False, OL(lr=1e-2), OS(**sc), 24, spike_ppm=3,
                       spike_exp=3, injections=inj)
    assert ref.found_inf.sum() >= 4 and ref.found_inf.sum() < 20
    assert len(set(ref.scale_used.tolist())) >= 3  # backoff and growth both exercised
    _compare(pipe, ref, su, fi)


def test_skipped_step_leaves_state_untouched(torch_cuda, oracle):
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 5)
    cfg = TrainerConfig(LambConfig(), 2, 1 << 20, False, 0, ScalerConfig(init_scale=1024.0))
    pipe, _, _ = run_pipeline(spec, cfg, p0, steps=2)
    w_before = pipe.read_params()
    m_before, v_before = pipe.read_moments()
    st0 = pipe.status()
    pipe, su, fi = run_pipeline(spec, cfg, None, steps=1, injections=[(0, 0, 1, 3, 0x7E00)],
                                pipe=pipe)
    assert fi.tolist() == [1]
    st1 = pipe.status()
    assert st1.lamb_step == st0.lamb_step and st1.skipped_steps == st0.skipped_steps + 1
    assert st1.loss_scale == st0.loss_scale / 2
    assert np.array_equal(pipe.read_params().view(np.uint32), w_before.view(np.uint32))
    m1, v1 = pipe.read_moments()
    assert np.array_equal(m1, m_before) and np.array_equal(v1, v_before)


def test_bucket_size_does_not_change_results_single_rank(torch_cuda, oracle):
    """One rank: bucketing is pure layout, results identical for any threshold."""
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 9)
    outs = []
    for bb in (1, 4096, 1 << 30):
        cfg = TrainerConfig(LambConfig(), 2, bb, False, 0, ScalerConfig(init_scale=256.0))
        pipe, _, _ = run_pipeline(spec, cfg, p0, steps=2)
        outs.append(pipe.read_params())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


@pytest.mark.slow
def test_bert_base_config1_matches_oracle(torch_cuda, oracle):
    """Config 1: BERT-base-shaped (110M) gradients, 1 worker, LAMB + dynamic scaling."""
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_BASE, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_BASE)
    p0 = oracle.build_params(spec, 1)
    sc = dict(init_scale=2.0 ** 15, growth_interval=2)
    cfg = TrainerConfig(LambConfig(lr=1e-4), 1, 4 << 20, False, 0, ScalerConfig(**sc))
    pipe, su, fi = run_pipeline(spec, cfg, p0, steps=3, spike_ppm=1, spike_exp=1)
    ref = oracle.train(spec, p0, 1, 1, 4 << 20, False, OL(lr=1e-4), OS(**sc), 3, spike_ppm=1,
                       spike_exp=1)
    _compare(pipe, ref, su, fi)


@pytest.mark.slow
@pytest.mark.parametrize("resident", [False, True])
def test_bert_large_config2_matches_oracle(torch_cuda, oracle, resident):
    """Config 2 at full size: BERT-large (336M), K=4, one optimizer step,
    through the per-micro API and through bo_train_step."""
    from oracle.oracle import LambConfig as OL, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_LARGE, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_LARGE)
    p0 = oracle.build_params(spec, 1)
    cfg = TrainerConfig(LambConfig(lr=1e-4), 4, 4 << 20, False, 0, ScalerConfig())
    pipe, su, fi = run_pipeline(spec, cfg, p0, steps=1, resident=resident)
    assert ("resident_micros" in pipe.path()) == resident
    ref = oracle.train(spec, p0, 1, 4, 4 << 20, False, OL(lr=1e-4), OS(), 1)
    _compare(pipe, ref, su, fi)


def test_checkpoint_resume_is_bit_identical(torch_cuda, oracle):
    """§8(f) row 2: export the device state after 3 steps, import it into a
    fresh context, run 2 more: identical to 5 uninterrupted steps."""
    from paper_2008_00177_b200.errors import BucketLayoutMismatch
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import (GradPipeline, LambConfig, ScalerConfig,
                                                TrainerConfig)
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    p0 = oracle.build_params(spec, 13)
    cfg = TrainerConfig(LambConfig(), 2, 8192, False, 0, ScalerConfig(init_scale=2.0 ** 14,
                                                                       growth_interval=2))
    kw = dict(spike_ppm=3, spike_exp=3)
    ref, _, _ = run_pipeline(spec, cfg, p0, steps=5, **kw)
    a, _, _ = run_pipeline(spec, cfg, p0, steps=3, **kw)
    blob = a.export_state()
    b = GradPipeline(spec, cfg)
    b.import_state(blob)
    b, _, _ = run_pipeline(spec, cfg, None, steps=2, pipe=b, first_step=3, **kw)
    assert np.array_equal(b.read_params().view(np.uint32), ref.read_params().view(np.uint32))
    mb, vb = b.read_moments()
    mr, vr = ref.read_moments()
    assert np.array_equal(mb.view(np.uint32), mr.view(np.uint32))
    assert np.array_equal(vb.view(np.uint32), vr.view(np.uint32))
    sb, sr = b.status(), ref.status()
    assert (sb.lamb_step, sb.loss_scale, sb.good_steps, sb.steps) == \
        (sr.lamb_step, sr.loss_scale, sr.good_steps, sr.steps)
    other = GradPipeline(spec, TrainerConfig(LambConfig(), 2, 1 << 20))
    with pytest.raises(BucketLayoutMismatch):
        other.import_state(blob)


@pytest.mark.parametrize("aligned", [True, False])
def test_overlapped_sync_micro_bit_identical(torch_cuda, oracle, aligned):
    """bo_sync_ready (bucket-level overlap, trainer.cpp:247-348) gives the same
    bits as bo_accumulate for the sync micro, overflow steps included."""
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    P = spec.param_count()
    p0 = oracle.build_params(spec, 5)
    cfg = TrainerConfig(LambConfig(lr=1e-2), 3, 4096, False, 0,
                        ScalerConfig(init_scale=2.0 ** 14, growth_interval=3))
    inj = [(2, 0, 2, P // 2, 0x7C00)]
    base, su0, fi0 = run_pipeline(spec, cfg, p0, steps=6, spike_ppm=3, spike_exp=3, injections=inj,
                                  aligned=aligned)
    ovl, su1, fi1 = run_pipeline(spec, cfg, p0, steps=6, spike_ppm=3, spike_exp=3, injections=inj,
                                 aligned=aligned, overlap=[1, 7, 3, 40])
    assert "overlap" in ovl.path()
    assert np.array_equal(su0, su1) and np.array_equal(fi0, fi1) and fi0.any()
    assert np.array_equal(base.read_params().view(np.uint32), ovl.read_params().view(np.uint32))
    m0, v0, m1, v1 = (np.zeros(P, np.float32) for _ in range(4))
    base.read_moments(m0, v0)
    ovl.read_moments(m1, v1)
    assert np.array_equal(m0.view(np.uint32), m1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))


def test_sync_ready_protocol_errors(torch_cuda, oracle):
    from paper_2008_00177_b200.errors import BertoptError
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import GradBuffers

    spec = bert_spec(BERT_TINY)
    cfg = TrainerConfig(LambConfig(), 1, 4096, False, 0, ScalerConfig())
    pipe = GradPipeline(spec, cfg, device=0)
    pipe.load_params(oracle.build_params(spec, 1))
    gb = GradBuffers(spec, 1, 0, True)
    pipe.sync_ready([0], [gb.ptrs[0][0]])
    with pytest.raises(BertoptError):
        pipe.sync_ready([0], [gb.ptrs[0][0]])  # delivered twice
    with pytest.raises(BertoptError):
        pipe.accumulate(0, gb.ptrs[0])  # bo_accumulate while a sync micro is open
    rest = [t for t in range(spec.n_tensors) if t != 0]
    pipe.sync_ready(rest, [gb.ptrs[0][t] for t in rest])
    pipe.synchronize()
    assert pipe.status().lamb_step == 1


def test_watchdog_wait(torch_cuda, oracle):
    """bo_wait: WatchdogTimeout while the context stream is still busy,
    success once it drains (transport.cpp:113-132 semantics)."""
    import torch

    from paper_2008_00177_b200.errors import WatchdogTimeout
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig

    spec = bert_spec(BERT_TINY)
    pipe = GradPipeline(spec, TrainerConfig(LambConfig(), 1, 4096, False, 0, ScalerConfig()))
    pipe.load_params(oracle.build_params(spec, 1))
    s = torch.cuda.Stream()
    pipe.set_stream(s)
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(1.5e9))  # ~0.8 s of device time queued on the context stream
    with pytest.raises(WatchdogTimeout):
        pipe.wait(20)
    pipe.wait(-1)
    pipe.wait(0)  # nothing pending: immediate success


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("aligned", [True, False])
def test_train_step_resident_micros_bit_identical(torch_cuda, oracle, K, aligned):
    """bo_train_step (all K micros resident, no accumulator) gives the same
    bits as K bo_accumulate calls, overflow steps included; unaligned slots
    take the per-micro path inside the call."""
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import run_pipeline

    spec = bert_spec(BERT_TINY)
    P = spec.param_count()
    p0 = oracle.build_params(spec, 8)
    cfg = TrainerConfig(LambConfig(lr=1e-2), K, 4096, False, 0,
                        ScalerConfig(init_scale=2.0 ** 14, growth_interval=3))
    inj = [(2, 0, K - 2, P // 3, 0x7E00), (4, 0, K - 1, 11, 0xFC00)]
    base, su0, fi0 = run_pipeline(spec, cfg, p0, steps=6, spike_ppm=3, spike_exp=3, injections=inj,
                                  aligned=aligned)
    res, su1, fi1 = run_pipeline(spec, cfg, p0, steps=6, spike_ppm=3, spike_exp=3, injections=inj,
                                 aligned=aligned, resident=True)
    assert ("resident_micros" in res.path()) == aligned
    assert np.array_equal(su0, su1) and np.array_equal(fi0, fi1) and fi0.sum() >= 2
    assert np.array_equal(base.read_params().view(np.uint32), res.read_params().view(np.uint32))
    m0, v0, m1, v1 = (np.zeros(P, np.float32) for _ in range(4))
    base.read_moments(m0, v0)
    res.read_moments(m1, v1)
    assert np.array_equal(m0.view(np.uint32), m1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))


def test_micro_order_protocol(torch_cuda, oracle):
    """Micros must arrive 0..K-1; bo_train_step cannot start inside a step fed
    by bo_accumulate (ProtocolError, the reference's protocol-violation class)."""
    from paper_2008_00177_b200.errors import ProtocolError
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import GradBuffers

    spec = bert_spec(BERT_TINY)
    pipe = GradPipeline(spec, TrainerConfig(LambConfig(), 3, 4096, False, 0, ScalerConfig()))
    pipe.load_params(oracle.build_params(spec, 1))
    gb = GradBuffers(spec, 3, 0, True)
    with pytest.raises(ProtocolError):
        pipe.accumulate(1, gb.ptrs[1])
    pipe.accumulate(0, gb.ptrs[0])
    with pytest.raises(ProtocolError):
        pipe.train_step(gb.ptrs)
    pipe.accumulate(1, gb.ptrs[1])
    pipe.accumulate(2, gb.ptrs[2])
    pipe.train_step(gb.ptrs)  # a fresh step
    pipe.synchronize()
    assert pipe.status().lamb_step == 2
