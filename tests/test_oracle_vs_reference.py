"""Pin the restated oracle against the REAL reference compiled from
/root/reference (oracle/_ref). Skipped where the reference was not built."""
import numpy as np
import pytest

from oracle.oracle import LambConfig, ScalerConfig
from paper_2008_00177_b200.model_spec import BERT_TINY, ModelConfig, bert_spec, flat_spec


def test_f16_random_bits(oracle, reference):
    rng = np.random.default_rng(7)
    x = rng.integers(0, 2 ** 32, 1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    a, b = oracle.f32_to_f16(x), reference.f32_to_f16(x)
    nan = np.isnan(x)
    assert np.array_equal(a[~nan], b[~nan])
    # the F16C block path agrees with the scalar path (graph.cpp:176-199)
    c = reference.narrow_block(x)
    assert np.array_equal(c[~nan], b[~nan])


def test_f16_all_patterns(oracle, reference):
    h = np.arange(65536, dtype=np.uint16)
    a, b = oracle.f16_to_f32(h), reference.f16_to_f32(h)
    nan = np.isnan(b)
    assert np.array_equal(a[~nan].view(np.uint32), b[~nan].view(np.uint32))
    assert np.array_equal(np.isnan(a), nan)


@pytest.mark.parametrize("numels", [[5, 1, 300, 4097], [1], [70000, 3]])
def test_lamb_step(oracle, reference, numels):
    rng = np.random.default_rng(len(numels))
    P = sum(numels)
    wa = (rng.standard_normal(P) * 0.02).astype(np.float32)
    wb = wa.copy()
    ma, va = np.zeros(P, np.float32), np.zeros(P, np.float32)
    mb, vb = ma.copy(), va.copy()
    sa = sb = 0
    cfg = LambConfig(lr=1e-2, weight_decay=0.05)
    for s in range(5):
        g = (rng.standard_normal(P) * 10.0 ** -rng.integers(2, 6)).astype(np.float32)
        if s == 4 and P > 10:
            g[P // 2] = np.nan
        ra, sa = oracle.lamb_step(numels, wa, g, ma, va, sa, cfg)
        rb, sb = reference.lamb_step(numels, wb, g, mb, vb, sb, cfg)
        assert ra == rb and sa == sb
        for x, y in ((wa, wb), (ma, mb), (va, vb)):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 5, 64, 1537])
def test_ring_allreduce(oracle, reference, world, n):
    rng = np.random.default_rng(world * 100 + n)
    data = rng.uniform(-2, 2, (world, n)).astype(np.float32)
    for kind in (0, 1):
        a = oracle.ring_allreduce(data, kind)
        b, sent = reference.ring_allreduce(data, kind)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        assert all(s == oracle.ring_allreduce_bytes(n, world, 2 if kind else 4) for s in sent)


def test_bucket_layout_and_hash(oracle, reference):
    spec = bert_spec(BERT_TINY)
    for bb in (1, 512, 4096, 1 << 16, 1 << 30):
        bo, off, ro, be = oracle.bucket_layout(spec.numels(), spec.first_consumer_ids(), bb)
        bo2, off2, ro2, be2, h = reference.bucket_layout(spec, spec.first_consumer_ids(), bb)
        assert np.array_equal(bo, bo2) and np.array_equal(off, off2)
        assert np.array_equal(ro, ro2) and np.array_equal(be, be2)
        assert oracle.layout_hash(spec, bo, ro, be) == h


SMALL = ModelConfig(layers=1, hidden=32, heads=4, vocab=300, max_seq=16)


@pytest.mark.parametrize("world,K,f16,bb", [(1, 1, False, 2048), (1, 4, False, 1 << 30),
                                            (2, 2, True, 4096), (3, 3, False, 700),
                                            (4, 1, True, 1 << 20), (8, 2, True, 3000)])
def test_train_real_trainer(oracle, reference, world, K, f16, bb):
    """The real DistributedTrainer::train_step (threads over InProcHub) vs the
    single-thread restatement, incl. the dynamic scaler with overflow injection."""
    spec = bert_spec(SMALL)
    P = spec.param_count()
    p0 = reference.build_params(spec, 3)
    assert np.array_equal(p0, oracle.build_params(spec, 3))
    sc = ScalerConfig(init_scale=2.0 ** 13, growth_interval=2)
    inj = [(1, world - 1, K - 1, P - 7, 0x7C00)]
    args = (world, K, bb, f16, LambConfig(lr=3e-3), sc, 6)
    kw = dict(grad_seed=world * 10 + K, spike_ppm=30, spike_exp=3, injections=inj)
    a = oracle.train(spec, p0, *args, **kw)
    b = reference.train(spec, 3, *args, **kw)
    assert a.found_inf.tolist() == b.found_inf.tolist() and a.found_inf.sum() >= 1
    assert np.array_equal(a.scale_used, b.scale_used)
    assert (a.lamb_step, a.final_scale, a.final_good) == (b.lamb_step, b.final_scale, b.final_good)
    for x, y in ((a.params, b.params), (a.m, b.m), (a.v, b.v)):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_overlap_on_off_identical(reference):
    """test_collective.cpp:817-912: identical bits with or without overlap."""
    spec = bert_spec(SMALL)
    kw = dict(grad_seed=3)
    a = reference.train(spec, 1, 2, 2, 2048, False, LambConfig(), ScalerConfig(), 2, overlap=True, **kw)
    b = reference.train(spec, 1, 2, 2, 2048, False, LambConfig(), ScalerConfig(), 2, overlap=False, **kw)
    assert np.array_equal(a.params, b.params)


def test_flat_spec_tensor_boundaries(oracle, reference):
    """Ragged tensors around chunk boundaries (sizes 1 and primes)."""
    spec = flat_spec([1, 7, 13, 1, 4099, 2, 31], first_use=[6, 0, 5, 1, 4, 2, 3])
    p0 = oracle.build_params(spec, 2)
    for world, f16 in ((3, True), (4, False), (8, True)):
        a = oracle.train(spec, p0, world, 2, 64, f16, LambConfig(), ScalerConfig(), 3)
        b = reference.train(spec, 2, world, 2, 64, f16, LambConfig(), ScalerConfig(), 3)
        assert np.array_equal(a.params.view(np.uint32), b.params.view(np.uint32))


def test_empty_tensors(oracle, reference):
    """Zero-element tensors (an empty bucket member, W = U = 0 -> trust 1)
    next to ragged ones, worlds 1-4, both wires."""
    spec = flat_spec([0, 5, 4097, 0, 3], first_use=[2, 0, 1, 4, 3])
    p0 = oracle.build_params(spec, 3)
    for world, f16 in ((1, False), (2, True), (3, False), (4, True)):
        a = oracle.train(spec, p0, world, 2, 4096, f16, LambConfig(), ScalerConfig(), 3)
        b = reference.train(spec, 3, world, 2, 4096, f16, LambConfig(), ScalerConfig(), 3)
        assert np.array_equal(a.params.view(np.uint32), b.params.view(np.uint32))
        assert np.array_equal(a.m.view(np.uint32), b.m.view(np.uint32))
