"""GPU parity of the operator-level drop-ins against the oracle and the
reference's own known-answer tests (restated from proj/tests)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


def test_synth_generator_matches_oracle(torch, oracle):
    from paper_2008_00177_b200.pipeline import synth_grads

    P = 1 << 20
    for (seed, rank, step, micro, scale, ppm, sexp) in [(1, 0, 0, 0, 4096.0, 0, 1),
                                                         (7, 3, 11, 2, 65536.0, 50, 1),
                                                         (9, 1, 2, 3, 1.0, 1000, -3)]:
        d = torch.empty(P, dtype=torch.int16, device="cuda")
        synth_grads(d, 0, seed, rank, step, micro, scale, ppm, sexp)
        got = d.cpu().numpy().view(np.uint16)
        want = oracle.synth_grads(P, seed, rank, step, micro, scale, ppm, sexp)
        assert np.array_equal(got, want)
        # offset windows agree with the flat index space
        d2 = torch.empty(1000, dtype=torch.int16, device="cuda")
        synth_grads(d2, 12345, seed, rank, step, micro, scale, ppm, sexp)
        assert np.array_equal(d2.cpu().numpy().view(np.uint16), want[12345:13345])


def test_narrow_widen_all_patterns(torch, oracle):
    from paper_2008_00177_b200.pipeline import narrow_f16, widen_f16

    h = torch.arange(65536, dtype=torch.int32).to(torch.int16).cuda()
    f = torch.empty(65536, dtype=torch.float32, device="cuda")
    widen_f16(h, f)
    torch.cuda.synchronize()
    got = f.cpu().numpy()
    want = oracle.f16_to_f32(np.arange(65536, dtype=np.uint16))
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), want[~nan].view(np.uint32))

    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2 ** 32, 1 << 22, dtype=np.uint64).astype(np.uint32)
    edges = []
    for e in range(-30, 18):
        for s in range(-4, 5):
            x = np.ldexp(np.float32(1.0), e) * np.float32(1.0 + s * 2.0 ** -13)
            edges += [x, -x]
    x = np.concatenate([bits.view(np.float32), np.array(edges, np.float32),
                        np.array([65504, 65519.99, 65520, 2 ** -25, 2 ** -24, np.inf, -np.inf],
                                 np.float32)])
    xd = torch.from_numpy(x).cuda()
    hd = torch.empty(x.size, dtype=torch.int16, device="cuda")
    narrow_f16(xd, hd)
    torch.cuda.synchronize()
    got = hd.cpu().numpy().view(np.uint16)
    want = oracle.f32_to_f16(x)
    nan = np.isnan(x)
    assert np.array_equal(got[~nan], want[~nan])
    assert np.all((got[nan] & 0x7C00) == 0x7C00) and np.all((got[nan] & 0x3FF) != 0)


def test_unscale_gradients(torch):
    from paper_2008_00177_b200.errors import InvalidConfig, OverflowDetected
    from paper_2008_00177_b200.pipeline import scale_loss, unscale_gradients

    g = torch.tensor([2048.0, -1.0, 3.0], device="cuda")
    unscale_gradients(g, 4096.0)
    assert g.cpu().tolist() == [0.5, -1.0 / 4096, 3.0 / 4096]
    bad = torch.tensor([1.0, float("inf")], device="cuda")
    with pytest.raises(OverflowDetected):
        unscale_gradients(bad, 4096.0)
    assert bad.cpu().tolist()[0] == 1.0  # untouched
    with pytest.raises(OverflowDetected):
        unscale_gradients(torch.tensor([float("nan")], device="cuda"), 2.0)
    with pytest.raises(InvalidConfig):
        unscale_gradients(torch.tensor([1.0], device="cuda"), 3.0)
    assert scale_loss(0.5, 4096.0) == 2048.0 and scale_loss(123.0, 8.0, False) == 123.0
    # scale then unscale is the identity (test_half.cpp:120-131)
    rng = np.random.default_rng(13)
    v = (np.exp2(rng.uniform(-100, 90, 20000)) * np.where(np.arange(20000) % 2, -1, 1)).astype(np.float32)
    d = torch.from_numpy(v * np.float32(4096.0)).cuda()
    unscale_gradients(d, 4096.0)
    assert np.array_equal(d.cpu().numpy(), v)


def _lamb_case(oracle, numels, seed, steps, cfg_kwargs, inf_at=None):
    import torch as T

    from oracle.oracle import LambConfig as OL
    from paper_2008_00177_b200.pipeline import LambConfig, lamb_step

    rng = np.random.default_rng(seed)
    P = sum(numels)
    w = (rng.standard_normal(P) * 0.02).astype(np.float32)
    w_ref = w.copy()
    m_ref = np.zeros(P, np.float32)
    v_ref = np.zeros(P, np.float32)
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(int)
    params = [T.from_numpy(w[offs[i]:offs[i + 1]].copy()).cuda() for i in range(len(numels))]
    state = {}
    step_ref = 0
    rcs = []
    for s in range(steps):
        g = (rng.standard_normal(P) * 1e-3).astype(np.float32)
        if inf_at is not None and s == steps - 1:
            g[inf_at] = np.inf
        grads = [T.from_numpy(g[offs[i]:offs[i + 1]].copy()).cuda() for i in range(len(numels))]
        rc_ref, step_ref = oracle.lamb_step(numels, w_ref, g, m_ref, v_ref, step_ref,
                                            OL(**cfg_kwargs))
        err = None
        try:
            lamb_step(params, grads, state, LambConfig(**cfg_kwargs))
        except Exception as e:  # noqa: BLE001
            err = e
        rcs.append((rc_ref, err))
    T.cuda.synchronize()
    w_got = np.concatenate([p.cpu().numpy() for p in params])
    m_got = np.concatenate([t.cpu().numpy() for t in state["m"]])
    v_got = np.concatenate([t.cpu().numpy() for t in state["v"]])
    return (w_got, m_got, v_got, state["step"]), (w_ref, m_ref, v_ref, step_ref), rcs


def test_lamb_step_operator_matches_oracle(torch, oracle):
    numels = [4096 * 3 + 17, 1, 1000, 50000, 7]
    got, ref, rcs = _lamb_case(oracle, numels, 1, 5, {})
    assert all(rc == 0 and e is None for rc, e in rcs)
    assert got[3] == ref[3] == 5
    assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))   # m exact
    assert np.array_equal(got[2].view(np.uint32), ref[2].view(np.uint32))   # v exact
    rel = np.abs(got[0].astype(np.float64) - ref[0]) / np.maximum(np.abs(ref[0]), 1e-6)
    assert rel.max() <= 1e-6


def test_lamb_step_nonfinite_partial_update(torch, oracle):
    from paper_2008_00177_b200.errors import NonFiniteGradient

    numels = [300, 5000, 200]
    got, ref, rcs = _lamb_case(oracle, numels, 2, 3, {}, inf_at=300 + 1234)
    rc_ref, err = rcs[-1]
    assert rc_ref == 2 and isinstance(err, NonFiniteGradient)
    assert got[3] == ref[3] == 3  # step incremented before the throw (lamb.cpp:40)
    assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))
    assert np.array_equal(got[2].view(np.uint32), ref[2].view(np.uint32))
    rel = np.abs(got[0].astype(np.float64) - ref[0]) / np.maximum(np.abs(ref[0]), 1e-6)
    assert rel.max() <= 1e-6


def test_lamb_closed_form_scalar(torch):
    """test_model.cpp:383-412: three steps of a scalar parameter vs the closed form."""
    import torch as T

    from paper_2008_00177_b200.pipeline import LambConfig, lamb_step

    cfg = LambConfig(lr=0.1, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=0.1)
    p = [T.tensor([0.5], device="cuda")]
    st = {}
    w, mm, vv = 0.5, 0.0, 0.0
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.99))
    for t, gs in enumerate([0.1, -0.3, 0.2], start=1):
        gs32 = float(np.float32(gs))
        lamb_step(p, [T.tensor([gs], device="cuda")], st, cfg)
        mm = b1 * mm + (1 - b1) * gs32
        vv = b2 * vv + (1 - b2) * gs32 * gs32
        mh = mm / (1 - b1 ** t)
        vh = vv / (1 - b2 ** t)
        u = mh / (np.sqrt(vh) + float(np.float32(1e-8))) + float(np.float32(0.1)) * w
        r = min(abs(w) / abs(u), 10.0) if (w != 0 and u != 0) else 1.0
        w -= float(np.float32(0.1)) * r * u
        assert abs(p[0].item() - w) <= 1e-6
    assert st["step"] == 3


def test_lamb_zero_grad_no_decay_is_noop(torch):
    """test_model.cpp:368-381."""
    import torch as T

    from paper_2008_00177_b200.pipeline import LambConfig, lamb_step

    params = [T.randn(4, 4, device="cuda"), T.randn(8, device="cuda")]
    before = [p.clone() for p in params]
    st = {}
    lamb_step(params, [T.zeros(4, 4, device="cuda"), T.zeros(8, device="cuda")], st,
              LambConfig(weight_decay=0.0))
    assert all(T.equal(a, b) for a, b in zip(params, before))
    assert st["step"] == 1


def test_lamb_scale_invariance_first_step(torch):
    """test_model.cpp:414-435: x7 gradients give the same first update (<=1e-5)."""
    import torch as T

    from paper_2008_00177_b200.pipeline import LambConfig, lamb_step

    g = T.Generator().manual_seed(5)
    pa = [T.randn(64, generator=g).cuda(), T.randn(32, generator=g).cuda()]
    pb = [p.clone() for p in pa]
    g1 = [T.randn(64, generator=g).cuda(), T.randn(32, generator=g).cuda()]
    g7 = [x * 7.0 for x in g1]
    lamb_step(pa, g1, {}, LambConfig(weight_decay=0.0))
    lamb_step(pb, g7, {}, LambConfig(weight_decay=0.0))
    for a, b, gg in zip(pa, pb, g1):
        mask = gg.abs() >= 1e-6
        assert float((a - b)[mask].abs().max()) <= 1e-5


def test_lamb_error_conditions(torch):
    """test_model.cpp:437-450."""
    import torch as T

    from paper_2008_00177_b200.errors import NonFiniteGradient, ShapeMismatch
    from paper_2008_00177_b200.pipeline import LambConfig, lamb_step

    params = [T.randn(4, device="cuda")]
    with pytest.raises(ShapeMismatch):
        lamb_step(params, [], {}, LambConfig())
    with pytest.raises(ShapeMismatch):
        lamb_step(params, [T.zeros(5, device="cuda")], {}, LambConfig())
    bad = T.zeros(4, device="cuda")
    bad[2] = float("inf")
    with pytest.raises(NonFiniteGradient):
        lamb_step(params, [bad], {}, LambConfig())


@pytest.mark.parametrize("step", [1, 7, 1000])
def test_fused_optimizer_step_bit_exact(torch, oracle, step):
    """bo_fused_optimizer_step vs the oracle restatement of
    fused_optimizer_step (graph.cpp:458-487): bit for bit, over ragged and
    misaligned tensors (the scalar path) and aligned ones (float4 path)."""
    from paper_2008_00177_b200.pipeline import fused_optimizer_step

    rng = np.random.default_rng(step)
    sizes = [1, 7, 4099, 130001, 4096 * 3]
    host = []
    for n in sizes:
        w = rng.uniform(-1.0, 1.0, n).astype(np.float32)
        g = rng.uniform(-0.2, 0.2, n).astype(np.float32)
        m = rng.uniform(-0.05, 0.05, n).astype(np.float32)
        v = (rng.uniform(0.0, 0.1, n) ** 2).astype(np.float32)
        host.append([w, g, m, v])
    # device copies; the second tensor set lives one element into a buffer
    dev = []
    for i, arrs in enumerate(host):
        off = 1 if i % 2 else 0
        ts = []
        for a in arrs:
            buf = torch.zeros(a.size + off, dtype=torch.float32, device="cuda")
            buf[off:] = torch.from_numpy(a).cuda()
            ts.append(buf[off:])
        dev.append(ts)
    args = (1e-3, 0.9, 0.999, 1e-6, 0.01, step)
    fused_optimizer_step([d[0] for d in dev], [d[1] for d in dev], [d[2] for d in dev],
                         [d[3] for d in dev], *args)
    torch.cuda.synchronize()
    for (w, g, m, v), d in zip(host, dev):
        oracle.fused_optimizer_step(w, g, m, v, *args)
        for want, got in ((w, d[0]), (m, d[2]), (v, d[3])):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_fused_optimizer_zero_gradient_is_noop(torch):
    """test_graph.cpp:439-452 on the device."""
    from paper_2008_00177_b200.pipeline import fused_optimizer_step

    w = (torch.rand(5000, device="cuda") * 4 - 2)
    w0 = w.clone()
    z = [torch.zeros(5000, device="cuda") for _ in range(3)]
    fused_optimizer_step([w], [z[0]], [z[1]], [z[2]], 1e-2, 0.9, 0.999, 1e-6, 0.0, 1)
    torch.cuda.synchronize()
    assert torch.equal(w, w0) and not z[1].any() and not z[2].any()


def test_f16_round_matches_oracle(torch, oracle):
    from paper_2008_00177_b200.pipeline import f16_round

    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(1 << 20).astype(np.float32) * 100,
                        np.array([65504, 65519.99, 65520, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.01,
                                  -0.0, np.inf, -np.inf], np.float32)])
    d = torch.from_numpy(x.copy()).cuda()
    f16_round(d)
    torch.cuda.synchronize()
    want = x.copy()
    oracle.f16_round(want)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), want.view(np.uint32))
