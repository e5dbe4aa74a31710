"""The paper's fused elementwise optimizer:
fused_optimizer_step (graph.cpp:458-487) run by run_fused_kernel, and the
AMP f16 cast. The oracle restatement is pinned by the reference's own tests
(test_graph.cpp:395-452, restated here; graph.cpp needs Eigen, so it cannot be
compiled in this image); the CUDA kernel is checked bit for bit against the
oracle in the gpu section."""
import numpy as np
import pytest


def _inputs(rng, n):
    w = rng.uniform(-1.0, 1.0, n).astype(np.float32)
    g = rng.uniform(-0.2, 0.2, n).astype(np.float32)
    m = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    v = (rng.uniform(0.0, 0.1, n).astype(np.float32)) ** 2
    return w, g, m, v.astype(np.float32)


def test_oracle_matches_double_closed_form(oracle):
    """test_graph.cpp:395-437: fused step vs a double-precision scalar oracle."""
    lr, b1, b2, eps, wd, step = 1e-3, 0.9, 0.999, 1e-6, 0.01, 7
    w, g, m, v = _inputs(np.random.default_rng(20), 256)
    w0, g0, m0, v0 = w.copy(), g.copy(), m.copy(), v.copy()
    oracle.fused_optimizer_step(w, g, m, v, lr, b1, b2, eps, wd, step)
    f = np.float32
    bc1 = 1.0 / (1.0 - float(f(b1)) ** step)
    bc2 = 1.0 / (1.0 - float(f(b2)) ** step)
    d = np.float64
    mn = float(f(b1)) * m0.astype(d) + (1.0 - float(f(b1))) * g0.astype(d)
    vn = float(f(b2)) * v0.astype(d) + (1.0 - float(f(b2))) * g0.astype(d) * g0
    u = mn * bc1 / (np.sqrt(vn * bc2) + float(f(eps))) + float(f(wd)) * w0.astype(d)
    wn = w0.astype(d) - float(f(lr)) * u
    assert np.max(np.abs(w - wn)) <= 1e-5
    assert np.max(np.abs(m - mn)) <= 1e-6
    assert np.max(np.abs(v - vn)) <= 1e-6


def test_oracle_zero_gradient_fresh_state_is_noop(oracle):
    """test_graph.cpp:439-452."""
    rng = np.random.default_rng(21)
    w = rng.uniform(-2.0, 2.0, 64).astype(np.float32)
    w0 = w.copy()
    z = np.zeros(64, np.float32)
    m, v = z.copy(), z.copy()
    oracle.fused_optimizer_step(w, z, m, v, 1e-2, 0.9, 0.999, 1e-6, 0.0, 1)
    assert np.array_equal(w, w0) and not m.any() and not v.any()


def test_oracle_f16_round_matches_reference_conversions(oracle):
    """quantize_inplace = f16_to_f32(f32_to_f16(x)) (half.cpp:23-79), checked
    against the oracle's own (reference-pinned) scalar conversions."""
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(4096).astype(np.float32) * 1e3,
                        np.array([65504, 65519.99, 65520, 2.0 ** -24, 2.0 ** -25, -0.0, np.inf],
                                 np.float32)])
    y = x.copy()
    oracle.f16_round(y)
    ref = oracle.f16_to_f32(oracle.f32_to_f16(x))
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))
