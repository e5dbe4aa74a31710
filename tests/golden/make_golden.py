"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs the reference hot path compiled from /root/reference (oracle/_ref, built
by oracle/ref/Makefile) and records inputs + outputs as small .npz files. The
fixtures are committed; /root/reference is NOT needed to use them (the GPU box
has no copy of it). Regenerate with:

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import LambConfig, Reference, ScalerConfig, build  # noqa: E402
from paper_2008_00177_b200.model_spec import (BERT_BASE, BERT_LARGE, ModelConfig,  # noqa: E402
                                              bert_spec)

GOLDEN_MODEL = ModelConfig(layers=1, hidden=32, heads=4, vocab=200, max_seq=16)
BUCKET_SIZES = [1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30]

# (name, world, K, bucket_bytes, f16, scaler kwargs, lamb kwargs, steps, spike_ppm, spike_exp, inj)
TRAIN_CASES = [
    ("w1_k1_static", 1, 1, 2048, False, dict(init_scale=4096.0, dynamic=0), {}, 3, 0, 1, []),
    ("w1_k3_dynamic", 1, 3, 1024, False, dict(init_scale=2.0 ** 14, growth_interval=3), dict(lr=1e-2),
     12, 40, 3, [(4, 0, 1, 7, 0x7C00), (7, 0, 2, 100, 0x7E00)]),
    ("w2_k2_f32", 2, 2, 4096, False, dict(init_scale=1024.0), {}, 3, 0, 1, []),
    ("w2_k2_f16", 2, 2, 4096, True, dict(init_scale=1024.0), {}, 3, 0, 1, []),
    ("w3_k1_f16_dynamic", 3, 1, 512, True, dict(init_scale=2.0 ** 13, growth_interval=2),
     dict(lr=5e-3), 8, 60, 3, [(3, 2, 0, 55, 0xFC00)]),
    ("w4_k4_f32_1bucket", 4, 4, 1 << 30, False, dict(init_scale=256.0), {}, 2, 0, 1, []),
]


def main() -> None:
    build()
    ref = Reference()
    rng = np.random.default_rng(20080177)

    # --- binary16 (half.cpp:23-77)
    bits = rng.integers(0, 2 ** 32, 1 << 16, dtype=np.uint64).astype(np.uint32)
    edges = []
    for e in range(-30, 18):
        for s in range(-4, 5):
            x = np.ldexp(np.float32(1.0), e) * np.float32(1.0 + s * 2.0 ** -13)
            edges += [x, -x]
    x = np.concatenate([bits.view(np.float32), np.asarray(edges, np.float32)])
    np.savez_compressed(os.path.join(HERE, "half.npz"), x=x, f16=ref.f32_to_f16(x),
                        widen_all=ref.f16_to_f32(np.arange(65536, dtype=np.uint16)).view(np.uint32))

    # --- bucket layouts (trainer.cpp:73-134)
    lay = {}
    for tag, cfg in (("large", BERT_LARGE), ("base", BERT_BASE)):
        spec = bert_spec(cfg)
        for bb in BUCKET_SIZES:
            bo, off, ro, be, h = ref.bucket_layout(spec, spec.first_consumer_ids(), bb)
            k = f"{tag}_{bb}"
            lay[k + "_bucket_of"] = bo
            lay[k + "_offset_of"] = off
            lay[k + "_ready"] = ro
            lay[k + "_elems"] = be
            lay[k + "_hash"] = np.array([h], np.uint64)
    np.savez_compressed(os.path.join(HERE, "layout.npz"), **lay)

    # --- lamb_step (lamb.cpp:23-84), including the NonFiniteGradient partial update
    numels = np.array([4097, 1, 300, 2048, 7], np.int64)
    P = int(numels.sum())
    w0 = (rng.standard_normal(P) * 0.02).astype(np.float32)
    gs = (rng.standard_normal((4, P)) * 1e-3).astype(np.float32)
    gs[3, 4097 + 1 + 150] = np.inf
    w, m, v = w0.copy(), np.zeros(P, np.float32), np.zeros(P, np.float32)
    step = 0
    out = {"numels": numels, "w0": w0, "g": gs}
    for s in range(4):
        rc, step = ref.lamb_step(numels, w, gs[s], m, v, step, LambConfig())
        out[f"w{s + 1}"], out[f"m{s + 1}"], out[f"v{s + 1}"] = w.copy(), m.copy(), v.copy()
        out[f"rc{s + 1}"] = np.array([rc])
        out[f"step{s + 1}"] = np.array([step])
    np.savez_compressed(os.path.join(HERE, "lamb.npz"), **out)

    # --- ring all-reduce (collective.hpp:53-99, collective.cpp:37-86)
    ring = {}
    for world in (2, 3, 4, 8):
        for n in (1, 5, 64, 1537):
            data = rng.uniform(-2, 2, (world, n)).astype(np.float32)
            ring[f"in_{world}_{n}"] = data
            ring[f"f32_{world}_{n}"] = ref.ring_allreduce(data, 0)[0][0]
            ring[f"f16_{world}_{n}"] = ref.ring_allreduce(data, 1)[0][0]
    ints = np.array([[r + 1, 10 * (r + 1), -r] for r in range(3)], np.int64)
    ring["i64_in"] = ints
    ring["i64_out"] = ref.ring_allreduce(ints, 2)[0][0]
    np.savez_compressed(os.path.join(HERE, "ring.npz"), **ring)

    # --- full train_step runs with the dynamic scaler extension (trainer.cpp:217-373)
    spec = bert_spec(GOLDEN_MODEL)
    tr = {"init": ref.build_params(spec, 11)}
    for (name, world, K, bb, f16, sc, lc, steps, ppm, sexp, inj) in TRAIN_CASES:
        r = ref.train(spec, 11, world, K, bb, f16, LambConfig(**lc), ScalerConfig(**sc), steps,
                      grad_seed=5, spike_ppm=ppm, spike_exp=sexp, injections=inj)
        tr[f"{name}_params"] = r.params
        tr[f"{name}_m"] = r.m
        tr[f"{name}_v"] = r.v
        tr[f"{name}_meta"] = np.array([r.lamb_step, r.final_good], np.int64)
        tr[f"{name}_scale_used"] = r.scale_used
        tr[f"{name}_found_inf"] = r.found_inf
        tr[f"{name}_final_scale"] = np.array([r.final_scale], np.float32)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **tr)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
