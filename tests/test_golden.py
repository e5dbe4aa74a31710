"""The restated oracle against golden fixtures produced by the REAL reference
(tests/golden/make_golden.py over oracle/_ref). Runs anywhere: the fixtures
are committed, /root/reference is not needed."""
import os

import numpy as np
import pytest

from oracle.oracle import LambConfig, ScalerConfig
from paper_2008_00177_b200.model_spec import BERT_BASE, BERT_LARGE, bert_spec
from tests.golden.make_golden import BUCKET_SIZES, GOLDEN_MODEL, TRAIN_CASES

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def test_half_golden(oracle):
    d = load("half.npz")
    x, want = d["x"], d["f16"]
    got = oracle.f32_to_f16(x)
    nan = np.isnan(x)
    assert np.array_equal(got[~nan], want[~nan])
    assert np.all((got[nan] & 0x7FFF) > 0x7C00)
    widen = oracle.f16_to_f32(np.arange(65536, dtype=np.uint16)).view(np.uint32)
    ref = d["widen_all"]
    isnan = ((np.arange(65536) & 0x7C00) == 0x7C00) & ((np.arange(65536) & 0x3FF) != 0)
    assert np.array_equal(widen[~isnan], ref[~isnan])


@pytest.mark.parametrize("tag,cfg", [("large", BERT_LARGE), ("base", BERT_BASE)])
def test_layout_golden(oracle, tag, cfg):
    d = load("layout.npz")
    spec = bert_spec(cfg)
    for bb in BUCKET_SIZES:
        k = f"{tag}_{bb}"
        bo, off, ro, be = oracle.bucket_layout(spec.numels(), spec.first_consumer_ids(), bb)
        assert np.array_equal(bo, d[k + "_bucket_of"])
        assert np.array_equal(off, d[k + "_offset_of"])
        assert np.array_equal(ro, d[k + "_ready"])
        assert np.array_equal(be, d[k + "_elems"])
        assert oracle.layout_hash(spec, bo, ro, be) == int(d[k + "_hash"][0])


def test_layout_bucket_counts_survey():
    """BERT-large bucket counts 295/294/122/25/6/2 at 1..1024 MiB."""
    d = load("layout.npz")
    counts = [len(d[f"large_{bb}_elems"]) for bb in BUCKET_SIZES]
    assert counts == [295, 294, 122, 25, 6, 2]
    assert bert_spec(BERT_LARGE).param_count() == 336226108
    assert bert_spec(BERT_BASE).param_count() == 110106428


def test_lamb_golden(oracle):
    d = load("lamb.npz")
    numels = d["numels"]
    w = d["w0"].copy()
    P = w.size
    m, v = np.zeros(P, np.float32), np.zeros(P, np.float32)
    step = 0
    for s in range(4):
        rc, step = oracle.lamb_step(numels, w, d["g"][s].copy(), m, v, step, LambConfig())
        assert rc == int(d[f"rc{s + 1}"][0]) and step == int(d[f"step{s + 1}"][0])
        for arr, key in ((w, "w"), (m, "m"), (v, "v")):
            assert np.array_equal(arr.view(np.uint32), d[f"{key}{s + 1}"].view(np.uint32)), (s, key)


def test_ring_golden(oracle):
    d = load("ring.npz")
    for world in (2, 3, 4, 8):
        for n in (1, 5, 64, 1537):
            data = d[f"in_{world}_{n}"]
            got32 = oracle.ring_allreduce(data, 0)
            got16 = oracle.ring_allreduce(data, 1)
            for r in range(world):  # identical bits on every rank
                assert np.array_equal(got32[r].view(np.uint32), d[f"f32_{world}_{n}"].view(np.uint32))
                assert np.array_equal(got16[r].view(np.uint32), d[f"f16_{world}_{n}"].view(np.uint32))
    got = oracle.ring_allreduce(d["i64_in"], 2)
    assert np.array_equal(got[0], d["i64_out"]) and d["i64_out"].tolist() == [6, 60, -3]


@pytest.mark.parametrize("case", TRAIN_CASES, ids=[c[0] for c in TRAIN_CASES])
def test_train_golden(oracle, case):
    name, world, K, bb, f16, sc, lc, steps, ppm, sexp, inj = case
    d = load("train.npz")
    spec = bert_spec(GOLDEN_MODEL)
    assert np.array_equal(oracle.build_params(spec, 11), d["init"])
    r = oracle.train(spec, d["init"], world, K, bb, f16, LambConfig(**lc), ScalerConfig(**sc), steps,
                     grad_seed=5, spike_ppm=ppm, spike_exp=sexp, injections=inj)
    assert np.array_equal(r.found_inf, d[f"{name}_found_inf"])
    assert np.array_equal(r.scale_used, d[f"{name}_scale_used"])
    assert r.final_scale == float(d[f"{name}_final_scale"][0])
    assert [r.lamb_step, r.final_good] == d[f"{name}_meta"].tolist()
    for key, arr in (("params", r.params), ("m", r.m), ("v", r.v)):
        assert np.array_equal(arr.view(np.uint32), d[f"{name}_{key}"].view(np.uint32)), key
