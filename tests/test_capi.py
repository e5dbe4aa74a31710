"""The C-ABI library: loads, exports every symbol include/bertopt_b200.h
declares, and its host-only entry points (layout, sharding) agree with the
reference. No device compute here."""
import ctypes as C
import os
import re
import struct

import numpy as np
import pytest

from paper_2008_00177_b200 import _lib
from paper_2008_00177_b200.model_spec import BERT_BASE, BERT_LARGE, BERT_TINY, bert_spec
from paper_2008_00177_b200.pipeline import BucketLayout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bertopt_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bo_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(names)


def test_abi_basics():
    lib = _lib.load()
    assert lib.bo_abi_version() == 1
    assert lib.bo_status_name(2) == b"NonFiniteGradient"
    assert lib.bo_status_name(6) == b"BucketLayoutMismatch"
    cfg = _lib.TrainerConfigC()
    lib.bo_default_config(C.byref(cfg))
    assert cfg.accumulation == 1 and cfg.bucket_bytes == 4 << 20
    assert abs(cfg.lamb.lr - 1e-3) < 1e-9 and abs(cfg.lamb.beta2 - 0.999) < 1e-7
    assert cfg.lamb.trust_clip == 10.0 and cfg.scaler.init_scale == 65536.0
    assert lib.bo_scale_loss(0.5, 4096.0, 1) == 2048.0


def test_errors_map_to_reference_classes():
    from paper_2008_00177_b200 import errors

    e = errors.from_status(2, "x")
    assert isinstance(e, errors.NonFiniteGradient) and isinstance(e, errors.BertoptError)
    assert isinstance(errors.from_status(5, "x"), errors.InvalidConfig)
    with pytest.raises(errors.InvalidConfig):
        spec = bert_spec(BERT_TINY)
        BucketLayout.build(spec, 0)


def _fnv(data: bytes, h: int) -> int:
    for b in data:
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.parametrize("tag,cfg", [("large", BERT_LARGE), ("base", BERT_BASE)])
def test_bucket_layout_matches_reference_golden(tag, cfg):
    from tests.golden.make_golden import BUCKET_SIZES

    d = np.load(os.path.join(ROOT, "tests", "golden", "layout.npz"))
    spec = bert_spec(cfg)
    for bb in BUCKET_SIZES:
        k = f"{tag}_{bb}"
        for f16, K in ((False, 1), (True, 4)):
            L = BucketLayout.build(spec, bb, f16, K)
            assert np.array_equal(L.bucket_of, d[k + "_bucket_of"])
            assert np.array_equal(L.offset_of, d[k + "_offset_of"])
            assert np.array_equal(L.ready_order, d[k + "_ready"])
            assert np.array_equal(L.bucket_elems, d[k + "_elems"])
            # ensure_layout's salted hash (trainer.cpp:165-168) over the golden hash
            h = _fnv(bytes([int(f16)]), int(d[k + "_hash"][0]))
            h = _fnv(struct.pack("<Q", K), h)
            assert L.hash == h


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_ranges_partition_every_bucket(world):
    spec = bert_spec(BERT_TINY)
    L = BucketLayout.build(spec, 3000)
    cover = [np.zeros(n, np.int32) for n in L.bucket_elems]
    for r in range(world):
        lo, hi = L.shard_ranges(world, r)
        for b, (a, z) in enumerate(zip(lo, hi)):
            cover[b][a:z] += 1
            c = -(-int(L.bucket_elems[b]) // world)
            assert a == min(r * c, L.bucket_elems[b])
    assert all(np.all(c == 1) for c in cover)


def test_create_without_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2008_00177_b200.errors import NoDevice
    from paper_2008_00177_b200.pipeline import GradPipeline, TrainerConfig

    with pytest.raises(NoDevice):
        GradPipeline(bert_spec(BERT_TINY), TrainerConfig())


def test_bucket_layout_with_empty_tensors_matches_reference():
    """Zero-element tensors join the current bucket with 0 bytes, exactly as
    BucketLayout::build does (trainer.cpp:100-114); a model with no element
    at all is rejected."""
    from oracle import oracle as o
    from paper_2008_00177_b200.model_spec import flat_spec

    spec = flat_spec([0, 5, 4097, 0, 3, 1, 8191], first_use=[2, 0, 1, 4, 3, 6, 5])
    for bb in (4, 64, 16384, 1 << 20):
        L = BucketLayout.build(spec, bb)
        bo, off, ro, be = o.Oracle().bucket_layout(spec.numels(), spec.first_consumer_ids(), bb)
        assert np.array_equal(L.bucket_of, bo) and np.array_equal(L.offset_of, off)
        assert np.array_equal(L.ready_order, ro) and np.array_equal(L.bucket_elems, be)
        if o.reference_available():
            bo2, off2, ro2, be2, _h = o.Reference().bucket_layout(spec, spec.first_consumer_ids(), bb)
            assert np.array_equal(L.bucket_of, bo2) and np.array_equal(L.bucket_elems, be2)
    from paper_2008_00177_b200.errors import ShapeMismatch

    with pytest.raises(ShapeMismatch):
        BucketLayout.build(flat_spec([0, 0]), 64)
