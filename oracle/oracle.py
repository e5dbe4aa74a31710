"""TEST INFRASTRUCTURE — ctypes front end to the two CPU checkers.

* ``Oracle``    — the restated oracle, ``oracle/liboracle.so`` (bo_oracle.cpp).
* ``Reference`` — the real reference hot path compiled from /root/reference
  (``oracle/_ref/libbertopt_ref.so``, built by ``oracle/ref/Makefile``).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbertopt_ref.so")
REFERENCE_SRC = "/root/reference/proj/core"

_f32p = C.POINTER(C.c_float)
_u16p = C.POINTER(C.c_uint16)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int)


def build(force: bool = False) -> None:
    """Compile the restated oracle, and the reference harness if its sources exist."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if os.path.isdir(REFERENCE_SRC):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "ref")], check=True)
        # the C++ adapter test binary links the product library: build it when
        # that exists (tests/test_gpu_adapter.py runs it on a GPU box)
        product = os.path.join(os.path.dirname(HERE), "paper_2008_00177_b200", "libbertopt_b200.so")
        if os.path.exists(product):
            subprocess.run(["make", "-s", "-C", os.path.join(HERE, "ref"), "adapter_test"], check=True)


@dataclass
class LambConfig:
    """Mirror of ``bertopt::LambConfig`` (lamb.hpp:30-37)."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-6
    weight_decay: float = 0.01
    trust_clip: float = 10.0

    def arr(self):
        return (C.c_float * 6)(self.lr, self.beta1, self.beta2, self.eps,
                               self.weight_decay, self.trust_clip)


@dataclass
class ScalerConfig:
    init_scale: float = 65536.0
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    min_scale: float = 1.0
    max_scale: float = 16777216.0
    growth_interval: int = 2000
    dynamic: int = 1


class _Scaler(C.Structure):
    _fields_ = [("init_scale", C.c_float), ("growth_factor", C.c_float),
                ("backoff_factor", C.c_float), ("min_scale", C.c_float),
                ("max_scale", C.c_float), ("growth_interval", C.c_int),
                ("dynamic", C.c_int)]


def _scaler(sc: ScalerConfig) -> _Scaler:
    return _Scaler(sc.init_scale, sc.growth_factor, sc.backoff_factor, sc.min_scale,
                   sc.max_scale, sc.growth_interval, sc.dynamic)


class _Spec(C.Structure):
    _fields_ = [("n_tensors", C.c_int), ("names", C.POINTER(C.c_char_p)),
                ("ndims", _i32p), ("dims", _i64p), ("init", _i32p), ("first_use", _i32p)]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class TrainResult:
    params: np.ndarray
    m: np.ndarray
    v: np.ndarray
    lamb_step: int
    scale_used: np.ndarray
    found_inf: np.ndarray
    final_scale: float
    final_good: int


def _inj_array(injections):
    arr = np.zeros((max(len(injections), 1), 5), dtype=np.int64)
    for i, e in enumerate(injections):
        arr[i] = e
    return arr


class Oracle:
    """The restated oracle (bo_oracle.cpp)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.or_f32_to_f16.argtypes = [_f32p, _u16p, C.c_size_t]
        L.or_f16_to_f32.argtypes = [_u16p, _f32p, C.c_size_t]
        L.or_fnv1a.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.or_fnv1a.restype = C.c_uint64
        L.or_ring_chunk_elems.argtypes = [C.c_size_t, C.c_int]
        L.or_ring_chunk_elems.restype = C.c_size_t
        L.or_ring_allreduce_bytes.argtypes = [C.c_size_t, C.c_int, C.c_size_t]
        L.or_ring_allreduce_bytes.restype = C.c_uint64
        L.or_bucket_layout.argtypes = [C.c_int, _i64p, _i32p, C.c_uint64, _i32p, _i64p, _i32p, _i64p]
        L.or_layout_hash.argtypes = [C.c_int, C.POINTER(C.c_char_p), _i32p, _i64p, _i32p,
                                     C.c_int, _i32p, _i64p]
        L.or_layout_hash.restype = C.c_uint64
        L.or_lamb_step.argtypes = [C.c_int, _i64p, _f32p, _f32p, _f32p, _f32p, _i64p, _f32p]
        L.or_fused_optimizer_step.argtypes = [C.c_int64, _f32p, _f32p, _f32p, _f32p, C.c_float,
                                              C.c_float, C.c_float, C.c_float, C.c_float, C.c_int]
        L.or_f16_round.argtypes = [_f32p, C.c_size_t]
        L.or_ring_allreduce.argtypes = [C.c_int, C.c_size_t, C.c_void_p, C.c_int]
        L.or_build_params.argtypes = [C.c_int, _i64p, _i32p, C.c_uint64, _f32p]
        L.or_synth_grads.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_float,
                                     C.c_uint32, C.c_int, _u16p]
        L.or_train.argtypes = [C.c_int, _i64p, _i32p, _f32p, C.c_int, C.c_int, C.c_uint64, C.c_int,
                               _f32p, C.POINTER(_Scaler), C.c_uint64, C.c_uint32, C.c_int, _i64p,
                               C.c_int, _u16p, C.c_int, _f32p, _f32p, _f32p, _i64p, _f32p, _i32p,
                               _f32p, _i32p]

    # -- binary16
    def f32_to_f16(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, dtype=np.uint16)
        self.lib.or_f32_to_f16(_ptr(x, _f32p), _ptr(out, _u16p), x.size)
        return out

    def f16_to_f32(self, h) -> np.ndarray:
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.shape, dtype=np.float32)
        self.lib.or_f16_to_f32(_ptr(h, _u16p), _ptr(out, _f32p), h.size)
        return out

    def fnv1a(self, data: bytes, seed: int = 14695981039346656037) -> int:
        return self.lib.or_fnv1a(data, len(data), seed)

    def ring_chunk_elems(self, n, world):
        return self.lib.or_ring_chunk_elems(n, world)

    def ring_allreduce_bytes(self, n, world, e):
        return self.lib.or_ring_allreduce_bytes(n, world, e)

    def bucket_layout(self, numels, firsts, bucket_bytes):
        T = len(numels)
        nm = np.asarray(numels, dtype=np.int64)
        fs = np.asarray(firsts, dtype=np.int32)
        bo = np.empty(T, np.int32)
        off = np.empty(T, np.int64)
        ro = np.empty(T, np.int32)
        be = np.empty(T, np.int64)
        nb = self.lib.or_bucket_layout(T, _ptr(nm, _i64p), _ptr(fs, _i32p), bucket_bytes,
                                       _ptr(bo, _i32p), _ptr(off, _i64p), _ptr(ro, _i32p),
                                       _ptr(be, _i64p))
        if nb < 0:
            raise ValueError("InvalidConfig: bucket_bytes must be > 0")
        return bo, off, ro, be[:nb]

    def layout_hash(self, spec, bucket_of, ready_order, bucket_elems) -> int:
        names = (C.c_char_p * spec.n_tensors)(*[n.encode() for n in spec.names])
        nd = np.array([len(s) for s in spec.shapes], np.int32)
        dims = np.array([d for s in spec.shapes for d in s], np.int64)
        bo = np.asarray(bucket_of, np.int32)
        ro = np.asarray(ready_order, np.int32)
        be = np.asarray(bucket_elems, np.int64)
        return self.lib.or_layout_hash(spec.n_tensors, names, _ptr(nd, _i32p), _ptr(dims, _i64p),
                                       _ptr(bo, _i32p), len(be), _ptr(ro, _i32p), _ptr(be, _i64p))

    def lamb_step(self, numels, w, g, m, v, step, cfg: LambConfig):
        """In place on w/m/v (float32 flat arrays); returns (status, new_step)."""
        nm = np.asarray(numels, np.int64)
        st = np.array([step], np.int64)
        rc = self.lib.or_lamb_step(len(numels), _ptr(nm, _i64p), _ptr(w, _f32p), _ptr(g, _f32p),
                                   _ptr(m, _f32p), _ptr(v, _f32p), _ptr(st, _i64p), cfg.arr())
        return rc, int(st[0])

    def ring_allreduce(self, data: np.ndarray, kind: int = 0) -> np.ndarray:
        """data [world, n] (float32, or int64 for kind 2); returns the reduced copy."""
        d = np.ascontiguousarray(data).copy()
        self.lib.or_ring_allreduce(d.shape[0], d.shape[1], d.ctypes.data, kind)
        return d

    def fused_optimizer_step(self, w, g, m, v, lr, beta1, beta2, eps, weight_decay, step):
        """fused_optimizer_step (graph.cpp:458-487) in place on float32 arrays."""
        self.lib.or_fused_optimizer_step(w.size, _ptr(w, _f32p), _ptr(g, _f32p), _ptr(m, _f32p),
                                         _ptr(v, _f32p), lr, beta1, beta2, eps, weight_decay, step)

    def f16_round(self, x):
        """quantize_inplace of a binary16 tensor, in place on a float32 array."""
        self.lib.or_f16_round(_ptr(x, _f32p), x.size)

    def build_params(self, spec, seed: int) -> np.ndarray:
        nm = np.asarray(spec.numels(), np.int64)
        init = np.asarray(spec.init, np.int32)
        out = np.empty(int(nm.sum()), np.float32)
        self.lib.or_build_params(spec.n_tensors, _ptr(nm, _i64p), _ptr(init, _i32p), seed,
                                 _ptr(out, _f32p))
        return out

    def synth_grads(self, P, seed, rank, step, micro, scale, spike_ppm=0, spike_exp=1):
        out = np.empty(P, np.uint16)
        self.lib.or_synth_grads(P, seed, rank, step, micro, scale, spike_ppm, spike_exp,
                                _ptr(out, _u16p))
        return out

    def train(self, spec, params, world, K, bucket_bytes, f16_wire, lamb: LambConfig,
              scaler: ScalerConfig, steps, grad_seed=1, spike_ppm=0, spike_exp=1,
              injections=(), grads=None) -> TrainResult:
        nm = np.asarray(spec.numels(), np.int64)
        P = int(nm.sum())
        fs = np.asarray(spec.first_consumer_ids(), np.int32)
        p_in = np.ascontiguousarray(params, np.float32)
        inj = _inj_array(injections)
        g = None if grads is None else np.ascontiguousarray(grads, np.uint16)
        po, mo, vo = (np.empty(P, np.float32) for _ in range(3))
        ls = np.zeros(1, np.int64)
        su = np.empty(steps, np.float32)
        fi = np.empty(steps, np.int32)
        fsc = np.empty(1, np.float32)
        fg = np.empty(1, np.int32)
        sc = _scaler(scaler)
        rc = self.lib.or_train(spec.n_tensors, _ptr(nm, _i64p), _ptr(fs, _i32p), _ptr(p_in, _f32p),
                               world, K, bucket_bytes, int(f16_wire), lamb.arr(), C.byref(sc),
                               grad_seed, spike_ppm, spike_exp, _ptr(inj, _i64p), len(injections),
                               None if g is None else _ptr(g, _u16p), steps, _ptr(po, _f32p),
                               _ptr(mo, _f32p), _ptr(vo, _f32p), _ptr(ls, _i64p), _ptr(su, _f32p),
                               _ptr(fi, _i32p), _ptr(fsc, _f32p), _ptr(fg, _i32p))
        if rc != 0:
            raise RuntimeError(f"oracle train failed: {rc}")
        return TrainResult(po, mo, vo, int(ls[0]), su, fi, float(fsc[0]), int(fg[0]))


class ReferenceError_(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Reference:
    """The real reference hot path (oracle/_ref/libbertopt_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_f32_to_f16.argtypes = [_f32p, _u16p, C.c_size_t]
        L.ref_f16_to_f32.argtypes = [_u16p, _f32p, C.c_size_t]
        L.ref_narrow_block.argtypes = [_f32p, _u16p, C.c_size_t]
        L.ref_widen_block.argtypes = [_u16p, _f32p, C.c_size_t]
        L.ref_fnv1a.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.ref_fnv1a.restype = C.c_uint64
        L.ref_ring_chunk_elems.argtypes = [C.c_size_t, C.c_int]
        L.ref_ring_chunk_elems.restype = C.c_size_t
        L.ref_ring_allreduce_bytes.argtypes = [C.c_size_t, C.c_int, C.c_size_t]
        L.ref_ring_allreduce_bytes.restype = C.c_uint64
        L.ref_unscale_gradients.argtypes = [_f32p, C.c_size_t, C.c_float, C.c_int, C.c_char_p, C.c_int]
        L.ref_lamb_step.argtypes = [C.c_int, _i64p, _f32p, _f32p, _f32p, _f32p, _i64p, _f32p,
                                    C.c_char_p, C.c_int]
        L.ref_ring_allreduce.argtypes = [C.c_int, C.c_size_t, C.c_void_p, C.c_int,
                                         C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.ref_bucket_layout.argtypes = [C.POINTER(_Spec), _i32p, C.c_uint64, _i32p, _i64p, _i32p,
                                        _i64p, C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.ref_build_params.argtypes = [C.POINTER(_Spec), C.c_uint64, _f32p]
        L.ref_train.argtypes = [C.POINTER(_Spec), C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                C.c_int, _f32p, C.POINTER(_Scaler), C.c_uint64, C.c_uint32, C.c_int,
                                _i64p, C.c_int, C.c_int, _f32p, _f32p, _f32p, _i64p, _f32p, _i32p,
                                _f32p, _i32p, C.c_char_p, C.c_int, C.POINTER(C.c_double)]
        L.ref_stage_bench.argtypes = [C.c_int, _i64p, _i32p, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.c_char_p, C.c_int, C.c_int]
        self._keep = []

    def stage_bench(self, numels, firsts, world, K, bucket_bytes, f16, groups, warmup, steps,
                    shared_micros=False):
        """Wall seconds per timed step (max over all threads) and rank-0 stage seconds."""
        nm = np.asarray(numels, np.int64)
        fs = np.asarray(firsts, np.int32)
        secs = (C.c_double * steps)()
        stages = (C.c_double * 4)()
        err = C.create_string_buffer(1024)
        rc = self.lib.ref_stage_bench(len(nm), _ptr(nm, _i64p), _ptr(fs, _i32p), world, K,
                                      bucket_bytes, int(f16), groups, warmup, steps, secs, stages,
                                      err, 1024, int(shared_micros))
        self._check(rc, err)
        return list(secs), list(stages)

    def _spec(self, spec):
        names = (C.c_char_p * spec.n_tensors)(*[n.encode() for n in spec.names])
        nd = np.array([len(s) for s in spec.shapes], np.int32)
        dims = np.array([d for s in spec.shapes for d in s] or [0], np.int64)
        init = np.array(spec.init, np.int32)
        fu = np.array(spec.first_use, np.int32)
        self._keep = [names, nd, dims, init, fu]
        return _Spec(spec.n_tensors, names, _ptr(nd, _i32p), _ptr(dims, _i64p), _ptr(init, _i32p),
                     _ptr(fu, _i32p))

    @staticmethod
    def _check(rc, err):
        if rc != 0:
            raise ReferenceError_(rc, err.value.decode(errors="replace"))

    def f32_to_f16(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, np.uint16)
        self.lib.ref_f32_to_f16(_ptr(x, _f32p), _ptr(out, _u16p), x.size)
        return out

    def f16_to_f32(self, h):
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.shape, np.float32)
        self.lib.ref_f16_to_f32(_ptr(h, _u16p), _ptr(out, _f32p), h.size)
        return out

    def narrow_block(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, np.uint16)
        self.lib.ref_narrow_block(_ptr(x, _f32p), _ptr(out, _u16p), x.size)
        return out

    def fnv1a(self, data: bytes, seed: int = 14695981039346656037) -> int:
        return self.lib.ref_fnv1a(data, len(data), seed)

    def unscale_gradients(self, g, scale, enabled=True):
        g = np.ascontiguousarray(g, np.float32).copy()
        err = C.create_string_buffer(512)
        rc = self.lib.ref_unscale_gradients(_ptr(g, _f32p), g.size, scale, int(enabled), err, 512)
        self._check(rc, err)
        return g

    def lamb_step(self, numels, w, g, m, v, step, cfg: LambConfig):
        """In place; returns (status, new_step) like Oracle.lamb_step."""
        nm = np.asarray(numels, np.int64)
        st = np.array([step], np.int64)
        err = C.create_string_buffer(512)
        rc = self.lib.ref_lamb_step(len(numels), _ptr(nm, _i64p), _ptr(w, _f32p), _ptr(g, _f32p),
                                    _ptr(m, _f32p), _ptr(v, _f32p), _ptr(st, _i64p), cfg.arr(),
                                    err, 512)
        return rc, int(st[0])

    def ring_allreduce(self, data: np.ndarray, kind: int = 0):
        d = np.ascontiguousarray(data).copy()
        sent = (C.c_uint64 * d.shape[0])()
        err = C.create_string_buffer(512)
        rc = self.lib.ref_ring_allreduce(d.shape[0], d.shape[1], d.ctypes.data, kind, sent, err, 512)
        self._check(rc, err)
        return d, list(sent)

    def bucket_layout(self, spec, firsts, bucket_bytes):
        T = spec.n_tensors
        s = self._spec(spec)
        fs = np.asarray(firsts, np.int32)
        bo = np.empty(T, np.int32)
        off = np.empty(T, np.int64)
        ro = np.empty(T, np.int32)
        be = np.empty(T, np.int64)
        h = C.c_uint64()
        err = C.create_string_buffer(512)
        nb = self.lib.ref_bucket_layout(C.byref(s), _ptr(fs, _i32p), bucket_bytes, _ptr(bo, _i32p),
                                        _ptr(off, _i64p), _ptr(ro, _i32p), _ptr(be, _i64p),
                                        C.byref(h), err, 512)
        if nb < 0:
            raise ReferenceError_(-nb, err.value.decode())
        return bo, off, ro, be[:nb], h.value

    def build_params(self, spec, seed):
        s = self._spec(spec)
        out = np.empty(spec.param_count(), np.float32)
        self.lib.ref_build_params(C.byref(s), seed, _ptr(out, _f32p))
        return out

    def train(self, spec, init_seed, world, K, bucket_bytes, f16_wire, lamb: LambConfig,
              scaler: ScalerConfig, steps, grad_seed=1, spike_ppm=0, spike_exp=1,
              injections=(), overlap=True, step_seconds=None) -> TrainResult:
        """step_seconds: optional list, filled with rank 0's wall seconds of
        every real train_step call."""
        s = self._spec(spec)
        P = spec.param_count()
        inj = _inj_array(injections)
        po, mo, vo = (np.empty(P, np.float32) for _ in range(3))
        ls = np.zeros(1, np.int64)
        su = np.empty(steps, np.float32)
        fi = np.empty(steps, np.int32)
        fsc = np.empty(1, np.float32)
        fg = np.empty(1, np.int32)
        sc = _scaler(scaler)
        err = C.create_string_buffer(1024)
        secs = (C.c_double * steps)()
        rc = self.lib.ref_train(C.byref(s), init_seed, world, K, bucket_bytes, int(f16_wire),
                                int(overlap), lamb.arr(), C.byref(sc), grad_seed, spike_ppm,
                                spike_exp, _ptr(inj, _i64p), len(injections), steps, _ptr(po, _f32p),
                                _ptr(mo, _f32p), _ptr(vo, _f32p), _ptr(ls, _i64p), _ptr(su, _f32p),
                                _ptr(fi, _i32p), _ptr(fsc, _f32p), _ptr(fg, _i32p), err, 1024,
                                secs)
        self._check(rc, err)
        if step_seconds is not None:
            step_seconds[:] = list(secs)
        return TrainResult(po, mo, vo, int(ls[0]), su, fi, float(fsc[0]), int(fg[0]))


def reference_available() -> bool:
    return os.path.exists(REF_SO)
