"""Host-side mirror of the reference hot-path interface over the C ABI.

Names and argument meaning follow the reference (proj/core/include/bertopt):

* ``LambConfig``     — lamb.hpp:30-37
* ``TrainerConfig``  — trainer.hpp:75-85 (hot-path fields) + the dynamic
  loss-scaler extension ``ScalerConfig``
* ``GradPipeline``   — one rank's DistributedTrainer gradient-to-update path
  (trainer.cpp:217-373): ``accumulate(k, grads)`` for each micro-batch; the
  last micro runs finalize → reduce-scatter → LAMB → scaler → all-gather.
* ``lamb_step``, ``ring_allreduce``, ``ring_allreduce_f16_wire``,
  ``unscale_gradients``, ``scale_loss`` — operator-level drop-ins with the
  reference signatures' meaning and error behaviour (errors.py).

Tensors are torch CUDA tensors (torch is the device-memory plumbing only);
all compute runs in libbertopt_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidConfig, ShapeMismatch
from .model_spec import ModelSpec

REDUCE_AUTO, REDUCE_RING, REDUCE_NCCL = 0, 1, 2


@dataclass
class LambConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-6
    weight_decay: float = 0.01
    trust_clip: float = 10.0

    def c(self) -> _lib.LambConfigC:
        return _lib.LambConfigC(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                                self.trust_clip)


@dataclass
class ScalerConfig:
    """Dynamic loss scaler (powers of two). dynamic=0: the reference's static S."""

    init_scale: float = 65536.0
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    min_scale: float = 1.0
    max_scale: float = 16777216.0
    growth_interval: int = 2000
    dynamic: int = 1

    def c(self) -> _lib.ScalerConfigC:
        return _lib.ScalerConfigC(self.init_scale, self.growth_factor, self.backoff_factor,
                                  self.min_scale, self.max_scale, self.growth_interval, self.dynamic)


@dataclass
class TrainerConfig:
    lamb: LambConfig = field(default_factory=LambConfig)
    accumulation: int = 1
    bucket_bytes: int = 4 << 20
    f16_exchange: bool = False
    reduce_algo: int = REDUCE_AUTO
    scaler: ScalerConfig = field(default_factory=ScalerConfig)

    def c(self) -> _lib.TrainerConfigC:
        return _lib.TrainerConfigC(self.lamb.c(), self.accumulation, self.bucket_bytes,
                                   int(self.f16_exchange), self.reduce_algo, self.scaler.c())


@dataclass
class StepStatus:
    loss_scale: float
    good_steps: int
    lamb_step: int
    steps: int
    skipped_steps: int
    found_inf: bool


def _ptr_array(ptrs) -> C.Array:
    return (C.c_void_p * len(ptrs))(*ptrs)


@dataclass
class BucketLayout:
    """``BucketLayout`` (trainer.hpp:59-73) as built by the library (host only)."""

    bucket_of: np.ndarray
    offset_of: np.ndarray
    ready_order: np.ndarray
    bucket_elems: np.ndarray
    hash: int

    @staticmethod
    def build(spec: ModelSpec, bucket_bytes: int, f16_exchange: bool = False,
              accumulation: int = 1) -> "BucketLayout":
        lib = _lib.load()
        T = spec.n_tensors
        numels = np.asarray(spec.numels(), np.int64)
        firsts = np.asarray(spec.first_consumer_ids(), np.int32)
        names = (C.c_char_p * T)(*[n.encode() for n in spec.names])
        ndims = np.asarray([len(s) for s in spec.shapes], np.int32)
        dims = np.asarray([d for s in spec.shapes for d in s] or [0], np.int64)
        bo = np.empty(T, np.int32)
        off = np.empty(T, np.int64)
        ro = np.empty(T, np.int32)
        be = np.empty(T, np.int64)
        nb = C.c_int32()
        h = C.c_uint64()
        i64p, i32p = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
        _lib.check(lib.bo_bucket_layout(T, numels.ctypes.data_as(i64p), firsts.ctypes.data_as(i32p),
                                        bucket_bytes, names, ndims.ctypes.data_as(i32p),
                                        dims.ctypes.data_as(i64p), int(f16_exchange), accumulation,
                                        bo.ctypes.data_as(i32p), off.ctypes.data_as(i64p),
                                        ro.ctypes.data_as(i32p), be.ctypes.data_as(i64p),
                                        C.byref(nb), C.byref(h)))
        return BucketLayout(bo, off, ro, be[:nb.value].copy(), h.value)

    def shard_ranges(self, world: int, rank: int):
        """Bucket-local [lo, hi) this rank owns in every bucket."""
        lib = _lib.load()
        B = len(self.bucket_elems)
        lo = np.empty(B, np.int64)
        hi = np.empty(B, np.int64)
        be = np.ascontiguousarray(self.bucket_elems, np.int64)
        i64p = C.POINTER(C.c_int64)
        _lib.check(lib.bo_shard_ranges(B, be.ctypes.data_as(i64p), world, rank,
                                       lo.ctypes.data_as(i64p), hi.ctypes.data_as(i64p)))
        return lo, hi


class GradPipeline:
    """One rank of the device-resident gradient-to-update pipeline."""

    def __init__(self, spec: ModelSpec, cfg: TrainerConfig, device: int = 0, rank: int = 0,
                 world: int = 1):
        self.lib = _lib.load()
        self.spec = spec
        self.cfg = cfg
        self.rank, self.world, self.device = rank, world, device
        T = spec.n_tensors
        self._numels = np.asarray(spec.numels(), np.int64)
        firsts = np.asarray(spec.first_consumer_ids(), np.int32)
        names = (C.c_char_p * T)(*[n.encode() for n in spec.names])
        ndims = np.asarray([len(s) for s in spec.shapes], np.int32)
        dims = np.asarray([d for s in spec.shapes for d in s], np.int64)
        ctx = C.c_void_p()
        cc = cfg.c()
        _lib.check(self.lib.bo_create(
            C.byref(cc), T, self._numels.ctypes.data_as(C.POINTER(C.c_int64)),
            firsts.ctypes.data_as(C.POINTER(C.c_int32)), names,
            ndims.ctypes.data_as(C.POINTER(C.c_int32)), dims.ctypes.data_as(C.POINTER(C.c_int64)),
            device, rank, world, C.byref(ctx)))
        self.ctx = ctx
        self.P = int(self._numels.sum())

    def close(self) -> None:
        if self.ctx:
            self.lib.bo_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- layout
    @property
    def num_buckets(self) -> int:
        return self.lib.bo_layout_num_buckets(self.ctx)

    def layout(self):
        T, B = self.spec.n_tensors, self.num_buckets
        bo = np.empty(T, np.int32)
        off = np.empty(T, np.int64)
        ro = np.empty(T, np.int32)
        be = np.empty(B, np.int64)
        _lib.check(self.lib.bo_layout_query(self.ctx, bo.ctypes.data_as(C.POINTER(C.c_int32)),
                                            off.ctypes.data_as(C.POINTER(C.c_int64)),
                                            ro.ctypes.data_as(C.POINTER(C.c_int32)),
                                            be.ctypes.data_as(C.POINTER(C.c_int64))))
        return bo, off, ro, be

    def layout_hash(self) -> int:
        return self.lib.bo_layout_hash(self.ctx)

    def shard_elems(self) -> int:
        return self.lib.bo_shard_elems(self.ctx)

    def device_bytes(self) -> int:
        return self.lib.bo_device_bytes(self.ctx)

    # -- comm
    @staticmethod
    def unique_id() -> bytes:
        lib = _lib.load()
        buf = C.create_string_buffer(128)
        _lib.check(lib.bo_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, uid: bytes) -> None:
        if len(uid) != 128:
            raise InvalidConfig("InvalidConfig: NCCL unique id must be 128 bytes")
        _lib.check(self.lib.bo_comm_init(self.ctx, uid))

    def comm_init_torch(self, nccl: bool | None = None) -> None:
        """Initialise the context's peers over an initialised torch.distributed
        group (any backend). By default without NCCL: every rank's
        communication record (bo_comm_export) is all-gathered on the host and
        imported (bo_comm_import) — the default binary16 / fp32 ring step uses
        no collective library, and several ranks may share one GPU. nccl=True
        (or a configuration that needs NCCL: the NCCL reduce-scatter,
        BO_RING_NCCL=1, BO_RING_BARRIER=nccl) exchanges an NCCL id instead and
        calls bo_comm_init. Raises BucketLayoutMismatch when ranks disagree on
        the layout (trainer.cpp:169-183)."""
        if self.world == 1:
            return
        if nccl is None:
            nccl = self.needs_nccl()
        agree_layout(self.layout_hash(), self.device)
        if nccl:
            self.comm_init(broadcast_unique_id(self.device))
        else:
            self.comm_import(all_gather_bytes(self.comm_export()))

    def needs_nccl(self) -> bool:
        """The configuration's step uses NCCL (otherwise IPC + flags only)."""
        import os

        algo = self.cfg.reduce_algo
        if algo == REDUCE_AUTO:
            algo = REDUCE_RING  # the library's AUTO (bo_create)
        return (algo == REDUCE_NCCL or os.environ.get("BO_RING_NCCL", "0") != "0"
                or os.environ.get("BO_RING_BARRIER", "") == "nccl")

    def comm_export(self) -> bytes:
        """This rank's communication record (layout/settings hashes, IPC handles)."""
        n = C.c_uint64()
        _lib.check(self.lib.bo_comm_export(self.ctx, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _lib.check(self.lib.bo_comm_export(self.ctx, buf, C.byref(n)))
        return buf.raw[:n.value]

    def comm_import(self, records: list[bytes]) -> None:
        """All ranks' records, in rank order."""
        if len(records) != self.world or len({len(r) for r in records}) != 1:
            raise InvalidConfig("InvalidConfig: one record per rank of equal size expected")
        blob = b"".join(records)
        _lib.check(self.lib.bo_comm_import(self.ctx, blob, len(records[0])))

    @staticmethod
    def world_init_local(pipes: list["GradPipeline"]) -> None:
        """All ranks of a world in this process, one device, lockstep on one
        stream (bo_world_init_local); then drive each rank from its own thread."""
        lib = _lib.load()
        arr = (C.c_void_p * len(pipes))(*[p.ctx.value for p in pipes])
        _lib.check(lib.bo_world_init_local(arr, len(pipes)))

    def set_watchdog(self, seconds: float) -> None:
        """Bound of the cross-rank waits inside a step (RunConfig::watchdog_s)."""
        _lib.check(self.lib.bo_set_watchdog(self.ctx, float(seconds)))


    # -- streams
    def set_stream(self, stream) -> None:
        handle = None if stream is None else C.c_void_p(int(stream.cuda_stream))
        _lib.check(self.lib.bo_set_stream(self.ctx, handle))

    def stream_handle(self) -> int:
        return int(self.lib.bo_get_stream(self.ctx) or 0)

    def synchronize(self) -> None:
        _lib.check(self.lib.bo_synchronize(self.ctx))

    def wait(self, timeout_ms: int = -1) -> None:
        """Watchdog wait: raises WatchdogTimeout if the queued step has not
        completed within timeout_ms, PeerDisconnected on a communicator
        failure (transport.cpp:113-132)."""
        _lib.check(self.lib.bo_wait(self.ctx, int(timeout_ms)))

    # -- introspection
    PATH_NAMES = {1: "one_rank_fused", 2: "one_rank_staged", 4: "ring_p2p", 8: "ring_sendrecv",
                  16: "last_hop_fused", 32: "nccl_reduce_scatter", 64: "overlap",
                  128: "resident_micros", 256: "ring_push", 512: "lamb_grouped"}

    def path(self) -> list[str]:
        """Implementation the last sync micro ran (BO_PATH_* names)."""
        f = int(self.lib.bo_path_flags(self.ctx))
        return [n for b, n in self.PATH_NAMES.items() if f & b]

    def trace_enable(self, enable: bool = True) -> None:
        """Record the step's event timeline (the reference's EventLog events,
        device-timed) from now on; trace_write() dumps it as JSON lines."""
        _lib.check(self.lib.bo_trace_enable(self.ctx, int(enable)))

    def trace_write(self, path: str) -> None:
        _lib.check(self.lib.bo_trace_write(self.ctx, path.encode()))

    def launch_count(self) -> int:
        return int(self.lib.bo_launch_count(self.ctx))

    # -- state
    def load_params(self, params) -> None:
        """params: flat float32 model-order array (numpy) or CUDA tensor."""
        if isinstance(params, np.ndarray):
            a = np.ascontiguousarray(params, np.float32)
            if a.size != self.P:
                raise ShapeMismatch("ShapeMismatch: parameter count")
            _lib.check(self.lib.bo_load_params(self.ctx, a.ctypes.data, 1))
        else:
            if params.numel() != self.P or not params.is_contiguous():
                raise ShapeMismatch("ShapeMismatch: parameter count")
            _lib.check(self.lib.bo_load_params(self.ctx, params.data_ptr(), 0))

    def read_params(self) -> np.ndarray:
        out = np.empty(self.P, np.float32)
        _lib.check(self.lib.bo_read_params(self.ctx, out.ctypes.data, 1))
        return out

    def replica_hash(self) -> int:
        """bo_replica_hash: the device-side hash of this rank's parameter
        replica (equal across ranks with identical replicas; the per-step
        divergence check of trainer.cpp:442-453)."""
        out = C.c_uint64()
        _lib.check(self.lib.bo_replica_hash(self.ctx, C.byref(out)))
        return int(out.value)

    def read_moments(self, m: np.ndarray | None = None, v: np.ndarray | None = None):
        m = np.zeros(self.P, np.float32) if m is None else m
        v = np.zeros(self.P, np.float32) if v is None else v
        _lib.check(self.lib.bo_read_moments(self.ctx, m.ctypes.data, v.ctypes.data, 1))
        return m, v

    def status(self) -> StepStatus:
        st = _lib.StepStatusC()
        _lib.check(self.lib.bo_get_status(self.ctx, C.byref(st)))
        return StepStatus(st.loss_scale, st.good_steps, st.lamb_step, st.steps, st.skipped_steps,
                          bool(st.found_inf))

    def export_state(self) -> bytes:
        """Checkpoint of this rank's device state (params, owned moments, step, scaler)."""
        n = C.c_uint64()
        _lib.check(self.lib.bo_export_state(self.ctx, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _lib.check(self.lib.bo_export_state(self.ctx, buf, C.byref(n)))
        return buf.raw[:n.value]

    def import_state(self, blob: bytes) -> None:
        _lib.check(self.lib.bo_import_state(self.ctx, blob, len(blob)))

    def param_ptr(self, t: int) -> int:
        p = C.c_void_p()
        _lib.check(self.lib.bo_param_ptr(self.ctx, t, C.byref(p)))
        return p.value

    # -- hot path
    # Stream contract (include/bertopt_b200.h "streams"): the library runs on
    # the context stream and does not synchronise with other streams. When the
    # gradients are passed as torch tensors, the wrapper orders the context
    # stream after torch's current stream (which produced them) and marks the
    # tensors as used on the context stream, so the caching allocator cannot
    # hand their memory out while the step still reads it. Raw pointers (ints,
    # prebuilt pointer arrays) are the caller's responsibility.
    def _order_after_producer(self, tensors) -> None:
        ts = [t for t in tensors if not isinstance(t, int)]
        if not ts:
            return
        import torch

        ctx_stream = torch.cuda.ExternalStream(self.stream_handle(), device=ts[0].device)
        producer = torch.cuda.current_stream(ts[0].device)
        if producer.cuda_stream != ctx_stream.cuda_stream:
            ctx_stream.wait_stream(producer)
            for t in ts:
                t.record_stream(ctx_stream)

    def accumulate(self, micro: int, grads) -> None:
        """grads: per-tensor device pointers (ints) or fp16/int16 CUDA tensors."""
        if len(grads) != self.spec.n_tensors:
            raise ShapeMismatch(f"ShapeMismatch: {len(grads)} gradients for "
                                f"{self.spec.n_tensors} parameters")
        self._order_after_producer(grads)
        ptrs = [g if isinstance(g, int) else g.data_ptr() for g in grads]
        _lib.check(self.lib.bo_accumulate(self.ctx, micro, _ptr_array(ptrs)))

    def accumulate_ptr_array(self, micro: int, arr) -> None:
        """Fast path: a prebuilt ctypes pointer array (see make_ptr_array)."""
        _lib.check(self.lib.bo_accumulate(self.ctx, micro, arr))

    @staticmethod
    def make_ptr_array(ptrs) -> C.Array:
        return _ptr_array(ptrs)

    def sync_ready(self, tensors, grads) -> None:
        """Overlapped sync micro (TrainerConfig.overlap): deliver the sync
        micro's gradients of `tensors` (indices) as they become final; buckets
        are reduced in layout order as soon as their communication group is
        complete; the call delivering the last tensor finishes the step."""
        tensors = [int(t) for t in tensors]
        if len(tensors) != len(grads):
            raise ShapeMismatch("ShapeMismatch: tensors and grads differ in length")
        self._order_after_producer(grads)
        ptrs = [g if isinstance(g, int) else g.data_ptr() for g in grads]
        ids = (C.c_int32 * max(1, len(tensors)))(*tensors)
        _lib.check(self.lib.bo_sync_ready(self.ctx, len(tensors), ids, _ptr_array(ptrs)))

    def ready_order(self) -> list[int]:
        """Tensor indices in gradient-ready order (BucketLayout::ready_order)."""
        return [int(t) for t in self.layout()[2]]

    def train_step(self, micro_grads) -> None:
        """All K micro-batches of one optimizer step (DistributedTrainer::train_step,
        trainer.cpp:217-373): micro_grads[k][p] is micro k's gradient of tensor p
        (device pointer or CUDA tensor), resident until the step has run."""
        K = self.cfg.accumulation
        if len(micro_grads) != K:
            raise InvalidConfig("InvalidConfig: train_step expects exactly K micro batches")
        ptrs = []
        for g in micro_grads:
            if len(g) != self.spec.n_tensors:
                raise ShapeMismatch(f"ShapeMismatch: {len(g)} gradients for "
                                    f"{self.spec.n_tensors} parameters")
            self._order_after_producer(g)
            ptrs += [x if isinstance(x, int) else x.data_ptr() for x in g]
        _lib.check(self.lib.bo_train_step(self.ctx, _ptr_array(ptrs)))

    def params_wait(self, tensor: int, stream=None) -> None:
        """Order `stream` (torch stream; default: torch's current stream)
        after the arrival of `tensor`'s parameter group from the most recent
        step (the next forward overlapping the parameter all-gather)."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream()
        _lib.check(self.lib.bo_params_wait(self.ctx, int(tensor), C.c_void_p(int(s.cuda_stream))))

    def param_group(self, tensor: int) -> int:
        return int(self.lib.bo_param_group(self.ctx, int(tensor)))

    def train_step_ptr_array(self, arr) -> None:
        """Fast path: a prebuilt ctypes array of the K x T pointers (make_ptr_array)."""
        _lib.check(self.lib.bo_train_step(self.ctx, arr))


# ---------------------------------------------------------------- operators
def _stream(stream) -> C.c_void_p:
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return C.c_void_p(int(stream.cuda_stream))


def lamb_step(params, grads, state: dict, cfg: LambConfig, stream=None) -> None:
    """``lamb_step(params, grads, state, cfg)`` (lamb.hpp:47-48) on CUDA fp32 tensors.

    ``state`` mirrors LambState: {'m': [...], 'v': [...], 'step': int}; m/v are
    created lazily as zeros (lamb.cpp:30-35). Raises ShapeMismatch /
    NonFiniteGradient like the reference (after the same partial update).
    """
    import torch

    lib = _lib.load()
    if len(grads) != len(params):
        raise ShapeMismatch(f"ShapeMismatch: lamb_step: {len(grads)} gradients for "
                            f"{len(params)} parameters")
    if not state.get("m"):
        state["m"] = [torch.zeros_like(p) for p in params]
        state["v"] = [torch.zeros_like(p) for p in params]
        state.setdefault("step", 0)
    if len(state["m"]) != len(params) or len(state["v"]) != len(params):
        raise ShapeMismatch("ShapeMismatch: lamb_step: optimizer state layout mismatch")
    for i, (p, g) in enumerate(zip(params, grads)):
        if g.shape != p.shape:
            raise ShapeMismatch(f"ShapeMismatch: lamb_step: gradient shape mismatch at tensor {i}")
    n = len(params)
    numels = (C.c_int64 * n)(*[p.numel() for p in params])
    step = C.c_int64(state["step"])
    st = lib.bo_lamb_step(n, numels, _ptr_array([p.data_ptr() for p in params]),
                          _ptr_array([g.data_ptr() for g in grads]),
                          _ptr_array([t.data_ptr() for t in state["m"]]),
                          _ptr_array([t.data_ptr() for t in state["v"]]), C.byref(step),
                          C.byref(cfg.c()), _stream(stream))
    state["step"] = step.value
    _lib.check(st)


def fused_optimizer_step(params, grads, m, v, lr: float, beta1: float, beta2: float, eps: float,
                         weight_decay: float, step: int, stream=None) -> None:
    """The paper's fused Adam-form optimizer kernel, ``run_fused_kernel(
    fused_optimizer_step(lr, beta1, beta2, eps, weight_decay, step), {w, g, m, v})``
    (graph.cpp:458-487), in place on lists of contiguous CUDA fp32 tensors."""
    lib = _lib.load()
    n = len(params)
    if not (len(grads) == len(m) == len(v) == n):
        raise ShapeMismatch("ShapeMismatch: fused_optimizer_step expects 4 equal-length lists")
    for i in range(n):
        if not (params[i].shape == grads[i].shape == m[i].shape == v[i].shape):
            raise ShapeMismatch(f"ShapeMismatch: fused_optimizer_step: shapes differ at tensor {i}")
    numels = (C.c_int64 * max(n, 1))(*[p.numel() for p in params])
    _lib.check(lib.bo_fused_optimizer_step(
        n, numels, _ptr_array([t.data_ptr() for t in params]), _ptr_array([t.data_ptr() for t in grads]),
        _ptr_array([t.data_ptr() for t in m]), _ptr_array([t.data_ptr() for t in v]), lr, beta1, beta2,
        eps, weight_decay, step, _stream(stream)))


def f16_round(x, stream=None) -> None:
    """In-place binary16 round trip of a contiguous CUDA fp32 tensor (the AMP
    cast, Tape::cast -> quantize_inplace, ops.cpp:655-668)."""
    lib = _lib.load()
    _lib.check(lib.bo_f16_round(x.data_ptr(), x.numel(), _stream(stream)))


def unscale_gradients(grads, scale: float, enabled: bool = True, stream=None) -> None:
    """In place on a contiguous CUDA fp32 tensor (half.cpp:105-115)."""
    lib = _lib.load()
    _lib.check(lib.bo_unscale_gradients(grads.data_ptr(), grads.numel(), scale, int(enabled),
                                        _stream(stream)))


def scale_loss(loss: float, scale: float, enabled: bool = True) -> float:
    return _lib.load().bo_scale_loss(loss, scale, int(enabled))


def narrow_f16(src, dst, stream=None) -> None:
    _lib.check(_lib.load().bo_narrow_f16(src.data_ptr(), dst.data_ptr(), src.numel(),
                                         _stream(stream)))


def widen_f16(src, dst, stream=None) -> None:
    _lib.check(_lib.load().bo_widen_f16(src.data_ptr(), dst.data_ptr(), src.numel(),
                                        _stream(stream)))


def ring_allreduce(pipe: GradPipeline, data) -> None:
    """ring_allreduce<float> over pipe's communicator, in place (collective.hpp:104-107)."""
    _lib.check(pipe.lib.bo_ring_allreduce_f32(pipe.ctx, data.data_ptr(), data.numel()))


def ring_allreduce_f16_wire(pipe: GradPipeline, data) -> None:
    """ring_allreduce_f16_wire (collective.hpp:113-114), in place."""
    _lib.check(pipe.lib.bo_ring_allreduce_f16_wire(pipe.ctx, data.data_ptr(), data.numel()))


def synth_grads(dst, flat_begin: int, seed: int, rank: int, step: int, micro: int, scale: float,
                spike_ppm: int = 0, spike_exp: int = 1, stream=None) -> None:
    """Fill an int16/fp16 CUDA tensor with the synthetic spec's binary16 bits."""
    _lib.check(_lib.load().bo_synth_grads(dst.data_ptr(), flat_begin, dst.numel(), seed, rank, step,
                                          micro, scale, spike_ppm, spike_exp, _stream(stream)))


def _dist_device(device: int):
    import torch
    import torch.distributed as dist

    return torch.device(f"cuda:{device}") if dist.get_backend() == "nccl" else torch.device("cpu")


def broadcast_unique_id(device: int = 0) -> bytes:
    """Rank 0 creates the 128-byte NCCL id; torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist

    buf = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank() == 0:
        buf[:] = torch.frombuffer(bytearray(GradPipeline.unique_id()), dtype=torch.uint8)
    buf = buf.to(_dist_device(device))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def all_gather_bytes(mine: bytes) -> list[bytes]:
    """Every rank's byte string, in rank order, over torch.distributed."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, mine)
    return [bytes(x) for x in out]


def agree_layout(layout_hash: int, device: int = 0) -> None:
    """All ranks must hold the same salted layout hash (trainer.cpp:169-183);
    raises BucketLayoutMismatch otherwise."""
    import torch
    import torch.distributed as dist

    from .errors import BucketLayoutMismatch

    mine = torch.tensor([layout_hash - (1 << 64) if layout_hash >= 1 << 63 else layout_hash],
                        dtype=torch.int64, device=_dist_device(device))
    allh = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(allh, mine)
    if any(int(h.item()) != int(mine.item()) for h in allh):
        raise BucketLayoutMismatch(f"BucketLayoutMismatch: rank {dist.get_rank()} bucket layout "
                                   "disagrees with peers")
