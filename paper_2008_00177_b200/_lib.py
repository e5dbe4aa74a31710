"""ctypes binding of ``libbertopt_b200.so`` (include/bertopt_b200.h).

The library is the product: there is no Python or CPU fallback. Importing this
module without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbertopt_b200.so")


class LambConfigC(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float), ("trust_clip", C.c_float)]


class ScalerConfigC(C.Structure):
    _fields_ = [("init_scale", C.c_float), ("growth_factor", C.c_float),
                ("backoff_factor", C.c_float), ("min_scale", C.c_float),
                ("max_scale", C.c_float), ("growth_interval", C.c_int32), ("dynamic", C.c_int32)]


class TrainerConfigC(C.Structure):
    _fields_ = [("lamb", LambConfigC), ("accumulation", C.c_int32), ("bucket_bytes", C.c_uint64),
                ("f16_exchange", C.c_int32), ("reduce_algo", C.c_int32), ("scaler", ScalerConfigC)]


class StepStatusC(C.Structure):
    _fields_ = [("loss_scale", C.c_float), ("good_steps", C.c_int32), ("lamb_step", C.c_int64),
                ("steps", C.c_int64), ("skipped_steps", C.c_int64), ("found_inf", C.c_int32),
                ("reserved", C.c_int32)]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_sz = C.c_size_t

# name -> (restype, argtypes); every symbol include/bertopt_b200.h declares.
SIGNATURES = {
    "bo_abi_version": (_i32, []),
    "bo_status_name": (C.c_char_p, [_i32]),
    "bo_last_error": (C.c_char_p, []),
    "bo_default_config": (None, [C.POINTER(TrainerConfigC)]),
    "bo_bucket_layout": (_i32, [_i32, C.POINTER(_i64), C.POINTER(_i32), _u64, C.POINTER(C.c_char_p),
                                C.POINTER(_i32), C.POINTER(_i64), _i32, _i32, C.POINTER(_i32),
                                C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i32),
                                C.POINTER(_u64)]),
    "bo_shard_ranges": (_i32, [_i32, C.POINTER(_i64), _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "bo_create": (_i32,[C.POINTER(TrainerConfigC), _i32, C.POINTER(_i64), C.POINTER(_i32),
                         C.POINTER(C.c_char_p), C.POINTER(_i32), C.POINTER(_i64), _i32, _i32, _i32,
                         C.POINTER(_vp)]),
    "bo_destroy": (None, [_vp]),
    "bo_layout_num_buckets": (_i32, [_vp]),
    "bo_layout_query": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64)]),
    "bo_layout_hash": (_u64, [_vp]),
    "bo_shard_elems": (_i64, [_vp]),
    "bo_device_bytes": (_u64, [_vp]),
    "bo_comm_unique_id": (_i32, [C.c_char_p]),
    "bo_comm_init": (_i32, [_vp, C.c_char_p]),
    "bo_comm_export": (_i32, [_vp, _vp, C.POINTER(_u64)]),
    "bo_comm_import": (_i32, [_vp, _vp, _u64]),
    "bo_set_watchdog": (_i32, [_vp, C.c_double]),
    "bo_world_init_local": (_i32, [C.POINTER(_vp), _i32]),
    "bo_set_stream": (_i32, [_vp, _vp]),
    "bo_get_stream": (_vp, [_vp]),
    "bo_synchronize": (_i32, [_vp]),
    "bo_wait": (_i32, [_vp, _i64]),
    "bo_load_params": (_i32, [_vp, _vp, _i32]),
    "bo_read_params": (_i32, [_vp, _vp, _i32]),
    "bo_read_moments": (_i32, [_vp, _vp, _vp, _i32]),
    "bo_replica_hash": (_i32, [_vp, _vp]),
    "bo_get_status": (_i32, [_vp, C.POINTER(StepStatusC)]),
    "bo_export_state": (_i32, [_vp, _vp, C.POINTER(_u64)]),
    "bo_import_state": (_i32, [_vp, _vp, _u64]),
    "bo_param_ptr":(_i32, [_vp, _i32, C.POINTER(_vp)]),
    "bo_accumulate": (_i32, [_vp, _i32, C.POINTER(_vp)]),
    "bo_sync_ready": (_i32, [_vp, _i32, C.POINTER(_i32), C.POINTER(_vp)]),
    "bo_train_step": (_i32, [_vp, C.POINTER(_vp)]),
    "bo_params_wait": (_i32, [_vp, _i32, _vp]),
    "bo_param_group": (_i32, [_vp, _i32]),
    "bo_profile_enable": (_i32, [_vp, _i32]),
    "bo_profile_read": (_i32, [_vp, C.POINTER(C.c_double), C.POINTER(_i64), _i32]),
    "bo_launch_count": (_i64, [_vp]),
    "bo_path_flags": (_i32, [_vp]),
    "bo_trace_enable": (_i32, [_vp, _i32]),
    "bo_trace_write": (_i32, [_vp, C.c_char_p]),
    "bo_lamb_step": (_i32, [_i32, C.POINTER(_i64), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                            C.POINTER(_vp), C.POINTER(_i64), C.POINTER(LambConfigC), _vp]),
    "bo_ring_allreduce_f32": (_i32, [_vp, _vp, _sz]),
    "bo_ring_allreduce_f16_wire": (_i32, [_vp, _vp, _sz]),
    "bo_unscale_gradients": (_i32, [_vp, _sz, C.c_float, _i32, _vp]),
    "bo_narrow_f16": (_i32, [_vp, _vp, _sz, _vp]),
    "bo_widen_f16": (_i32, [_vp, _vp, _sz, _vp]),
    "bo_fused_optimizer_step": (_i32, [_i32, C.POINTER(_i64), C.POINTER(_vp), C.POINTER(_vp),
                                       C.POINTER(_vp), C.POINTER(_vp), C.c_float, C.c_float,
                                       C.c_float, C.c_float, C.c_float, _i32, _vp]),
    "bo_f16_round": (_i32, [_vp, _sz, _vp]),
    "bo_scale_loss": (C.c_float, [C.c_float, C.c_float, _i32]),
    "bo_malloc": (_i32, [C.POINTER(_vp), _sz, _i32]),
    "bo_free": (_i32, [_vp]),
    "bo_memcpy": (_i32, [_vp, _vp, _sz, _i32]),
    "bo_synth_grads":(_i32, [_vp, _i64, _i64, _u64, _i32, _i32, _i32, C.c_float, C.c_uint32, _i32, _vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load the library; raise if it has not been built (no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 pipeline has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        lib = load()
        msg = (lib.bo_last_error() or b"").decode(errors="replace")
        raise errors.from_status(status, msg)
