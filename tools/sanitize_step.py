"""Product-path driver for compute-sanitizer (tests/test_gpu_sanitizer.py).

Runs the one-rank pipeline through both step APIs (K bo_accumulate calls and
bo_train_step), plus the operator drop-ins, on ragged tensors whose binary16
gradients each END EXACTLY at the end of their own cudaMalloc allocation
(bo_malloc of numel * 2 bytes, or numel * 2 + 2 with the slot one element
in: the unaligned scalar paths), so that any load past a tensor's last
element is an out-of-bounds access memcheck reports. No torch: only this
library's kernels run under the tool.

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_step.py
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2008_00177_b200 import _lib  # noqa: E402
from paper_2008_00177_b200.model_spec import flat_spec  # noqa: E402
from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig  # noqa: E402

# sizes with every residue mod 4 and 8, a tile boundary (4096) +- 1, a
# zero-element tensor and a multi-tile tensor
SIZES = [1, 2, 3, 5, 7, 13, 4095, 4097, 0, 9001, 64, 12347]


def alloc_grads(lib, K, aligned):
    """K x T device pointers; tensor t of micro k ends at its allocation's end."""
    bufs, ptrs = [], []
    for k in range(K):
        row = []
        for n in SIZES:
            extra = 0 if aligned else 2  # unaligned: the slot starts one binary16 in
            p = C.c_void_p()
            _lib.check(lib.bo_malloc(C.byref(p), n * 2 + extra, 0))
            bufs.append(p)
            row.append((p.value or 0) + extra)
        ptrs.append(row)
    return bufs, ptrs


def fill(lib, ptrs, step, scale):
    off = np.concatenate([[0], np.cumsum(SIZES)[:-1]])
    for k, row in enumerate(ptrs):
        for t, n in enumerate(SIZES):
            if n:
                _lib.check(lib.bo_synth_grads(row[t], int(off[t]), n, 7, 0, step, k, scale, 0, 1, None))


def run(aligned, resident):
    lib = _lib.load()
    K = 3
    spec = flat_spec(SIZES, first_use=list(range(len(SIZES)))[::-1])
    cfg = TrainerConfig(LambConfig(lr=1e-2), K, 8192, False, 0, ScalerConfig(init_scale=1024.0))
    pipe = GradPipeline(spec, cfg)
    P = spec.param_count()
    pipe.load_params(np.linspace(-0.1, 0.1, P, dtype=np.float32))
    bufs, ptrs = alloc_grads(lib, K, aligned)
    for step in range(2):
        fill(lib, ptrs, step, pipe.status().loss_scale)
        if resident:
            pipe.train_step_ptr_array(GradPipeline.make_ptr_array([p for row in ptrs for p in row]))
        else:
            for k in range(K):
                pipe.accumulate_ptr_array(k, GradPipeline.make_ptr_array(ptrs[k]))
        pipe.synchronize()
    st = pipe.status()
    assert st.lamb_step == 2, st
    pipe.close()
    for b in bufs:
        lib.bo_free(b)


def run_operators():
    """bo_lamb_step and the binary16 operators on exact-size allocations."""
    lib = _lib.load()
    T = len(SIZES)
    numels = (C.c_int64 * T)(*SIZES)
    arrs = []
    for _ in range(4):  # w, g, m, v
        row = []
        for n in SIZES:
            p = C.c_void_p()
            _lib.check(lib.bo_malloc(C.byref(p), max(n, 1) * 4, 0))
            host = np.full(max(n, 1), 1e-3, np.float32)
            _lib.check(lib.bo_memcpy(p, host.ctypes.data, max(n, 1) * 4, 0))
            row.append(p.value)
        arrs.append((C.c_void_p * T)(*row))
    step = C.c_int64(0)
    cfg = _lib.LambConfigC(1e-3, 0.9, 0.999, 1e-6, 0.01, 10.0)
    _lib.check(lib.bo_lamb_step(T, numels, arrs[0], arrs[1], arrs[2], arrs[3], C.byref(step),
                                C.byref(cfg), None))
    n = 12347
    src, half = C.c_void_p(), C.c_void_p()
    _lib.check(lib.bo_malloc(C.byref(src), n * 4, 0))
    _lib.check(lib.bo_malloc(C.byref(half), n * 2, 0))
    _lib.check(lib.bo_memcpy(src, np.linspace(-1, 1, n, dtype=np.float32).ctypes.data, n * 4, 0))
    _lib.check(lib.bo_narrow_f16(src, half, n, None))
    _lib.check(lib.bo_widen_f16(half, src, n, None))
    _lib.check(lib.bo_f16_round(src, n, None))
    _lib.check(lib.bo_unscale_gradients(src, n, 1024.0, 1, None))


if __name__ == "__main__":
    for aligned in (True, False):
        for resident in (False, True):
            run(aligned, resident)
    run_operators()
    print("SANITIZE_STEP_OK", flush=True)
