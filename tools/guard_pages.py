"""Guard-page bounds check of the product kernels (compute-sanitizer is closed
on this pool): every caller-owned tensor the kernels read or write is placed
so that it ENDS exactly at the end of a mapped 2 MiB granule whose successor
granule is reserved but unmapped (CUDA virtual memory management: cuMemCreate
/ cuMemAddressReserve / cuMemMap). A load or store one element past a tensor's
end faults (illegal address) instead of silently reading a neighbour, so a
clean run proves the tail handling of every kernel the run exercises.

Runs the one-rank pipeline through both step APIs (K bo_accumulate calls and
bo_train_step) with aligned and unaligned gradient slots, and the operator
drop-ins, on ragged sizes (every residue mod 4 and 8, tile boundaries +- 1).
The library's own buffers are padded by construction; the caller's are not.

    python tools/guard_pages.py      -> prints GUARD_PAGES_OK
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

from paper_2008_00177_b200 import _lib  # noqa: E402
from paper_2008_00177_b200.model_spec import flat_spec  # noqa: E402
from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig  # noqa: E402

SIZES = [1, 2, 3, 5, 7, 13, 4095, 4097, 0, 9001, 64, 12347]


def _ok(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


class GuardedArena:
    """Tensors ending at a mapped granule's end, the next granule unmapped."""

    def __init__(self, device=0):
        self.dev = device
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device
        self.prop = prop
        self.gran = _ok(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
        self.maps = []

    def alloc_tail(self, nbytes):
        """Device pointer p with [p, p + nbytes) ending at a mapped granule's end."""
        g = self.gran
        size = max(g, (nbytes + g - 1) // g * g)
        va = _ok(cu.cuMemAddressReserve(size + g, g, 0, 0))  # + one unmapped guard granule
        handle = _ok(cu.cuMemCreate(size, self.prop, 0))
        _ok(cu.cuMemMap(va, size, 0, handle, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = self.dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ok(cu.cuMemSetAccess(va, size, [acc], 1))
        self.maps.append((va, size, g, handle))
        return int(va) + size - nbytes

    def close(self):
        for va, size, g, handle in self.maps:
            cu.cuMemUnmap(va, size)
            cu.cuMemRelease(handle)
            cu.cuMemAddressFree(va, size + g)
        self.maps = []


def upload(lib, ptr, arr):
    if arr.nbytes:
        _lib.check(lib.bo_memcpy(C.c_void_p(ptr), arr.ctypes.data, arr.nbytes, 0))


def run_pipeline_case(lib, arena, aligned, resident):
    K = 3
    spec = flat_spec(SIZES, first_use=list(range(len(SIZES)))[::-1])
    cfg = TrainerConfig(LambConfig(lr=1e-2), K, 8192, False, 0, ScalerConfig(init_scale=1024.0))
    pipe = GradPipeline(spec, cfg)
    P = spec.param_count()
    pipe.load_params(np.linspace(-0.1, 0.1, P, dtype=np.float32))
    off = np.concatenate([[0], np.cumsum(SIZES)[:-1]])
    ptrs = []
    for k in range(K):
        row = []
        for n in SIZES:
            if aligned:
                # 16-byte aligned slot (the vector paths): the tensor ends at
                # most 14 bytes before the guard (its last 16-byte group)
                nb = max(16, (n * 2 + 15) // 16 * 16)
                row.append(arena.alloc_tail(nb))
            else:
                # one binary16 into an allocation (the scalar paths): the
                # tensor ends exactly at the guard
                row.append(arena.alloc_tail(n * 2 + 2) + 2)
        ptrs.append(row)
    for step in range(2):
        S = pipe.status().loss_scale
        for k in range(K):
            for t, n in enumerate(SIZES):
                if n:
                    _lib.check(lib.bo_synth_grads(C.c_void_p(ptrs[k][t]), int(off[t]), n, 7, 0, step, k,
                                                  S, 0, 1, None))
        if resident:
            pipe.train_step_ptr_array(GradPipeline.make_ptr_array([p for row in ptrs for p in row]))
        else:
            for k in range(K):
                pipe.accumulate_ptr_array(k, GradPipeline.make_ptr_array(ptrs[k]))
        pipe.synchronize()
    assert pipe.status().lamb_step == 2
    path = pipe.path()
    pipe.close()
    return path


def run_operator_cases(lib, arena):
    T = len(SIZES)
    numels = (C.c_int64 * T)(*SIZES)
    rows = []
    for _ in range(4):  # w, g, m, v: every tensor ends at a guard
        row = []
        for n in SIZES:
            p = arena.alloc_tail(max(n, 1) * 4)
            upload(lib, p, np.full(max(n, 1), 1e-3, np.float32))
            row.append(p + (max(n, 1) - n) * 4)
        rows.append((C.c_void_p * T)(*row))
    step = C.c_int64(0)
    cfg = _lib.LambConfigC(1e-3, 0.9, 0.999, 1e-6, 0.01, 10.0)
    _lib.check(lib.bo_lamb_step(T, numels, rows[0], rows[1], rows[2], rows[3], C.byref(step),
                                C.byref(cfg), None))
    _lib.check(lib.bo_fused_optimizer_step(T, numels, rows[0], rows[1], rows[2], rows[3], 1e-3, 0.9,
                                           0.999, 1e-6, 0.01, 1, None))
    for n in (1, 3, 5, 4097, 12347):
        src = arena.alloc_tail(n * 4)
        half = arena.alloc_tail(n * 2)
        upload(lib, src, np.linspace(-1, 1, n, dtype=np.float32))
        _lib.check(lib.bo_narrow_f16(C.c_void_p(src), C.c_void_p(half), n, None))
        _lib.check(lib.bo_widen_f16(C.c_void_p(half), C.c_void_p(src), n, None))
        _lib.check(lib.bo_f16_round(C.c_void_p(src), n, None))
        _lib.check(lib.bo_unscale_gradients(C.c_void_p(src), n, 1024.0, 1, None))


def main():
    lib = _lib.load()
    p = C.c_void_p()
    _lib.check(lib.bo_malloc(C.byref(p), 16, 0))  # initialises the device's primary context
    _ok(cu.cuInit(0))
    arena = GuardedArena(0)
    paths = []
    for aligned in (True, False):
        for resident in (False, True):
            path = run_pipeline_case(lib, arena, aligned, resident)
            # aligned slots take the fused vector kernels, unaligned the scalar ones
            assert ("one_rank_fused" in path) == aligned, (aligned, path)
            assert ("resident_micros" in path) == (aligned and resident), (aligned, resident, path)
            paths.append(path)
    run_operator_cases(lib, arena)
    _lib.check(lib.bo_free(p))
    arena.close()
    print("paths:", paths)
    print("GUARD_PAGES_OK", flush=True)


if __name__ == "__main__":
    main()
