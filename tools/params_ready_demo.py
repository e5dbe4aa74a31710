"""The next step's forward overlapping this step's parameter all-gather
(VERDICT r01 "hide the parameter all-gather"; bo_params_wait).

Every rank pushes its updated shard into every replica group by group in
model (= forward first-use) order and publishes each parameter group as it
lands (k_shard_p2_push). The next forward, emulated by bf16 matmuls on its own
(high-priority) stream with work per parameter group proportional to the
group's size, waits per group instead of for the whole step:

  serial      forward waits for the whole step (event on the step's stream)
  overlapped  forward waits group by group (bo_params_wait)

One iteration = one optimizer step (bo_train_step, BERT-large, K = 4, binary16
ring) followed by the next forward; the next step waits for the forward. Times
are CUDA events, max over ranks. Both pipelines see the same gradients and
must end with bit-identical replicas; the overlapped forward also snapshots
every group's parameters right after its wait and checks them against the
step's final parameters (a gating error would show stale values).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/params_ready_demo.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _Dev:
    """A raw device range as a torch tensor (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="bert-large")
    ap.add_argument("--forward-ms", type=float, default=4.0, help="emulated next forward")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    import numpy as np
    import torch
    import torch.distributed as dist

    from bench import model_spec
    from paper_2008_00177_b200.pipeline import (REDUCE_RING, GradPipeline, LambConfig, ScalerConfig,
                                                TrainerConfig, synth_grads)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    ngpu = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= ngpu:
        raise SystemExit("one GPU per rank")
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("gloo")
    spec = model_spec(args.model)
    P, T, K = spec.param_count(), spec.n_tensors, 4
    cfg = TrainerConfig(LambConfig(lr=1e-4), K, 4 << 20, world > 1, REDUCE_RING,
                        ScalerConfig(init_scale=65536.0, growth_interval=1 << 30))
    w0 = torch.randn(P, device=dev, generator=torch.Generator(device=dev).manual_seed(7)) * 0.02
    s_step = torch.cuda.Stream()
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    s_fwd = torch.cuda.Stream(priority=-1)
    pipes = []
    for _ in range(2):
        p = GradPipeline(spec, cfg, device=local, rank=rank, world=world)
        p.comm_init_torch()
        p.load_params(w0)
        p.set_stream(s_step)
        pipes.append(p)
    del w0
    numels = spec.numels()
    slots, off = [], 0
    for n in numels:
        slots.append(off)
        off += (n + 127) // 128 * 128
    model_off = np.concatenate([[0], np.cumsum(numels)[:-1]])
    bufs = []
    for k in range(K):
        b = torch.empty(off, dtype=torch.int16, device=dev)
        for t, n in enumerate(numels):
            synth_grads(b[slots[t]:slots[t] + n], int(model_off[t]), 1, rank, 0, k, 65536.0)
        bufs.append(b)
    arr = GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for b in bufs for s in slots])

    # parameter groups in forward order, and the emulated forward's work per group
    groups = {}
    for t in range(T):
        groups.setdefault(pipes[1].param_group(t), []).append(t)
    order = sorted(groups)
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    bm = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    c = torch.empty_like(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_fwd):
        for _ in range(3):
            torch.mm(a, bm, out=c)
        e0.record(s_fwd)
        for _ in range(20):
            torch.mm(a, bm, out=c)
        e1.record(s_fwd)
    torch.cuda.synchronize()
    mm_ms = e0.elapsed_time(e1) / 20
    total_mm = max(1, int(round(args.forward_ms / mm_ms)))
    gsize = {g: sum(numels[t] for t in groups[g]) for g in order}
    cum, work = 0, {}
    for g in order:
        before = int(round(cum / P * total_mm))
        cum += gsize[g]
        work[g] = int(round(cum / P * total_mm)) - before
    views = [[torch.as_tensor(_Dev(pipes[i].param_ptr(t), numels[t]), device=dev) if numels[t] else None
              for t in range(T)] for i in range(2)]
    step_done = torch.cuda.Event()
    fwd_done = torch.cuda.Event()

    def iteration(pipe, overlapped, snapshot=None):
        s_step.wait_event(fwd_done)  # the step's gradients come from the previous forward/backward
        pipe.train_step_ptr_array(arr)
        step_done.record(s_step)
        with torch.cuda.stream(s_fwd):
            if not overlapped:
                s_fwd.wait_event(step_done)
            for g in order:
                if overlapped:
                    pipe.params_wait(groups[g][0], s_fwd)
                if snapshot is not None:
                    for t in groups[g]:
                        if numels[t]:
                            snapshot[t].copy_(views[1][t])
                for _ in range(work[g]):
                    torch.mm(a, bm, out=c)
            fwd_done.record(s_fwd)

    def timed(pipe, overlapped):
        for _ in range(args.warmup):
            iteration(pipe, overlapped)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s_step)
        for _ in range(args.steps):
            iteration(pipe, overlapped)
        s_step.wait_event(fwd_done)
        t1.record(s_step)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / args.steps
        if world > 1:
            x = torch.tensor([ms])
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            ms = float(x.item())
        return ms

    fwd_done.record(s_fwd)
    # forward alone and step alone
    def fwd_only():
        with torch.cuda.stream(s_fwd):
            for g in order:
                for _ in range(work[g]):
                    torch.mm(a, bm, out=c)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(s_fwd)
    for _ in range(args.steps):
        fwd_only()
    f1.record(s_fwd)
    torch.cuda.synchronize()
    fwd_ms = f0.elapsed_time(f1) / args.steps
    ser = timed(pipes[0], False)
    ovl = timed(pipes[1], True)
    # one more iteration each, the overlapped one snapshotting every group right after its wait
    snap = [torch.empty(numels[t], device=dev) if numels[t] else None for t in range(T)]
    iteration(pipes[0], False)
    iteration(pipes[1], True, snapshot=snap)
    torch.cuda.synchronize()
    w_ser, w_ovl = pipes[0].read_params(), pipes[1].read_params()
    gated_ok = all(snap[t] is None or torch.equal(snap[t], views[1][t]) for t in range(T))
    same = bool(np.array_equal(w_ser.view(np.uint32), w_ovl.view(np.uint32)))
    ok = torch.tensor([int(same and gated_ok)])
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # the step alone (no forward)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(s_step)
    for _ in range(args.steps):
        pipes[0].train_step_ptr_array(arr)
    s1.record(s_step)
    torch.cuda.synchronize()
    step_ms = s0.elapsed_time(s1) / args.steps
    if world > 1:
        x = torch.tensor([step_ms, fwd_ms])
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        step_ms, fwd_ms = float(x[0]), float(x[1])
    if rank == 0:
        line = {"tool": "params_ready_demo", "world": world, "gpus": ngpu, "model": args.model,
                "param_groups": len(order), "step_ms": round(step_ms, 4),
                "forward_ms": round(fwd_ms, 4),
                "serial_iteration_ms": round(ser, 4), "overlapped_iteration_ms": round(ovl, 4),
                "hidden_ms": round(ser - ovl, 4),
                "exposed_step_ms_serial": round(ser - fwd_ms, 4),
                "exposed_step_ms_overlapped": round(ovl - fwd_ms, 4),
                "replicas_bit_identical_and_gated": bool(ok.item())}
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    for p in pipes:
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for p in pipes:
        p.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
