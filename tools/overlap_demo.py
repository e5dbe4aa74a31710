"""Bucket-level overlap of the reduce-scatter with backward (SURVEY §8(f)
rank 1; the reference's TrainerConfig::overlap, trainer.cpp:247-348).

The sync micro's backward pass is emulated by bf16 matmuls on the pipeline
stream, issued in gradient-ready order, one bucket at a time (work per bucket
proportional to its element count). Two pipelines start from the same
weights and see the same gradients:

  serialized  all backward work, then bo_accumulate(K-1)      (overlap off)
  overlapped  after each bucket's work, bo_sync_ready(bucket)  (overlap on)

Step times are CUDA events on the pipeline stream, max over ranks; the final
parameters of the two pipelines must be bit-identical (the reference's own
overlap on/off test, test_collective.cpp:817-912).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/overlap_demo.py --gpus N
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="bert-large")
    ap.add_argument("--backward-ms", type=float, default=12.0, help="emulated backward per step")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
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
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(dev))
    spec = model_spec(args.model)
    P = spec.param_count()
    cfg = TrainerConfig(LambConfig(lr=1e-4), 1, 4 << 20, world > 1, REDUCE_RING,
                        ScalerConfig(init_scale=65536.0, growth_interval=1 << 30))
    w0 = torch.randn(P, device=dev, generator=torch.Generator(device=dev).manual_seed(7)) * 0.02
    stream = torch.cuda.Stream()
    pipes = []
    for _ in range(2):
        p = GradPipeline(spec, cfg, device=local, rank=rank, world=world)
        if world > 1:
            p.comm_init_torch()
        p.load_params(w0)
        p.set_stream(stream)
        pipes.append(p)
    serial, overlapped = pipes

    numels = spec.numels()
    slots, off = [], 0
    for n in numels:
        slots.append(off)
        off += (n + 127) // 128 * 128
    model_off = np.concatenate([[0], np.cumsum(numels)[:-1]])
    buf = torch.empty(off, dtype=torch.int16, device=dev)
    for t, n in enumerate(numels):
        synth_grads(buf[slots[t]:slots[t] + n], int(model_off[t]), 1, rank, 0, 0, 65536.0)
    ptrs = [buf.data_ptr() + 2 * s for s in slots]
    ptr_array = GradPipeline.make_ptr_array(ptrs)

    bucket_of, _, ready, bucket_elems = serial.layout()
    buckets = [[] for _ in range(len(bucket_elems))]
    for t in ready:
        buckets[int(bucket_of[t])].append(int(t))

    # emulated backward: 4096^3 bf16 matmuls (~0.1 ms each), split by bucket size
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    b = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    c = torch.empty_like(a)
    with torch.cuda.stream(stream):
        for _ in range(3):
            torch.mm(a, b, out=c)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(20):
            torch.mm(a, b, out=c)
        ev1.record(stream)
    torch.cuda.synchronize()
    mm_ms = ev0.elapsed_time(ev1) / 20
    total_mm = max(1, int(round(args.backward_ms / mm_ms)))
    cum, work = 0, []
    for be in bucket_elems:
        before = int(round(cum / P * total_mm))
        cum += int(be)
        work.append(int(round(cum / P * total_mm)) - before)

    def backward_bucket(j):
        for _ in range(work[j]):
            torch.mm(a, b, out=c)

    def step_backward_only():
        for j in range(len(buckets)):
            backward_bucket(j)

    def step_serial():
        step_backward_only()
        serial.accumulate_ptr_array(0, ptr_array)

    def step_overlap():
        for j, ts in enumerate(buckets):
            backward_bucket(j)
            overlapped.sync_ready(ts, [ptrs[t] for t in ts])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            x = torch.tensor([ms], device=dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            ms = float(x.item())
        return ms

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step_serial()
            step_overlap()
    t_bwd = timed(step_backward_only, args.steps)
    t_ser = timed(step_serial, args.steps)
    t_ovl = timed(step_overlap, args.steps)
    barrier()
    same = bool(np.array_equal(serial.read_params().view(np.uint32),
                               overlapped.read_params().view(np.uint32)))
    st0, st1 = serial.status(), overlapped.status()
    same = same and st0.lamb_step == st1.lamb_step and st0.loss_scale == st1.loss_scale
    if world > 1:
        x = torch.tensor([1 if same else 0], device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MIN)
        same = bool(x.item())
    if rank == 0:
        out = {"n_gpus": world, "model": args.model, "params": P, "buckets": len(buckets),
               "comm_groups_env": os.environ.get("BO_COMM_GROUP_ELEMS", "default (16Mi elements)"),
               "backward_ms": round(t_bwd, 3), "serialized_step_ms": round(t_ser, 3),
               "overlapped_step_ms": round(t_ovl, 3),
               "exposed_sync_ms_serialized": round(t_ser - t_bwd, 3),
               "exposed_sync_ms_overlapped": round(t_ovl - t_bwd, 3),
               "path_overlapped": overlapped.path(), "bit_identical": same}
        os.write(json_fd, (json.dumps(out) + "\n").encode())
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
