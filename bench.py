#!/usr/bin/env python
"""BERT-large gradient-to-update step on B200: accumulate -> unscale/overflow
-> reduce-scatter -> sharded LAMB -> loss-scaler -> all-gather.

One JSON line on rank 0:
  value       = world * P / step_time  (gradient-params/s; every rank consumes
                a full P-parameter gradient of K micro-batches per step)
  ms_per_step = device time of one optimizer step (CUDA events, max over ranks)
  e2e         = the same metric through the public API with the K micro-batch
                fp16 gradients copied from pinned host memory every step and
                the step status read back
  roofline    = dominant kernel's algorithmic bytes / its average duration
  step_roofline = SURVEY §8(d) stage-sum roofline of the whole step
  cpu_baseline  = the reference's own CPU hot path (oracle/_ref) on this host

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under
torch.distributed.run (one process per GPU). --impl reference times the
reference CPU implementation instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BERT-large optimizer step params/sec"
UNIT = "params/s"

# Algorithmic HBM bytes per element of each stage.
BYTES_ACCUMULATE_FIRST = 2 + 4          # read fp16, write fp32 acc
BYTES_ACCUMULATE = 2 + 4 + 4            # read fp16 + acc, write acc
BYTES_FINALIZE = 2 + 4 + 4              # read fp16 + acc, write fusion buffer (fp32)
BYTES_FINALIZE_K1 = 2 + 4
BYTES_LAMB_NORMS = 4 * 4                # read g, w, m, v
BYTES_LAMB_UPDATE = 4 * 4 + 3 * 4       # read g, w, m, v; write w, m, v
# one rank, k_lamb_p1 (read h, acc, w, m, v; write m', v', u) + k_lamb_p2 (read w, u; write w)
BYTES_LAMB_FUSED = (2 + 4 + 3 * 4 + 3 * 4) + (2 * 4 + 4)

# index = BO_STAGE_* in include/bertopt_b200.h
STAGES = ["accumulate", "finalize", "reduce", "lamb_norms", "trust", "lamb_update", "allgather",
          "hop_kernels", "reserved"]

MODELS = {"bert-large": "BERT_LARGE", "bert-large-128": "BERT_LARGE_PHASE1", "bert-base": "BERT_BASE",
          "bert-tiny": "BERT_TINY"}

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x20: "sync_boost", 0x40: "sw_thermal_slowdown",
           0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown",
           0x200: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="bert-large", choices=sorted(MODELS))
    ap.add_argument("--accumulation", type=int, default=4)
    ap.add_argument("--bucket-mb", type=float, default=4.0)
    ap.add_argument("--wire", default="f16", choices=["f16", "f32"])
    ap.add_argument("--algo", default="auto", choices=["auto", "ring", "nccl"])
    ap.add_argument("--api", default="train_step", choices=["train_step", "accumulate"],
                    help="train_step: one bo_train_step per step (all K micros resident); "
                         "accumulate: K bo_accumulate calls per step")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e: copy each step's inputs, then compute (no prefetch of the next step)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def model_spec(name):
    from paper_2008_00177_b200 import model_spec as ms

    return ms.bert_spec(getattr(ms, MODELS[name]))


def cpu_sample(spec):
    """Fallback sample when the host cannot hold the full workload: layer0 plus the heads."""
    idx = [i for i, n in enumerate(spec.names)
           if n.startswith("layer0.") or n.startswith(("mlm.transform", "mlm.ln", "pooler.", "nsp."))]
    numels = [spec.numels()[i] for i in idx]
    firsts = [spec.first_consumer_ids()[i] for i in idx]
    return numels, firsts, f"{len(idx)} BERT tensors (layer0 + MLM/pooler/NSP heads), {sum(numels)} params"


def host_bytes_needed(P, world, K, shared):
    """Host memory of the reference stage bench: per rank params, accumulator,
    fusion buckets, unpacked gradients, LAMB m and v (6 x 4 B x P), plus the K
    fp32 micro-batch gradient sets (per rank, or once when shared)."""
    return world * 6 * 4 * P + (1 if shared else world) * K * 4 * P


def run_cpu_reference(spec, world, K, bucket_bytes, f16, warmup, steps):
    """The reference's own CPU hot path (oracle/_ref: the real ring_allreduce* over
    InProcHub threads and the real lamb_step, with trainer.cpp's accumulate /
    flatten / unpack loops) on the SAME workload as the GPU arm: all tensors,
    P parameters, one rank thread per rank (the reference has no intra-rank
    threading, so N ranks use N cores), best of `steps` timed steps
    (BASELINE.md §4). Falls back to a sample only when the host cannot hold
    the full workload (reported in `sample` and `same_config`)."""
    from oracle import oracle as orc

    if not orc.reference_available():
        raise RuntimeError("oracle/_ref missing: build it with __graft_entry__.build()")
    ref = orc.Reference()
    numels, firsts = spec.numels(), spec.first_consumer_ids()
    P = sum(numels)
    shared = world > 1
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = None
    same = avail is None or host_bytes_needed(P, world, K, shared) < 0.8 * avail
    if same:
        sample = (f"full workload: {len(numels)} tensors, {P} params, {world} rank thread(s)"
                  + (" (the K fp32 micro-batch sets shared read-only by the rank threads)"
                     if shared else ""))
    else:
        numels, firsts, sample = cpu_sample(spec)
        sample += f" (host memory {avail / 2**30:.0f} GiB cannot hold the full workload)"
    secs, stages = ref.stage_bench(numels, firsts, world, K, bucket_bytes, f16, 1, warmup, steps,
                                   shared_micros=shared)
    t = min(secs)
    Ps = sum(numels)
    return {"value": world * Ps / t, "unit": UNIT, "cores": world, "kind": "reference",
            "same_config": same, "ms_per_step": round(t * 1e3, 1),
            "sample": f"{sample}; K={K}, best of {steps} step(s) after {warmup} warm-up "
                      f"({t * 1e3:.0f} ms/step)",
            "cpu": cpu_model(),
            "stage_seconds_rank0": dict(zip(["accumulate", "flatten", "reduce", "lamb"],
                                            [x / max(steps, 1) for x in stages]))}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return f"{ln.split(':', 1)[1].strip()} x {os.cpu_count()}"
    except OSError:
        pass
    return f"{os.cpu_count()} cpus"


def real_train_step_seconds(spec, K, bucket_bytes):
    """Cross-check: one step of the REAL
    DistributedTrainer::train_step (world 1, synthetic forward shim) on the full
    workload; rank 0's wall seconds of the train_step call."""
    from oracle import oracle as orc

    ref = orc.Reference()
    secs = [0.0]
    ref.train(spec, 1, 1, K, bucket_bytes, False, orc.LambConfig(lr=1e-4),
              orc.ScalerConfig(init_scale=65536.0, growth_interval=1 << 30), 1, step_seconds=secs)
    return secs[0]


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, gpus):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in gpus]
            self.max_mhz = max(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                               for h in self.handles)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.ok = False

    def _poll(self):
        nv = self.nv
        while True:
            for h in self.handles:
                try:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                except Exception:  # noqa: BLE001
                    pass
            if self._stop.wait(0.01):
                break

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for b, n in REASONS.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def traffic_from_profiles(kernel):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:  # noqa: BLE001
        return None


def max_over_ranks(x, world, local, emulated):
    """The max of a per-rank time over all ranks (the slowest rank bounds the step)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device="cpu" if emulated else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main_b200(args):
    # Libraries print to stdout (NCCL's version banner); the contract is ONE
    # JSON line there, so everything else goes to stderr.
    json_fd = os.dup(1)
    os.dup2(2, 1)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2008_00177_b200.pipeline import (REDUCE_AUTO, REDUCE_NCCL, REDUCE_RING, GradPipeline,
                                                LambConfig, ScalerConfig, TrainerConfig, synth_grads)

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ngpu = torch.cuda.device_count()
    # one rank per GPU: ranks must never share a device (their flag-spinning
    # kernels must run concurrently); worlds larger than the box run through
    # tools/world_emu.py (all ranks in one process, lockstep on one stream)
    if local >= ngpu:
        raise SystemExit(f"rank {rank}: {world} ranks need {world} GPUs ({ngpu} visible)")
    emulated = False
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    K = args.accumulation
    spec = model_spec(args.model)
    P = spec.param_count()
    f16 = args.wire == "f16" and world > 1
    algo = {"auto": REDUCE_AUTO, "ring": REDUCE_RING, "nccl": REDUCE_NCCL}[args.algo]
    bucket_bytes = int(args.bucket_mb * (1 << 20))
    cfg = TrainerConfig(LambConfig(lr=1e-4), K, bucket_bytes, f16, algo,
                        ScalerConfig(init_scale=65536.0, growth_interval=1 << 30))
    pipe = GradPipeline(spec, cfg, device=local, rank=rank, world=world)
    if world > 1:
        pipe.comm_init_torch()
    # random-init weights of the BERT-large architecture (synthetic)
    gen = torch.Generator(device=f"cuda:{local}").manual_seed(1234 + rank * 0)
    w0 = torch.randn(P, device=f"cuda:{local}", generator=gen) * 0.02
    pipe.load_params(w0)
    del w0

    # K micro-batches of fp16 gradients, resident in HBM (per-tensor 256 B slots)
    numels = spec.numels()
    slots, off = [], 0
    for n in numels:
        slots.append(off)
        off += (n + 127) // 128 * 128
    total = off
    model_off = np.concatenate([[0], np.cumsum(numels)[:-1]])
    S0 = pipe.status().loss_scale
    bufs = []
    for k in range(K):
        b = torch.empty(total, dtype=torch.int16, device=f"cuda:{local}")
        for t, n in enumerate(numels):
            synth_grads(b[slots[t]:slots[t] + n], int(model_off[t]), 1, rank, 0, k, S0)
        bufs.append(b)
    ptr_arrays = [GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for s in slots]) for b in bufs]
    all_ptrs = GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for b in bufs for s in slots])
    torch.cuda.synchronize()

    # the pipeline runs on a torch-owned stream (torch's allocators record on it)
    stream = torch.cuda.Stream()
    pipe.set_stream(stream)

    def step_per_micro():
        for k in range(K):
            pipe.accumulate_ptr_array(k, ptr_arrays[k])

    def step_train():
        pipe.train_step_ptr_array(all_ptrs)

    step = step_train if args.api == "train_step" else step_per_micro

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = pipe.lib.bo_launch_count(pipe.ctx)
    gpus = list(range(min(world, ngpu))) if rank == 0 else []
    sampler = ClockSampler(gpus) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    if sampler:
        sampler.__enter__()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    if sampler:
        sampler.__exit__()
    ms = e0.elapsed_time(e1) / args.steps
    launches = pipe.lib.bo_launch_count(pipe.ctx) - launches0
    ms = max_over_ranks(ms, world, local, emulated)
    st = pipe.status()
    assert st.found_inf is False and st.skipped_steps == 0, "synthetic bench overflowed"

    # stage profile: an identical pass with CUDA events around every stage
    pipe.lib.bo_profile_enable(pipe.ctx, 1)
    stage_ms = (C.c_double * len(STAGES))()
    stage_n = (C.c_int64 * len(STAGES))()
    pipe.lib.bo_profile_read(pipe.ctx, stage_ms, stage_n, 1)
    barrier()
    for _ in range(args.steps):
        step()
    barrier()
    pipe.lib.bo_profile_read(pipe.ctx, stage_ms, stage_n, 1)
    pipe.lib.bo_profile_enable(pipe.ctx, 0)
    S_shard = pipe.shard_elems()
    hbm, peak_kind = peaks()
    E = 2 if f16 else 4
    path = pipe.path()
    fused_last = "last_hop_fused" in path
    resident = "resident_micros" in path
    # the sync gradient's source per element: the K resident micros (2K B,
    # bo_train_step) or the live micro + the fp32 accumulator (2 + 4 B)
    xb = 2 * K if resident else (6 if K > 1 else 2)
    # algorithmic bytes per launch of each stage (HBM) / per rank (NVLink)
    hbm_bytes = {
        "accumulate": (BYTES_ACCUMULATE_FIRST + BYTES_ACCUMULATE * (K - 2)) * P / max(K - 1, 1),
        # (resident micros, NCCL wire: the K micros read, the fp32 fusion buffer written)
        "finalize": ((2 * K + 4) if resident else (BYTES_FINALIZE if K > 1 else BYTES_FINALIZE_K1)) * P,
        # LAMB phase 1: one rank k_lamb_p1 (the gradient source xb + w, m, v
        # read; m', v', u written); world > 1 k_p1w (reduced wire E or, with
        # the last ring hop fused in, xb with the wire over NVLink; + wsh, m, v
        # read; m', v', u written); phase 2: k_lamb_p2 / k_shard_p2_push (w, u
        # read; w written)
        "lamb_norms": ((xb + 24) if world == 1 else ((xb if fused_last else E) + 24)) * S_shard,
        "lamb_update": 12 * S_shard,
        # one ring hop kernel (nested in "reduce"): the gradient source of one
        # chunk of every bucket, wire in and out
        "hop_kernels": (xb + 2 * E) * S_shard,
    }
    # NVLink bytes sent per rank: ring reduce-scatter; the parameter push
    # (k_shard_p2_push stores every updated element into the N-1 other replicas)
    nvl_bytes = {"reduce": (world - 1) / world * E * P, "lamb_update": (world - 1) * 4 * S_shard}
    grouped = "lamb_grouped" in path
    if grouped:
        # grouped LAMB (default at world >= 4): one bracket holds phase 1, the
        # per-group trust ratios and the posted parameter push that overlaps
        # the next group's phase 1 — its bytes are both stages'
        hbm_bytes["lamb_norms"] += hbm_bytes["lamb_update"]
        nvl_bytes["lamb_norms"] = nvl_bytes["lamb_update"]
    if fused_last and "ring_push" not in path:
        # pull form: the fused last hop reads the left neighbour's partial over
        # NVLink (push form: it was pushed here by the previous hop; local read)
        nvl_bytes["lamb_norms"] = nvl_bytes.get("lamb_norms", 0) + E * S_shard
    stages = {}
    for i, name in enumerate(STAGES):
        if stage_n[i] == 0:
            continue
        avg = stage_ms[i] / stage_n[i]
        entry = {"ms": round(avg, 5), "launches_per_step": round(stage_n[i] / args.steps, 2)}
        if name in hbm_bytes:
            nbytes = hbm_bytes[name]
            gbs = nbytes / (avg * 1e-3) / 1e9
            entry.update({"bytes": int(nbytes), "GB/s": round(gbs, 1), "frac": round(gbs / hbm, 4)})
        if name in nvl_bytes and world > 1:
            nbytes = nvl_bytes[name]
            gbs = nbytes / (avg * 1e-3) / 1e9
            entry.update({"nvlink_bytes": int(nbytes), "nvlink_GB/s": round(gbs, 1),
                          "nvlink_frac": round(gbs / NVLINK_GBS, 4)})
        stages[name] = entry
    dom = max((n for n in stages if "bytes" in stages[n]),
              key=lambda n: stages[n]["ms"] * stages[n]["launches_per_step"])
    # Shares of the step: the all-stage pass above brackets every stage with
    # events (which itself costs time between kernels), so its stage times
    # are used only as shares of the event-free ms_per_step.
    top = [n for n in stages if n != "hop_kernels"]  # hop kernels nest inside "reduce"
    tot = sum(stages[n]["ms"] * stages[n]["launches_per_step"] for n in top) or 1.0
    for n in stages:
        share = stages[n]["ms"] * stages[n]["launches_per_step"] / tot
        stages[n]["share"] = round(share, 4)
        stages[n]["ms_in_step"] = round(share * ms, 5)
    # The dominant stage timed ALONE: a third pass with events around that
    # stage only (BO_PROFILE_STAGES), so no other bracket perturbs it; the
    # roofline's achieved GB/s comes from this duration.
    dom_bit = STAGES.index(dom)
    os.environ["BO_PROFILE_STAGES"] = str(1 << dom_bit)
    pipe.lib.bo_profile_enable(pipe.ctx, 1)
    pipe.lib.bo_profile_read(pipe.ctx, stage_ms, stage_n, 1)
    barrier()
    for _ in range(args.steps):
        step()
    barrier()
    pipe.lib.bo_profile_read(pipe.ctx, stage_ms, stage_n, 1)
    pipe.lib.bo_profile_enable(pipe.ctx, 0)
    del os.environ["BO_PROFILE_STAGES"]
    alone = stage_ms[dom_bit] / max(stage_n[dom_bit], 1)
    st_dom = stages[dom]
    st_dom["ms_evented_all_stages"] = st_dom["ms"]
    st_dom["ms_alone"] = round(alone, 5)
    # The kernel's in-step duration: its share of the event-free step (the
    # all-stage pass's shares x ms_per_step). A bracket of its own, however
    # tight, serialises the kernel's tail against its neighbours and reads
    # 2-9 % long (profiles/r02_notes.md); ms_alone is kept beside it.
    in_step = st_dom["ms_in_step"] / max(st_dom["launches_per_step"], 1e-9)
    st_dom["ms"] = round(in_step, 5)
    st_dom["timed"] = "share of the event-free step (ms_in_step); ms_alone: events around this stage only"
    if "bytes" in st_dom:
        gbs = st_dom["bytes"] / (in_step * 1e-3) / 1e9
        st_dom.update({"GB/s": round(gbs, 1), "frac": round(gbs / hbm, 4),
                       "frac_alone": round(st_dom["bytes"] / (alone * 1e-3) / 1e9 / hbm, 4)})
    if "nvlink_bytes" in st_dom:
        gbs = st_dom["nvlink_bytes"] / (in_step * 1e-3) / 1e9
        st_dom.update({"nvlink_GB/s": round(gbs, 1), "nvlink_frac": round(gbs / NVLINK_GBS, 4),
                       "nvlink_frac_alone": round(st_dom["nvlink_bytes"] / (alone * 1e-3) / 1e9 / NVLINK_GBS, 4)})
    # The other stages on the same footing: "ms" (and the rates derived from
    # it) is the stage's share of the event-free step per launch, so the stage
    # times add up to ms_per_step; the bracketed time stays as ms_evented.
    for n, entry in stages.items():
        if n == dom:
            continue
        per = entry["ms_in_step"] / max(entry["launches_per_step"], 1e-9)
        entry["ms_evented"] = entry["ms"]
        entry["ms"] = round(per, 5)
        if "bytes" in entry:
            gbs = entry["bytes"] / (per * 1e-3) / 1e9
            entry.update({"GB/s": round(gbs, 1), "frac": round(gbs / hbm, 4)})
        if "nvlink_bytes" in entry:
            gbs = entry["nvlink_bytes"] / (per * 1e-3) / 1e9
            entry.update({"nvlink_GB/s": round(gbs, 1), "nvlink_frac": round(gbs / NVLINK_GBS, 4)})
    kernel_names = {"accumulate": "k_accumulate", "finalize": "k_finalize",
                    "lamb_norms": ("k_lamb_p1r" if resident else "k_lamb_p1") if world == 1 else
                                  ("k_p1w + k_push_posted (grouped, overlapped)" if grouped else "k_p1w"),
                    "lamb_update": "k_lamb_p2" if world == 1 else "k_shard_p2_push",
                    "hop_kernels": "k_hopx"}
    if st_dom.get("nvlink_frac", 0.0) > st_dom["frac"]:
        # the parameter push / ring hops at world > 1: NVLink is the bound
        roofline = {"kernel": kernel_names[dom], "bound": "nvlink", "achieved": st_dom["nvlink_GB/s"],
                    "peak": NVLINK_GBS, "peak_kind": "measured (B200_PROFILING.md peer copy)",
                    "unit": "GB/s", "frac": st_dom["nvlink_frac"], "traffic": None,
                    "frac_alone": st_dom.get("nvlink_frac_alone"), "ms": st_dom["ms"],
                    "ms_alone": st_dom["ms_alone"],
                    "algorithmic_bytes_per_launch": st_dom["nvlink_bytes"],
                    "hbm_frac": st_dom["frac"]}
    else:
        roofline = {"kernel": kernel_names[dom], "bound": "hbm", "achieved": st_dom["GB/s"],
                    "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s", "frac": st_dom["frac"],
                    "traffic": traffic_from_profiles(kernel_names[dom]),
                    "frac_alone": st_dom.get("frac_alone"), "ms": st_dom["ms"],
                    "ms_alone": st_dom["ms_alone"],
                    "algorithmic_bytes_per_launch": st_dom["bytes"]}
    if roofline["frac"] > 1.0:
        roofline["note"] = ("the measured HBM peak is a 1:1 read:write copy; this kernel's "
                            "read-heavy mix streams slightly above it")

    # whole-step roofline: sum over stages of max(HBM, NVLink)
    # time, with A = accumulate + finalize (36 B/param, 34 with the binary16
    # wire: the fusion buffer element is E bytes), C = LAMB on the shard
    # (24 + E B/param: g, w, m, v read; w, m, v written; one rank reads the
    # fp32 fusion buffer), B = reduce-scatter, D = all-gather of fp32 weights;
    # plus the stricter pipelined bound max(sum HBM / BW_hbm, sum NVL / BW_nvl)
    E = 2 if f16 else 4
    E_lamb = E if world > 1 else 4
    if resident:
        # all K micros read once in the sync pass, no accumulator and, on one
        # rank, no fusion buffer (the gradient feeds LAMB in registers)
        hbm_a = (2 * K + (E if world > 1 else 0)) * P
        hbm_c = (24 + (E if world > 1 else 0)) * P / world
    else:
        hbm_a = (BYTES_ACCUMULATE_FIRST + BYTES_ACCUMULATE * (K - 2) + 2 + 4 + E) * P if K > 1 \
            else (2 + E) * P
        hbm_c = (24 + E_lamb) * P / world
    nvl_b = (world - 1) / world * E * P
    nvl_d = (world - 1) / world * 4 * P
    t_roof = hbm_a / (hbm * 1e9) + hbm_c / (hbm * 1e9) + nvl_b / (NVLINK_GBS * 1e9) + \
        nvl_d / (NVLINK_GBS * 1e9)
    t_pipe = max((hbm_a + hbm_c) / (hbm * 1e9), (nvl_b + nvl_d) / (NVLINK_GBS * 1e9))
    step_roofline = {"t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / ms, 4),
                     "t_pipelined_ms": round(t_pipe * 1e3, 4),
                     "pipelined_frac": round(t_pipe * 1e3 / ms, 4),
                     "hbm_bytes": int(hbm_a + hbm_c), "nvlink_bytes": int(nvl_b + nvl_d),
                     "hbm_gbs": hbm, "nvlink_gbs": NVLINK_GBS,
                     "formula": "frac: sum over stages of max(HBM/BW_hbm, NVL/BW_nvl) with "
                                "A=gradient accumulation + finalize (per-micro API: SURVEY's "
                                "36 B/param at K=4; train_step API: the K binary16 micros read "
                                "once, 2K B/param, + the fusion-buffer write at N>1), C=LAMB on "
                                "the shard, B=RS, D=AG (no overlap; > 1 when stages overlap, "
                                "e.g. the fused last hop); pipelined_frac: max(sum HBM/BW_hbm, "
                                "sum NVL/BW_nvl)"}

    # the same step through the per-micro API (K bo_accumulate calls, fp32
    # accumulator in HBM), timed the same way, for comparison
    per_micro = None
    if args.api == "train_step":
        for _ in range(2):
            step_per_micro()
        barrier()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(args.steps):
            step_per_micro()
        p1.record(stream)
        barrier()
        pm = max_over_ranks(p0.elapsed_time(p1) / args.steps, world, local, emulated)
        per_micro = {"ms_per_step": round(pm, 4), "value": world * P / (pm * 1e-3), "unit": UNIT,
                     "api": "bo_accumulate x K (accumulator in HBM)"}

    # end to end through the public API with host buffers
    e2e = None
    host = None
    if not args.no_e2e:
        # pinned host buffers + a second device slot set per rank: agree on
        # them across ranks first, so a rank that cannot allocate them skips
        # the e2e leg together with every other rank instead of hanging them
        try:
            host = [torch.empty(total, dtype=torch.int16, pin_memory=True) for _ in range(K)]
        except Exception as e:  # noqa: BLE001
            host, e2e = None, {"value": None, "error": f"pinned host buffers: {e}"[:200]}
        ok = max_over_ranks(0.0 if host is not None else 1.0, world, local, emulated) == 0.0
        if not ok:
            host = None
            if e2e is None:
                e2e = {"value": None, "error": "a rank could not allocate its pinned host buffers"}
    if host is not None:
        for k in range(K):
            host[k].copy_(bufs[k])
        stage_dev = bufs  # reuse the device slots as the H2D destination
        n_e2e = max(1, min(args.e2e_steps, args.steps))
        pipelined = args.api == "train_step" and not args.e2e_serial

        def e2e_step():
            with torch.cuda.stream(stream):
                for k in range(K):
                    stage_dev[k].copy_(host[k], non_blocking=True)
                step()
            return pipe.status()  # D2H of the step result (syncs the stream)

        if pipelined:
            # A training loop that prefetches: step i+1's micro-batches are
            # copied (own stream, second device slot set) while step i
            # computes; every step still copies all its inputs from pinned
            # host memory and reads its result back.
            bufs2 = [torch.empty(total, dtype=torch.int16, device=f"cuda:{local}") for _ in range(K)]
            ptrs2 = GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for b in bufs2 for s in slots])
            sets = [(bufs, all_ptrs), (bufs2, ptrs2)]
            copy_stream = torch.cuda.Stream()
            ready = [torch.cuda.Event(), torch.cuda.Event()]
            free = [torch.cuda.Event(), torch.cuda.Event()]

            def issue_copy(j):
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_event(free[j])  # the step that last read slot set j is done
                    for k in range(K):
                        sets[j][0][k].copy_(host[k], non_blocking=True)
                    ready[j].record(copy_stream)

            def e2e_run(n):
                issue_copy(0)
                for i in range(n):
                    j = i % 2
                    stream.wait_event(ready[j])
                    pipe.train_step_ptr_array(sets[j][1])
                    free[j].record(stream)
                    if i + 1 < n:
                        issue_copy(1 - j)
                    pipe.status()  # D2H of step i's result (syncs the pipeline stream only)
        else:
            def e2e_run(n):
                for _ in range(n):
                    e2e_step()

        e2e_run(1)
        barrier()
        t0 = time.perf_counter()
        e2e_run(n_e2e)
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / n_e2e, world, local, emulated)
        e2e = {"value": world * P / e2e_s, "unit": UNIT, "ms_per_step": round(e2e_s * 1e3, 3),
               "h2d_bytes_per_step": int(K * total * 2),
               "d2h_bytes_per_step": int(C.sizeof(C.c_int64) * 5), "steps": n_e2e,
               "pipelined": "inputs of step i+1 copied on a second stream into a second slot set "
                            "while step i computes" if pipelined else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = run_cpu_reference(spec, 1, K, bucket_bytes, False, 1, args.cpu_steps)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": world * P / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (counter-based fp16 gradients, random-init fp32 weights)",
            "config": {"workload": f"{args.model} optimizer step, K={K} micro-batch fp16 gradient "
                                   f"accumulation, dynamic loss scaling, "
                                   f"{'sharded LAMB + ' + args.wire + '-wire reduce-scatter/all-gather' if world > 1 else 'LAMB'}",
                       "params": P, "tensors": spec.n_tensors, "accumulation": K,
                       "bucket_bytes": bucket_bytes, "buckets": pipe.num_buckets,
                       "wire": args.wire if world > 1 else None,
                       "reduce_algo": args.algo if world > 1 else None,
                       "api": "bo_train_step (K micros resident)" if args.api == "train_step"
                              else "bo_accumulate x K",
                       "kernel_path": path,
                       "parallelism": f"dp{world} (reduce-scatter + sharded LAMB + all-gather)",
                       "l2": "inputs (K x 2 B x P) larger than L2, no flush"},
            "roofline": roofline, "step_roofline": step_roofline, "stages": stages,
            "e2e": e2e, "per_micro_api": per_micro, "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": sampler.summary() if sampler else None,
        }
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    pipe.close()
    if world > 1:
        dist.destroy_process_group()


def main_lockstep(args):
    """`python bench.py --gpus N` without torchrun: the N-rank world emulated
    in this process on ONE GPU (bo_world_init_local: one host thread per rank,
    every rank's kernels serialized on one stream, the cross-rank waits as
    host rendezvous). Runs the world-N step end to end — same kernels, same
    data flow — but its time is the sum of all ranks' work on one device, not
    a scaling number (the JSON line says so)."""
    json_fd = os.dup(1)
    os.dup2(2, 1)
    import threading

    import numpy as np
    import torch

    from paper_2008_00177_b200.pipeline import (REDUCE_AUTO, REDUCE_NCCL, REDUCE_RING, GradPipeline,
                                                LambConfig, ScalerConfig, TrainerConfig, synth_grads)

    world, K = args.gpus, args.accumulation
    torch.cuda.set_device(0)
    spec = model_spec(args.model)
    P = spec.param_count()
    algo = {"auto": REDUCE_AUTO, "ring": REDUCE_RING, "nccl": REDUCE_NCCL}[args.algo]
    cfg = TrainerConfig(LambConfig(lr=1e-4), K, int(args.bucket_mb * (1 << 20)), args.wire == "f16",
                        REDUCE_RING if algo == REDUCE_AUTO else algo,
                        ScalerConfig(init_scale=65536.0, growth_interval=1 << 30))
    pipes = [GradPipeline(spec, cfg, device=0, rank=r, world=world) for r in range(world)]
    w0 = torch.randn(P, device="cuda:0", generator=torch.Generator(device="cuda:0").manual_seed(1234)) * 0.02
    for p in pipes:
        p.load_params(w0)
    del w0
    GradPipeline.world_init_local(pipes)
    numels = spec.numels()
    slots, off = [], 0
    for n in numels:
        slots.append(off)
        off += (n + 127) // 128 * 128
    model_off = np.concatenate([[0], np.cumsum(numels)[:-1]])
    arrays, keep = [], []
    for r in range(world):
        bufs = []
        for k in range(K):
            b = torch.empty(off, dtype=torch.int16, device="cuda:0")
            for t, n in enumerate(numels):
                synth_grads(b[slots[t]:slots[t] + n], int(model_off[t]), 1, r, 0, k, 65536.0)
            bufs.append(b)
        keep.append(bufs)
        arrays.append(GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for b in bufs for s in slots]))
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(pipes[0].stream_handle())
    gate = threading.Barrier(world)
    errors = []

    def run(r, n):
        try:
            gate.wait()
            for _ in range(n):
                pipes[r].train_step_ptr_array(arrays[r])
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    def steps(n):
        th = [threading.Thread(target=run, args=(r, n)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errors:
            raise errors[0]

    steps(args.warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    w = [p.read_params() for p in pipes]
    same = all(np.array_equal(w[0].view(np.uint32), x.view(np.uint32)) for x in w[1:])
    st = pipes[0].status()
    line = {"metric": METRIC, "value": world * P / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (counter-based fp16 gradients, random-init fp32 weights)",
            "config": {"workload": f"{args.model} optimizer step, world {world} emulated on one GPU",
                       "params": P, "accumulation": K, "wire": args.wire,
                       "kernel_path": pipes[0].path(),
                       "emulated": f"lockstep world of {world} ranks in one process on 1 GPU: every "
                                   "rank's kernels serialized on one stream, cross-rank waits as "
                                   "host-thread rendezvous; ms_per_step is ALL ranks' work on one "
                                   "device, not a scaling number",
                       "replicas_identical": bool(same), "lamb_step": st.lamb_step,
                       "skipped_steps": st.skipped_steps}}
    os.write(json_fd, (json.dumps(line) + "\n").encode())
    for p in pipes:
        p.close()


def main_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    spec = model_spec(args.model)
    K = args.accumulation
    bucket_bytes = int(args.bucket_mb * (1 << 20))
    f16 = args.wire == "f16" and world > 1
    # documented cap: ~5 s (N=1) to ~15 s (N=8) per full BERT-large step on
    # one core per rank, so best of 3 timed steps after 1 warm-up step
    steps = max(1, min(args.steps, 3))
    warmup = 1
    cpu = run_cpu_reference(spec, world, K, bucket_bytes, f16, warmup, steps)
    if world == 1 and cpu.get("same_config"):
        try:
            cpu["real_train_step_ms"] = round(real_train_step_seconds(spec, K, bucket_bytes) * 1e3, 1)
        except Exception as e:  # noqa: BLE001
            cpu["real_train_step_ms"] = f"failed: {e}"
    line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": cpu["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.model} optimizer step, K={K} micro-batch gradient "
                                   f"accumulation, LAMB (reference CPU path)",
                       "params": spec.param_count(), "tensors": spec.n_tensors,
                       "accumulation": K, "bucket_bytes": bucket_bytes,
                       "wire": args.wire if world > 1 else None,
                       "parallelism": f"{world} rank thread(s) (InProcHub ring, replicated lamb_step)",
                       "steps_cap": "best of min(--steps, 3) after 1 warm-up step"},
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        main_reference(a)
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        main_lockstep(a)
    else:
        main_b200(a)
