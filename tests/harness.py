"""GPU test harness: drive GradPipeline with the synthetic gradient spec.

Per step, the fp16 inputs of every micro-batch are produced on the device by
bo_synth_grads with the pipeline's CURRENT loss scale (read back from the
device), exactly as oracle.train regenerates them on the CPU, then the
scheduled injections (step, rank, micro, flat_index, bits) overwrite single
elements.
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2008_00177_b200.pipeline import GradPipeline, synth_grads


class GradBuffers:
    """K per-micro gradient buffers with per-tensor slots.

    aligned=True gives every tensor a 256-byte aligned slot (vectorised
    accumulate path); aligned=False packs tensors back to back in model order
    starting one element into the buffer, so that the slots are misaligned
    (scalar paths) whatever the tensor sizes.
    """

    def __init__(self, spec, K: int, device: int = 0, aligned: bool = True):
        self.spec = spec
        self.numels = spec.numels()
        self.model_off = np.concatenate([[0], np.cumsum(self.numels)[:-1]]).astype(np.int64)
        offs, o = [], 0 if aligned else 1
        for n in self.numels:
            offs.append(o)
            o += (n + 127) // 128 * 128 if aligned else n
        self.slot = offs
        self.total = o
        self.aligned = aligned
        self.bufs = [torch.zeros(self.total, dtype=torch.int16, device=f"cuda:{device}")
                     for _ in range(K)]
        self.ptrs = [[b.data_ptr() + 2 * s for s in self.slot] for b in self.bufs]

    def fill(self, k: int, seed: int, rank: int, step: int, scale: float, spike_ppm=0,
             spike_exp=1) -> None:
        buf = self.bufs[k]
        if not self.aligned:
            synth_grads(buf[1:], 0, seed, rank, step, k, scale, spike_ppm, spike_exp)
            return
        for t, n in enumerate(self.numels):
            s = self.slot[t]
            synth_grads(buf[s:s + n], int(self.model_off[t]), seed, rank, step, k, scale,
                        spike_ppm, spike_exp)

    def inject(self, k: int, flat_index: int, bits: int) -> None:
        t = int(np.searchsorted(self.model_off, flat_index, side="right") - 1)
        pos = self.slot[t] + (flat_index - int(self.model_off[t]))
        self.bufs[k][pos] = np.int16(np.uint16(bits).view(np.int16))

    def model_order(self, k: int) -> np.ndarray:
        """This micro's binary16 bits in model order (uint16)."""
        h = self.bufs[k].cpu().numpy().view(np.uint16)
        return np.concatenate([h[s:s + n] for s, n in zip(self.slot, self.numels)])


def run_pipeline(spec, cfg, params0, steps, grad_seed=1, spike_ppm=0, spike_exp=1, injections=(),
                 rank=0, world=1, aligned=True, pipe=None, device=0, first_step=0, overlap=None,
                 resident=False):
    """Run optimizer steps first_step .. first_step+steps-1 (the step index
    seeds the synthetic gradients); returns (pipe, scale_used, found_inf).

    overlap: None (the sync micro through bo_accumulate) or a list of chunk
    sizes: the sync micro is then delivered through bo_sync_ready in the
    layout's ready order, in chunks of these sizes (cycled).
    resident: all K micros filled first, then one bo_train_step."""
    if pipe is None:
        pipe = GradPipeline(spec, cfg, device=device, rank=rank, world=world)
        pipe.load_params(np.asarray(params0, np.float32))
    K = cfg.accumulation
    gb = GradBuffers(spec, K, device, aligned)
    scale_used, found = [], []
    torch.cuda.set_device(device)
    for step in range(first_step, first_step + steps):
        S = pipe.status().loss_scale
        scale_used.append(S)
        for k in range(K):
            gb.fill(k, grad_seed, rank, step, S, spike_ppm, spike_exp)
            for (st, r, mk, idx, bits) in injections:
                if st == step and r == rank and mk == k:
                    gb.inject(k, idx, bits)
            torch.cuda.synchronize()
            if resident:
                if k == K - 1:
                    pipe.train_step(gb.ptrs)
            elif overlap is None or k < K - 1:
                pipe.accumulate(k, gb.ptrs[k])
            else:
                order = pipe.ready_order()
                i = j = 0
                while i < len(order):
                    n = max(1, overlap[j % len(overlap)])
                    ids = order[i:i + n]
                    pipe.sync_ready(ids, [gb.ptrs[k][t] for t in ids])
                    i += n
                    j += 1
        pipe.synchronize()
        found.append(int(pipe.status().found_inf))
    return pipe, np.array(scale_used, np.float32), np.array(found, np.int32)


def rel_err(a: np.ndarray, b: np.ndarray) -> float:
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    denom = np.maximum(np.abs(b), 1e-30)
    return float(np.max(np.abs(a - b) / denom)) if a.size else 0.0


def max_rel_or_abs(a, b, floor=1e-6) -> float:
    """max |a-b| / max(|b|, floor): relative error with an absolute floor for ~0 values."""
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def run_world_lockstep(spec, cfg, params0, world, steps, device=0, grad_seed=1, spike_ppm=0,
                       spike_exp=1, injections=(), resident=False, overlap=None):
    """A whole world in this process on one GPU (bo_world_init_local): one
    host thread per rank, as the reference's run_data_parallel, every rank's
    kernels on one shared stream in lockstep. Returns (pipes, scale_used,
    found_inf) with rank 0's sequences."""
    import threading

    pipes = [GradPipeline(spec, cfg, device=device, rank=r, world=world) for r in range(world)]
    for p in pipes:
        p.load_params(np.asarray(params0, np.float32))
    GradPipeline.world_init_local(pipes)
    out = [None] * world
    errors = []

    def rank_thread(r):
        try:
            torch.cuda.set_device(device)
            out[r] = run_pipeline(spec, cfg, None, steps, grad_seed=grad_seed, spike_ppm=spike_ppm,
                                  spike_exp=spike_exp, injections=injections, rank=r, world=world,
                                  pipe=pipes[r], device=device, resident=resident, overlap=overlap)
        except BaseException as e:  # noqa: BLE001
            errors.append((r, e))

    threads = [threading.Thread(target=rank_thread, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0][1]
    return pipes, out[0][1], out[0][2]
