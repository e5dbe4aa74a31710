"""Probe: how the event-bracketed duration of the dominant one-rank kernel
(k_lamb_p1r) depends on what brackets it (BERT-large, K=4, bo_train_step).

Prints the step time without events, and for masks {p1r alone, p2 alone,
all stages}: the per-stage mean durations and the step time with events."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_00177_b200 import model_spec as ms  # noqa: E402
from paper_2008_00177_b200.pipeline import (GradPipeline, LambConfig, ScalerConfig,  # noqa: E402
                                            TrainerConfig, synth_grads)

STAGES = ["accumulate", "finalize", "reduce", "lamb_norms", "trust", "lamb_update", "allgather",
          "hop_kernels", "reserved"]


def main():
    spec = ms.bert_spec(ms.BERT_LARGE)
    K, P = 4, spec.param_count()
    cfg = TrainerConfig(LambConfig(lr=1e-4), K, 4 << 20, False, 0,
                        ScalerConfig(init_scale=65536.0, growth_interval=1 << 30))
    pipe = GradPipeline(spec, cfg)
    pipe.load_params(torch.randn(P, device="cuda") * 0.02)
    numels = spec.numels()
    slots, off = [], 0
    for n in numels:
        slots.append(off)
        off += (n + 127) // 128 * 128
    model_off = np.concatenate([[0], np.cumsum(numels)[:-1]])
    bufs = []
    for k in range(K):
        b = torch.empty(off, dtype=torch.int16, device="cuda")
        for t, n in enumerate(numels):
            synth_grads(b[slots[t]:slots[t] + n], int(model_off[t]), 1, 0, 0, k, 65536.0)
        bufs.append(b)
    arr = GradPipeline.make_ptr_array([b.data_ptr() + 2 * s for b in bufs for s in slots])
    stream = torch.cuda.Stream()
    pipe.set_stream(stream)
    steps = 20
    out = {}

    def timed(sync_each=False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            pipe.train_step_ptr_array(arr)
            if sync_each:
                stream.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    for _ in range(5):
        pipe.train_step_ptr_array(arr)
    out["step_ms_no_events"] = timed()
    for name, mask in [("p1r_alone", 1 << 3), ("p2_alone", 1 << 5), ("all", 0x1FF)]:
        os.environ["BO_PROFILE_STAGES"] = str(mask)
        pipe.lib.bo_profile_enable(pipe.ctx, 1)
        sm = (C.c_double * 9)()
        sn = (C.c_int64 * 9)()
        pipe.lib.bo_profile_read(pipe.ctx, sm, sn, 1)
        t = timed()
        pipe.lib.bo_profile_read(pipe.ctx, sm, sn, 1)
        pipe.lib.bo_profile_enable(pipe.ctx, 0)
        out[name] = {"step_ms": t, **{STAGES[i]: sm[i] / sn[i] for i in range(9) if sn[i]}}
    out["step_ms_no_events_again"] = timed()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
