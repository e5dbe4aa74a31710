"""Roofline of bo_fused_optimizer_step (the paper's fused Adam-form optimizer
kernel) on BERT-large's 398 tensors: 28 B/param of HBM
traffic (w, g, m, v read; w, m, v written). Prints one JSON line.

    python tools/fused_opt_bench.py [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--model", default="bert-large")
    args = ap.parse_args()
    import torch

    from bench import model_spec, peaks
    from paper_2008_00177_b200.pipeline import fused_optimizer_step

    spec = model_spec(args.model)
    numels = spec.numels()
    P = sum(numels)
    bufs = [torch.randn(P, device="cuda") * s for s in (0.02, 1e-3, 1e-4, 1e-3)]
    bufs[3] = bufs[3] * bufs[3]
    views = [[], [], [], []]
    off = 0
    for n in numels:
        for k in range(4):
            views[k].append(bufs[k][off:off + n])
        off += n
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for step in range(1, 4):
            fused_optimizer_step(*views, 1e-4, 0.9, 0.999, 1e-6, 0.01, step, stream=s)
        torch.cuda.synchronize()
        e0.record(s)
        for step in range(4, 4 + args.steps):
            fused_optimizer_step(*views, 1e-4, 0.9, 0.999, 1e-6, 0.01, step, stream=s)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    hbm, kind = peaks()
    gbs = 28 * P / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": "k_fused_adam", "model": args.model, "params": P, "tensors": len(numels),
                      "ms": round(ms, 4), "bytes_per_param": 28, "achieved_GBs": round(gbs, 1),
                      "peak_GBs": hbm, "peak_kind": kind, "frac": round(gbs / hbm, 4),
                      "note": "per-call host table build included; the table travels as a kernel parameter"}))


if __name__ == "__main__":
    main()
