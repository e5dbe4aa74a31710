#!/usr/bin/env python
"""Config 5: fusion-buffer (bucket) size sweep of the step at N GPUs.

Runs bench.py once per (parameter set, wire, bucket size) — BERT-large with the
phase-1 (max_seq 128) and phase-2 (max_seq 512) parameter sets, bucket_bytes in
{1, 4, 16, 64, 256, 1024} MiB (BucketLayout::build gives 295/294/122/25/6/2
buckets for BERT-large) — and writes one summary JSON (stdout and --out).

    python sweep.py --gpus 4 --steps 10 --warmup 3 --out profiles/r02_sweep_n4.json
    (wires: the binary16 ring, the bit-exact fp32 ring, the NCCL fp32 reduce-scatter)
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
BUCKETS_MB = [1, 4, 16, 64, 256, 1024]


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_one(n, model, wire, algo, mb, steps, warmup):
    args = [os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", str(steps), "--warmup",
            str(warmup), "--model", model, "--wire", wire, "--algo", algo, "--bucket-mb", str(mb),
            "--no-e2e", "--no-cpu-baseline"]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}"] + args
    else:
        cmd = [sys.executable] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"error": (r.stderr or r.stdout)[-500:]}
    d = json.loads(lines[-1])
    return {"ms_per_step": d["ms_per_step"], "value": d["value"], "buckets": d["config"]["buckets"],
            "step_roofline_frac": d["step_roofline"]["frac"],
            "stages_ms": {k: v["ms"] for k, v in d["stages"].items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--wires", default="f16:ring,f32:ring,f32:nccl")
    ap.add_argument("--models", default="bert-large-128,bert-large")
    ap.add_argument("--buckets", default=",".join(str(b) for b in BUCKETS_MB))
    args = ap.parse_args()
    rows = []
    for model in args.models.split(","):
        for wa in args.wires.split(","):
            wire, algo = wa.split(":")
            for mb in [float(b) for b in args.buckets.split(",")]:
                res = run_one(args.gpus, model, wire, algo, mb, args.steps, args.warmup)
                row = {"model": model, "wire": wire, "algo": algo, "bucket_mb": mb, **res}
                rows.append(row)
                print(json.dumps(row), file=sys.stderr, flush=True)
    out = {"config": "fusion-buffer sweep (BASELINE config 5)", "n_gpus": args.gpus,
           "metric": "BERT-large optimizer step params/sec", "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
