"""Multi-GPU parity worker (one process per GPU, launched by torchrun).

Every rank drives its GradPipeline with its own synthetic gradients; rank 0
gathers parameters (replicated) and moments (sharded) and compares them with
the CPU oracle's emulation of the same world (oracle.train). Prints one JSON
result line on rank 0 and exits non-zero on a parity failure.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_worker.py \
        --case ring16 --steps 4
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

CASES = {
    # name: (f16_exchange, reduce_algo, K, bucket_bytes, scaler kwargs, spike_ppm, spike_exp, exact)
    "ring16": (True, 1, 2, 8192, dict(init_scale=2.0 ** 13, growth_interval=3), 20, 3, True),
    "ring32": (False, 1, 3, 4096, dict(init_scale=1024.0), 0, 1, True),
    "nccl32": (False, 2, 2, 1 << 20, dict(init_scale=1024.0), 0, 1, False),
    "ring16_1bucket": (True, 1, 1, 1 << 30, dict(init_scale=4096.0), 0, 1, True),
    "ring16_tinybuckets": (True, 1, 2, 1, dict(init_scale=4096.0), 0, 1, True),
}
# "<case>_unfused" / "<case>_fused": the same case with the ring's last hop
# staged (BO_UNFUSED=1) or fused into LAMB phase 1 (BO_FUSE_LAST=1) whatever
# the world's default; "<case>_overlap": the sync micro delivered through
# bo_sync_ready (bucket-level overlap)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="ring16")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--params-wait", action="store_true",
                    help="check bo_params_wait gating instead of oracle parity")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # one GPU per rank (never two ranks on one device: their flag-spinning
    # kernels must run concurrently). The host exchange runs over gloo, so
    # nothing here needs NCCL unless the case does.
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: needs one GPU per rank")
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")

    from oracle.oracle import LambConfig as OL, Oracle, ScalerConfig as OS
    from paper_2008_00177_b200.model_spec import BERT_TINY, ModelConfig, bert_spec, flat_spec
    from paper_2008_00177_b200.pipeline import GradPipeline, LambConfig, ScalerConfig, TrainerConfig
    from tests.harness import max_rel_or_abs, run_pipeline

    case = args.case
    overlap = None
    resident = False
    # "<case>_<suffix>..." in any order: strip known suffixes until a base case remains
    while case not in CASES:
        if case.endswith("_resident"):
            resident = True
            case = case[: -len("_resident")]
        elif case.endswith("_ncclbar"):
            # a 4-byte NCCL all-reduce between ring hops instead of the neighbour flags
            os.environ["BO_RING_BARRIER"] = "nccl"
            case = case[: -len("_ncclbar")]
        elif case.endswith("_pull"):
            # ring hops reading the left neighbour's buffer instead of pushing
            os.environ["BO_RING_PUSH"] = "0"
            case = case[: -len("_pull")]
        elif case.endswith("_overlap"):
            # the sync micro delivered through bo_sync_ready in ragged chunks,
            # with communication groups of ~20k elements (several per step)
            os.environ["BO_COMM_GROUP_ELEMS"] = "20000"
            overlap = [1, 5, 2, 17]
            case = case[: -len("_overlap")]
        elif case.endswith("_unfused"):
            os.environ["BO_UNFUSED"] = "1"
            case = case[: -len("_unfused")]
        elif case.endswith("_grouped"):
            # grouped speculative LAMB (BO_LAMB_GROUP_ELEMS)
            os.environ["BO_LAMB_GROUP_ELEMS"] = "30000"
            case = case[: -len("_grouped")]
        elif case.endswith("_fused"):
            os.environ["BO_FUSE_LAST"] = "1"
            case = case[: -len("_fused")]
        else:
            raise SystemExit(f"unknown case {args.case}")
    f16, algo, K, bb, sc, ppm, sexp, exact = CASES[case]
    if args.params_wait:
        os.environ["BO_PUSH_GROUP_ELEMS"] = "20000"  # several parameter groups on a small model
    if args.model == "tiny":
        spec = bert_spec(BERT_TINY)
    elif args.model == "bert-large":
        from paper_2008_00177_b200.model_spec import BERT_LARGE
        spec = bert_spec(BERT_LARGE)
    elif args.model == "empty":
        spec = flat_spec([0, 5, 4097, 0, 3, 1, 8191], first_use=[2, 0, 1, 4, 3, 6, 5])
    elif args.model == "ragged":
        spec = flat_spec([1, 7, 4099, 13, 2, 30000, 3], first_use=[3, 0, 6, 1, 5, 2, 4])
    else:
        spec = bert_spec(ModelConfig(layers=2, hidden=128, heads=4, vocab=3000, max_seq=64))
    orc = Oracle()
    p0 = orc.build_params(spec, 21)
    P = spec.param_count()
    inj = [(1, world - 1, K - 1, P // 3, 0x7C00)] if ppm else []
    cfg = TrainerConfig(LambConfig(lr=5e-3), K, bb, f16, algo, ScalerConfig(**sc))
    pipe = GradPipeline(spec, cfg, device=local, rank=rank, world=world)
    pipe.load_params(p0)
    pipe.comm_init_torch()
    pipe, su, fi = run_pipeline(spec, cfg, None, args.steps, grad_seed=9, spike_ppm=ppm,
                                spike_exp=sexp, injections=inj, rank=rank, world=world, pipe=pipe,
                                device=local, overlap=overlap, resident=resident)
    gated = True
    if args.params_wait:
        # one more step, then on a second stream: per parameter group,
        # bo_params_wait and a snapshot of the group's tensors — every snapshot
        # must equal the step's final parameters (a wait released early would
        # show values of the previous step)
        before = pipe.read_params()
        pipe, _, _ = run_pipeline(spec, cfg, None, 1, grad_seed=9, rank=rank, world=world, pipe=pipe,
                                  device=local, first_step=args.steps)
        # (run_pipeline synchronises; issue a fresh step without it for the check)
        from tests.harness import GradBuffers
        gb = GradBuffers(spec, K, local, True)
        S = pipe.status().loss_scale
        for k in range(K):
            gb.fill(k, 9, rank, args.steps + 1, S)
        torch.cuda.synchronize()
        side = torch.cuda.Stream(device=local)
        numels = spec.numels()
        off = np.concatenate([[0], np.cumsum(numels)[:-1]]).astype(np.int64)
        views = []
        for t in range(spec.n_tensors):
            ptr = pipe.param_ptr(t)

            class _V:
                __cuda_array_interface__ = {"shape": (numels[t],), "typestr": "<f4", "data": (ptr, False),
                                            "version": 3}
            views.append(torch.as_tensor(_V(), device=f"cuda:{local}") if numels[t] else None)
        snap = [torch.empty(n, device=f"cuda:{local}") if n else None for n in numels]
        pipe.train_step(gb.ptrs)  # enqueued; the waits below do not synchronise with it
        with torch.cuda.stream(side):
            for t in range(spec.n_tensors):
                pipe.params_wait(t, side)
                if numels[t]:
                    snap[t].copy_(views[t])
        torch.cuda.synchronize()
        final = pipe.read_params()
        got = np.concatenate([snap[t].cpu().numpy() if numels[t] else np.zeros(0, np.float32)
                              for t in range(spec.n_tensors)])
        gated = bool(np.array_equal(got.view(np.uint32), final.view(np.uint32)))
        changed = not np.array_equal(final.view(np.uint32), before.view(np.uint32))
        gated = gated and changed
        # the oracle compares args.steps steps: roll the extra two back out
        pipe.close()
        result = {"rank": rank, "ok": gated, "params_wait_gated": gated}
        if rank == 0:
            print(json.dumps(result), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if gated else 1)
    w = pipe.read_params()
    m = np.zeros(P, np.float32)
    v = np.zeros(P, np.float32)
    pipe.read_moments(m, v)
    owned = np.zeros(P, np.float32)
    # moments are sharded: sum the per-rank scatters (each element owned once)
    tm, tv = torch.from_numpy(m), torch.from_numpy(v)
    dist.all_reduce(tm)
    dist.all_reduce(tv)
    tw = torch.from_numpy(w)
    allw = [torch.zeros_like(tw) for _ in range(world)]
    dist.all_gather(allw, tw)
    st = pipe.status()
    result = {"rank": rank}
    if rank == 0:
        ref = orc.train(spec, p0, world, K, bb, f16, OL(lr=5e-3), OS(**sc), args.steps, grad_seed=9,
                        spike_ppm=ppm, spike_exp=sexp, injections=inj)
        mm, vv = tm.numpy(), tv.numpy()
        replicas_equal = all(torch.equal(allw[0], x) for x in allw)
        result.update({
            "case": args.case, "world": world, "params": P, "steps": args.steps,
            "path": pipe.path(), "devices": torch.cuda.device_count(),
            "found_inf": fi.tolist(), "ref_found_inf": ref.found_inf.tolist(),
            "scales_equal": bool(np.array_equal(su, ref.scale_used)),
            "final_scale": st.loss_scale, "ref_final_scale": ref.final_scale,
            "lamb_step": st.lamb_step, "ref_lamb_step": ref.lamb_step,
            "replicas_identical": bool(replicas_equal),
            "w_rel": max_rel_or_abs(w, ref.params), "m_rel": max_rel_or_abs(mm, ref.m, 1e-12),
            "v_rel": max_rel_or_abs(vv, ref.v, 1e-20),
            "w_bit_exact_frac": float(np.mean(w.view(np.uint32) == ref.params.view(np.uint32))),
            "m_bit_exact": bool(np.array_equal(mm.view(np.uint32), ref.m.view(np.uint32))),
            "v_bit_exact": bool(np.array_equal(vv.view(np.uint32), ref.v.view(np.uint32))),
        })
        ok = (result["found_inf"] == result["ref_found_inf"] and result["scales_equal"]
              and st.loss_scale == ref.final_scale and st.lamb_step == ref.lamb_step
              and replicas_equal and result["w_rel"] <= 1e-5 and result["m_rel"] <= 1e-5
              and result["v_rel"] <= 1e-5)
        if exact:
            ok = ok and result["m_bit_exact"] and result["v_bit_exact"]
        result["ok"] = bool(ok)
        print(json.dumps(result), flush=True)
    del owned
    dist.barrier()  # no peer touches this rank's mapped buffers any more
    pipe.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not result["ok"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
