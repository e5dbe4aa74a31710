"""One rank of the ring all-reduce operator drop-ins under torchrun (one GPU
per rank): bo_ring_allreduce_f32 / bo_ring_allreduce_f16_wire
(collective.hpp:104-114) on the sizes of the reference's own ring tests
(test_collective.cpp:403-436) plus one that runs in slices, checked bit for
bit against the oracle's ring (itself pinned to the compiled reference).
Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.test_gpu_ring_ops import SIZES, case_data  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from oracle.oracle import Oracle
    from paper_2008_00177_b200.model_spec import BERT_TINY, bert_spec
    from paper_2008_00177_b200.pipeline import (REDUCE_RING, GradPipeline, LambConfig, ScalerConfig,
                                                TrainerConfig, ring_allreduce, ring_allreduce_f16_wire)

    orc = Oracle()
    spec = bert_spec(BERT_TINY)
    cfg = TrainerConfig(LambConfig(), 1, 16 << 10, True, REDUCE_RING, ScalerConfig())
    pipe = GradPipeline(spec, cfg, device=local, rank=rank, world=world)
    pipe.comm_init_torch()
    bad = []
    for n in SIZES:
        for kind in (0, 1):
            data = case_data(world, n, kind)
            ref = orc.ring_allreduce(data, kind)
            x = torch.from_numpy(data[rank].copy()).cuda(local)
            (ring_allreduce if kind == 0 else ring_allreduce_f16_wire)(pipe, x)
            got = x.cpu().numpy()
            if not np.array_equal(got.view(np.uint32), ref[rank].view(np.uint32)):
                bad.append((n, kind))
    pipe.close()
    print(json.dumps({"rank": rank, "world": world, "ok": not bad, "mismatch": bad}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
