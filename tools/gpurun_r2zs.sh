# round 2, run zs: the ring all-reduce operator drop-ins over the library's own NVLink ring, against the oracle (lockstep worlds 2-8 on one GPU; 2 / 3 / 4 processes on 4 GPUs)
(time timeout 1200 python -m pytest tests/test_gpu_ring_ops.py -q -rs -x) > gpurun_out/r2zs_ops.log 2>&1
