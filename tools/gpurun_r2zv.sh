# round 2, run zv: bo_replica_hash (one rank, lockstep worlds, numpy restatement) and the adapter's param_hash / replica_hash
(time timeout 900 python -m pytest tests/test_gpu_replica_hash.py tests/test_gpu_adapter.py -q -rs) > gpurun_out/r2zv.log 2>&1
(timeout 300 oracle/_ref/adapter_test) > gpurun_out/r2zv_adapter_bin.log 2>&1
