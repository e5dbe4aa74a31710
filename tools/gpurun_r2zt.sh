# round 2, run zt: the C++ adapter test with the ring all-reduce operators against the real reference collectives (lockstep worlds 2-4 on one GPU)
(time timeout 900 python -m pytest tests/test_gpu_adapter.py -q -rs) > gpurun_out/r2zt_adapter.log 2>&1
(timeout 600 oracle/_ref/adapter_test) > gpurun_out/r2zt_adapter_bin.log 2>&1
