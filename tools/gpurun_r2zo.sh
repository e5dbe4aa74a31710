# round 2, run zo: world 3 (non-power-of-two) with one process per GPU on a 4-GPU box, every ring/push variant against the oracle
(time timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rs -k "more_gpus") > gpurun_out/r2zo_multi.log 2>&1
