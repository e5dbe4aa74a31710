# round 2, run zn: lockstep worlds 3 and 6 (non-power-of-two) against the oracle, with the existing 2 / 4 / 8
(time timeout 1500 python -m pytest tests/test_gpu_world_emu.py -q -rs -k "not bert_large") > gpurun_out/r2zn_emu.log 2>&1
