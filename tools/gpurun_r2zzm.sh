# round 2, run zzm: lockstep parity with the layout-dependent grouped default (all worlds and cases)
(timeout 600 python -m pytest tests/test_gpu_world_emu.py -q -rs -k "not bert_large") > gpurun_out/r2zzm_emu.log 2>&1
