# round 2, run zzg: after the k_p1w select fix: worlds 3 / 4 one process per GPU (grouped default at 4) and every lockstep world incl. BERT-large at 8
(time timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_world_emu.py -q -rs -k "more_gpus or lockstep or world8") > gpurun_out/r2zzg_tests.log 2>&1
