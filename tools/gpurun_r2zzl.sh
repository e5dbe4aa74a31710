# round 2, run zzl: the grouped default now falls back to serial for layouts with > 10 % phase-mismatched chunks: lockstep parity + the 1 GiB / 64 MiB sweep points at N = 4
(timeout 600 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "not bert_large") > gpurun_out/r2zzl_emu.log 2>&1
timeout 600 python sweep.py --gpus 4 --steps 10 --warmup 3 --wires f16:ring --models bert-large --buckets 64,1024 --out gpurun_out/r2zzl_sweep_n4.json > gpurun_out/r2zzl_sweep.log 2>&1
