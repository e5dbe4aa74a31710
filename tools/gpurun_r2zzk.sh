# round 2, run zzk: config-5 bucket sweep at N = 4 with the grouped LAMB default (binary16 ring, phase-2 parameter set)
timeout 900 python sweep.py --gpus 4 --steps 10 --warmup 3 --wires f16:ring --models bert-large --buckets 1,4,64,1024 --out gpurun_out/r2zzk_sweep_n4.json > gpurun_out/r2zzk_sweep.log 2>&1
