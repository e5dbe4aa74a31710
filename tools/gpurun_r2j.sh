# round 2, run j: BASELINE config 5 sweep at 4 GPUs with the bit-exact fp32 ring next to the NCCL fp32 reduce-scatter
timeout 2400 python sweep.py --gpus 4 --steps 10 --warmup 3 --out gpurun_out/r2j_sweep_n4.json > gpurun_out/r2j_sweep.log 2>&1
timeout 900 python sweep.py --gpus 2 --steps 10 --warmup 3 --models bert-large --buckets 4,64 --out gpurun_out/r2j_sweep_n2.json > gpurun_out/r2j_sweep2.log 2>&1
