# round 2, run zzj: HEAD bench line at N = 4 (grouped default, 128-CTA posted push, e2e included)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 > gpurun_out/r2zzj_bench4.json 2> gpurun_out/r2zzj.err
