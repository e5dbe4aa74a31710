# round 2, run zzh: posted-push CTA count at N = 4 with the grouped default (eight groups)
for p in 48 80 96 128; do
  BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2zzh_bench4_p$p.json 2>> gpurun_out/r2zzh.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2zzh_bench4_p64.json 2>> gpurun_out/r2zzh.err
