# round 2, run zc: k_p1w in-warp prefetch distance sweep (BO_P1W_PREFETCH) at 2 / 4 GPUs
for n in 2 4; do
  for p in 0 2 4 8 16; do
    BO_P1W_PREFETCH=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2zc_bench${n}_p$p.json 2>> gpurun_out/r2zc.err
  done
done
