# round 2, run zb: k_p1w self-prefetch (BO_P1W_PREFETCH) at 2 / 4 GPUs; k_lamb_p1 prefetch (per-micro API) at 1
for n in 2 4; do
  for p in 0 1 0 1; do
    BO_P1W_PREFETCH=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2zb_bench${n}_p$p.json 2>> gpurun_out/r2zb.err
  done
done
for d in 0 200; do
  CUDA_VISIBLE_DEVICES=0 BO_P1R_PREFETCH=$d timeout 300 python bench.py --steps 20 --api accumulate --no-e2e --no-cpu-baseline > gpurun_out/r2zb_bench1_acc_pf$d.json 2>> gpurun_out/r2zb.err
done
