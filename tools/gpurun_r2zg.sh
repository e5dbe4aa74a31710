# round 2, run zg: world > 1 phase 1 as one CTA per tile + L2 prefetch (BO_P1_CTA=1): parity + benches at 2 / 4 GPUs
(BO_P1_CTA=1 timeout 600 python -m pytest tests/test_gpu_world_emu.py -q -x -rs) > gpurun_out/r2zg_emu.log 2>&1
(BO_P1_CTA=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -rs -k "two_gpus and not bert_large and not shapes") > gpurun_out/r2zg_multi.log 2>&1
for n in 2 4; do
  BO_P1_CTA=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2zg_bench${n}_w.json 2>> gpurun_out/r2zg.err
  for d in 0 100 197 296; do
    BO_P1_CTA=1 BO_P1R_PREFETCH=$d timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2zg_bench${n}_c$d.json 2>> gpurun_out/r2zg.err
  done
done
