# round 2, run zp: world > 1 phase 1 as one CTA per quarter tile + bulk L2 prefetch (k_p1q, BO_P1Q=1): lockstep parity, then benches at 2 / 4 GPUs
(BO_P1Q=1 timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "not bert_large") > gpurun_out/r2zp_emu.log 2>&1
for n in 2 4; do
  BO_P1Q=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zp_bench${n}_w.json 2>> gpurun_out/r2zp.err
  for d in 0 400 789 1200; do
    BO_P1Q=1 BO_P1Q_PREFETCH=$d timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zp_bench${n}_q$d.json 2>> gpurun_out/r2zp.err
  done
  BO_P1Q=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zp_bench${n}_w2.json 2>> gpurun_out/r2zp.err
done
