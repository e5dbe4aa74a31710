# round 2, run zy: grouped speculative LAMB with the few-CTA posted-store push (BO_PUSH_POSTED_CTAS) overlapping phase 1 of the next group: lockstep parity, then benches at 2 / 4 GPUs
(BO_PUSH_POSTED_CTAS=32 timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "grouped") > gpurun_out/r2zy_emu.log 2>&1
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zy_bench${n}_serial.json 2>> gpurun_out/r2zy.err
  for g in 16000000 42000000; do
    for p in 32 48; do
      BO_LAMB_GROUP_ELEMS=$g BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zy_bench${n}_g${g}_p$p.json 2>> gpurun_out/r2zy.err
    done
  done
done
