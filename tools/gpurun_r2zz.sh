# round 2, run zz: grouped LAMB + posted push (32-register k_push_posted): lockstep parity, benches at 2 / 4 GPUs
(BO_PUSH_POSTED_CTAS=48 timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "grouped") > gpurun_out/r2zz_emu.log 2>&1
for n in 4 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zz_bench${n}_serial.json 2>> gpurun_out/r2zz.err
  for g in 28000000 42000000 84000000; do
    for p in 48 96; do
      BO_LAMB_GROUP_ELEMS=$g BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zz_bench${n}_g${g}_p$p.json 2>> gpurun_out/r2zz.err
    done
  done
done
