# round 2, run zza: grouped LAMB + posted push (two tiles in flight per thread), repeated A/B at 4 and 2 GPUs
(BO_PUSH_POSTED_CTAS=48 timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "grouped") > gpurun_out/r2zza_emu.log 2>&1
for rep in 1 2; do
for n in 4 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zza_bench${n}_serial_$rep.json 2>> gpurun_out/r2zza.err
  for cfg in 42000000:48 42000000:64 84000000:96; do
    g=${cfg%%:*}; p=${cfg##*:}
    BO_LAMB_GROUP_ELEMS=$g BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zza_bench${n}_g${g}_p${p}_$rep.json 2>> gpurun_out/r2zza.err
  done
done
done
