# round 2, run zzb: grouped LAMB + posted push with phase 1 of group g+1 issued ahead of group g's partials barrier (BO_LAMB_GROUP_AHEAD=1): lockstep parity, A/B at 4 and 2 GPUs
(BO_PUSH_POSTED_CTAS=48 BO_LAMB_GROUP_AHEAD=1 timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "grouped") > gpurun_out/r2zzb_emu.log 2>&1
for n in 4 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zzb_bench${n}_serial.json 2>> gpurun_out/r2zzb.err
  for cfg in 42000000:64:0 42000000:64:1 42000000:80:1 28000000:64:1 84000000:80:1; do
    g=$(echo $cfg | cut -d: -f1); p=$(echo $cfg | cut -d: -f2); a=$(echo $cfg | cut -d: -f3)
    BO_LAMB_GROUP_AHEAD=$a BO_LAMB_GROUP_ELEMS=$g BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --no-e2e > gpurun_out/r2zzb_bench${n}_g${g}_p${p}_a$a.json 2>> gpurun_out/r2zzb.err
  done
done
