# round 2, run zze: k_p1w with the double-buffered master shard selected arithmetically (no extra spills): lockstep parity, bench N = 4 (grouped default) and N = 2 grouped vs serial
(timeout 900 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "not bert_large") > gpurun_out/r2zze_emu.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2zze_bench4.json 2>> gpurun_out/r2zze.err
for cfg in 84000000:96 42000000:64; do
  g=${cfg%%:*}; p=${cfg##*:}
  BO_LAMB_GROUP_ELEMS=$g BO_PUSH_POSTED_CTAS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29962 bench.py --gpus 2 --no-e2e > gpurun_out/r2zze_bench2_g${g}_p$p.json 2>> gpurun_out/r2zze.err
done
