# round 2, run w: copy-engine parameter all-gather (BO_PUSH_CE) parity + benches at 2 / 4 GPUs
(timeout 600 python -m pytest tests/test_gpu_world_emu.py -q -x -rs -k "ce") > gpurun_out/r2w_emu.log 2>&1
(timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -rs -k "ce") > gpurun_out/r2w_multi.log 2>&1
for n in 2 4; do
  for ce in 0 1; do
    BO_PUSH_CE=$ce timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2997$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2w_bench${n}_ce$ce.json 2> gpurun_out/r2w_bench${n}_ce$ce.err
  done
  for g in 8388608 16777216 67108864; do
    BO_PUSH_CE=1 BO_CE_GROUP_ELEMS=$g timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2998$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2w_bench${n}_g$g.json 2>> gpurun_out/r2w_sweep.err
  done
done
