# round 2, run zi: HEAD validation on 4 GPUs: the multi-GPU parity suite (one process per GPU) and bench lines at N = 2 / 4
(time timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rs) > gpurun_out/r2zi_multi.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2997$n bench.py --gpus $n > gpurun_out/r2zi_bench$n.json 2>> gpurun_out/r2zi_bench.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29981 bench.py --gpus 4 --wire f32 --no-e2e > gpurun_out/r2zi_bench4_f32.json 2>> gpurun_out/r2zi_bench.err
