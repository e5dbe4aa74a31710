# round 2, run p: full -m gpu suite on 4 GPUs (one GPU per rank for the multi-process cases) + benches
(time timeout 2000 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2p_tests_4gpu.log 2>&1
for n in 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2996$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2p_bench$n.json 2> gpurun_out/r2p_bench$n.err; done
