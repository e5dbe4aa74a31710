# round 2, run l: the round's bench lines (N = 1, 2, 4; world 8 in lockstep on one GPU),
# then the whole -m gpu suite on ONE GPU, as the driver's round-end box runs it
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench1.json 2> gpurun_out/r2l_bench1.err
for n in 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2992$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2l_bench$n.json 2> gpurun_out/r2l_bench$n.err; done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --gpus 8 --steps 10 --warmup 3 > gpurun_out/r2l_bench8_lockstep.json 2> gpurun_out/r2l_bench8_lockstep.err
(time CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2l_tests_1gpu.log 2>&1
