# round 2, run e: lockstep world emulation (GPU 0), benches N=2/4 after the
# per-group push publication, the params-ready demo, compute-sanitizer memcheck
(time CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_world_emu.py -x -q) > gpurun_out/r2e_world_emu.log 2>&1
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2e_bench$n.json 2> gpurun_out/r2e_bench$n.err; done
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tools/params_ready_demo.py --gpus $n > gpurun_out/r2e_demo$n.json 2> gpurun_out/r2e_demo$n.err; done
CUDA_VISIBLE_DEVICES=0 BO_SANITIZER_TOOLS=memcheck BO_SANITIZER_LOG=gpurun_out/r2e_memcheck.txt timeout 900 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/r2e_sanitizer.log 2>&1
