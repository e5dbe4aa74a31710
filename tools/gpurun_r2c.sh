free -g > gpurun_out/r2c_free.txt
nvidia-smi topo -m >> gpurun_out/r2c_free.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench1.json 2> gpurun_out/r2c_bench1.err
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2c_bench$n.json 2> gpurun_out/r2c_bench$n.err; done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29508 bench.py --gpus 8 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2c_bench8emu.json 2> gpurun_out/r2c_bench8emu.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c_ref1.json 2> gpurun_out/r2c_ref1.err
