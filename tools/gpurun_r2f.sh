# round 2, run f: guard pages, lockstep world emulation, push-grid variants, params-ready demo
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/guard_pages.py > gpurun_out/r2f_guard.log 2>&1; echo rc=$? >> gpurun_out/r2f_guard.log
(CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_world_emu.py -x -q) > gpurun_out/r2f_world_emu.log 2>&1
for ctas in 0 296 1184; do for n in 2 4; do BO_PUSH_CTAS=$ctas timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2f_bench${n}_c$ctas.json 2> gpurun_out/r2f_bench${n}_c$ctas.err; done; done
for ctas in 16 48 0; do BO_PUSH_CTAS=$ctas timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29714 tools/params_ready_demo.py --gpus 4 > gpurun_out/r2f_demo4_c$ctas.json 2> gpurun_out/r2f_demo4_c$ctas.err; done
