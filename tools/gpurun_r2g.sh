# round 2, run g: guard pages (aligned vector paths), default vs copy-engine push
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/guard_pages.py > gpurun_out/r2g_guard.log 2>&1; echo rc=$? >> gpurun_out/r2g_guard.log
for ce in 0 1; do for n in 2 4; do BO_PUSH_CE=$ce timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2g_bench${n}_ce$ce.json 2> gpurun_out/r2g_bench${n}_ce$ce.err; done; done
for ce in 0 1; do BO_PUSH_CE=$ce timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 tools/params_ready_demo.py --gpus 4 > gpurun_out/r2g_demo4_ce$ce.json 2> gpurun_out/r2g_demo4_ce$ce.err; done
(BO_PUSH_CE=1 CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_world_emu.py -x -q -k "not full_size") > gpurun_out/r2g_world_emu_ce.log 2>&1
(BO_PUSH_CE=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "two_gpus and (ring16_resident or ring32 or ring16_overlap) and not shapes and not bert") > gpurun_out/r2g_multi_ce.log 2>&1
