# round 2, run i: grouped speculative LAMB — parity (lockstep world, 2 GPUs) and step time
(CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_world_emu.py -x -q -k "grouped") > gpurun_out/r2i_world_emu.log 2>&1
(timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "two_gpus and grouped") > gpurun_out/r2i_multi.log 2>&1
for g in 0 24000000 48000000 96000000; do for n in 2 4; do BO_LAMB_GROUP_ELEMS=$g timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2i_bench${n}_g$g.json 2> gpurun_out/r2i_bench${n}_g$g.err; done; done
