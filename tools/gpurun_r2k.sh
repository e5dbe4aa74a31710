# round 2, run k: params_wait gating, adapter vs the real train_step, plain-store push
(timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "params_wait") > gpurun_out/r2k_paramswait.log 2>&1
(CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_gpu_adapter.py -x -q) > gpurun_out/r2k_adapter.log 2>&1
for cfg in "BO_PUSH_STORES=0" "BO_PUSH_STORES=1" "BO_PUSH_STORES=1 BO_LAMB_GROUP_ELEMS=96000000"; do for n in 2 4; do tag=$(echo $cfg | tr ' =' '__'); env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2991$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2k_bench${n}_$tag.json 2> gpurun_out/r2k_bench${n}_$tag.err; done; done
