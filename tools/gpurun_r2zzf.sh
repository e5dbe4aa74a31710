# round 2, run zzf: same-box A/B after the k_p1w spill fix: N = 2 serial vs grouped (84 M-element groups, 96-CTA posted push), N = 4 serial vs the grouped default
for rep in 1 2; do
  BO_LAMB_GROUP_ELEMS=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29962 bench.py --gpus 2 --no-e2e > gpurun_out/r2zzf_bench2_serial_$rep.json 2>> gpurun_out/r2zzf.err
  BO_LAMB_GROUP_ELEMS=84000000 BO_PUSH_POSTED_CTAS=96 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29962 bench.py --gpus 2 --no-e2e > gpurun_out/r2zzf_bench2_g84_$rep.json 2>> gpurun_out/r2zzf.err
done
BO_LAMB_GROUP_ELEMS=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2zzf_bench4_serial.json 2>> gpurun_out/r2zzf.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2zzf_bench4_default.json 2>> gpurun_out/r2zzf.err
