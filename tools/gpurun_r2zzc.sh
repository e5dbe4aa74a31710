# round 2, run zzc: grouped LAMB + posted push as the default at world >= 4: the full -m gpu suite on a 4-GPU box, then bench lines at N = 2 / 4 (defaults, e2e included)
(time timeout 2400 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zzc_tests.log 2>&1
for n in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2997$n bench.py --gpus $n > gpurun_out/r2zzc_bench$n.json 2>> gpurun_out/r2zzc_bench.err
done
BO_LAMB_GROUP_ELEMS=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29981 bench.py --gpus 4 --no-e2e > gpurun_out/r2zzc_bench4_serial.json 2>> gpurun_out/r2zzc_bench.err
