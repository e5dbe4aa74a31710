# round 2, run m: phase-1 occupancy variants (registers vs resident CTAs)
for v in 2 1; do BO_P1R_MINB=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2m_bench1_p1r$v.json 2> gpurun_out/r2m_bench1_p1r$v.err; done
for v in 4 3; do for n in 2 4; do BO_P1W_MINB=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2993$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2m_bench${n}_p1w$v.json 2> gpurun_out/r2m_bench${n}_p1w$v.err; done; done
