# round 2, run za: finer k_lamb_p1r prefetch sweep + k_lamb_p2 prefetch, one GPU
for d in 48 96 148 200 250; do
  BO_P1R_PREFETCH=$d timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2za_bench1_pf$d.json 2>> gpurun_out/r2za.err
done
for d2 in 148 296 592 1184; do
  BO_P1R_PREFETCH=148 BO_P2_PREFETCH=$d2 timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2za_bench1_pf148_p2$d2.json 2>> gpurun_out/r2za.err
done
BO_P1R_PREFETCH=148 timeout 300 python bench.py --steps 20 --api accumulate --no-e2e --no-cpu-baseline > gpurun_out/r2za_bench1_acc_pf148.json 2>> gpurun_out/r2za.err
