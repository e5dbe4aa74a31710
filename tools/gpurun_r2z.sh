# round 2, run z: k_lamb_p1r bulk L2 prefetch distance sweep (BO_P1R_PREFETCH), one GPU
for d in 0 148 296 444 592 0; do
  BO_P1R_PREFETCH=$d timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2z_bench1_pf$d.json 2>> gpurun_out/r2z.err
done
BO_P1R_PREFETCH=296 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:'k_lamb_p1r' -c 3 --csv --log-file gpurun_out/r2z_ncu.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2z_ncu.log 2>&1
