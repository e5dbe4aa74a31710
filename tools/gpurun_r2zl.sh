for i in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zl_bench_base_$i.json 2>> gpurun_out/r2zl.err
  BO_P1R_PROBE=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zl_bench_probe_$i.json 2>> gpurun_out/r2zl.err
done
BO_P1R_PROBE=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'k_lamb_p1r' -c 6 --csv --log-file gpurun_out/r2zl_probe_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2zl_ncu.log 2>&1
