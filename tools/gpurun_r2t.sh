# round 2, run t: paired blockIdx-ordered k_lamb_stream
(timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_config4_full.py -q -x -rs) > gpurun_out/r2t_tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2t_bench1.json 2> gpurun_out/r2t_bench1.err

for lag in 64 256 1024; do
  BO_STREAM_LAG=$lag timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r2t_bench1_lag$lag.json 2>> gpurun_out/r2t_sweep.err
done
for win in 2097152 33554432; do
  BO_STREAM_WINDOW=$win timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r2t_bench1_win$win.json 2>> gpurun_out/r2t_sweep.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_lamb|k_stream' -c 6 --csv --log-file gpurun_out/r2t_ncu_stream.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2t_ncu.log 2>&1
