# round 2, run s: streamed one-rank LAMB (k_lamb_stream) after the item-kind fix
(timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_config4_full.py -q -x -rs) > gpurun_out/r2s_tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2s_bench1.json 2> gpurun_out/r2s_bench1.err
BO_STREAM=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2s_bench1_twopass.json 2> gpurun_out/r2s_bench1_twopass.err
for lag in 128 1024 2048; do
  BO_STREAM_LAG=$lag timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r2s_bench1_lag$lag.json 2>> gpurun_out/r2s_sweep.err
done
for win in 2097152 33554432; do
  BO_STREAM_WINDOW=$win timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r2s_bench1_win$win.json 2>> gpurun_out/r2s_sweep.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_lamb|k_stream' -c 6 --csv --log-file gpurun_out/r2s_ncu_stream.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2s_ncu.log 2>&1
