# round 2, run zf: streamed one-rank LAMB (BO_STREAM=1) with the L2 prefetch, distance / lag sweep
(timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -rs -k "stream") > gpurun_out/r2zf_tests.log 2>&1
timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2zf_bench1_twopass.json 2>> gpurun_out/r2zf.err
for d in 100 197 296; do for lag in 64 256; do
  BO_STREAM=1 BO_STREAM_LAG=$lag BO_P1R_PREFETCH=$d timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2zf_bench1_d${d}_lag$lag.json 2>> gpurun_out/r2zf.err
done; done
BO_STREAM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_lamb_stream' -c 2 --csv --log-file gpurun_out/r2zf_ncu.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2zf_ncu.log 2>&1
