# round 2, run u: k_lamb_stream with up to 3 phase-2 tiles per item (phase 2 catches up)
(timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -rs -k "stream or resident or config2 or ragged") > gpurun_out/r2u_tests.log 2>&1
for p2 in 1 2 3; do for lag in 16 64 256; do
  BO_STREAM_P2=$p2 BO_STREAM_LAG=$lag timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r2u_bench1_p${p2}_lag$lag.json 2>> gpurun_out/r2u_sweep.err
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_lamb|k_stream' -c 4 --csv --log-file gpurun_out/r2u_ncu_stream.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2u_ncu.log 2>&1
