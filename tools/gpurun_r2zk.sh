# round 2, run zk: programmatic dependent launch for the one-rank LAMB chain (BO_PDL): parity suites, then A/B bench at N = 1
(timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_ops.py tests/test_gpu_adapter.py tests/test_gpu_trace.py -q -x -rs) > gpurun_out/r2zk_tests.log 2>&1
for i in 1 2 3; do
  for p in 1 0; do
    BO_PDL=$p timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zk_bench_pdl${p}_$i.json 2>> gpurun_out/r2zk_bench.err
  done
done
(timeout 900 python -m pytest tests/test_gpu_config4_full.py -q -x -rs) > gpurun_out/r2zk_config4.log 2>&1
