# round 2, run q: HEAD re-check on one GPU (the driver's round-end tiers): -m gpu suite, smoke, bench N=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2q_gpu.txt 2>&1
(time timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15) > gpurun_out/r2q_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2q_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2q_bench1.json 2> gpurun_out/r2q_bench1.err
