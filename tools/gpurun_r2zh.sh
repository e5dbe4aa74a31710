# round 2, run zh: HEAD validation after the container re-creation: full -m gpu suite, smoke, default bench (N=1), ncu launch list
(time timeout 1500 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zh_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2zh_smoke.log 2>&1
(timeout 600 python bench.py) > gpurun_out/r2zh_bench.json 2> gpurun_out/r2zh_bench.err
