# round 2, run zzi: final 1-GPU validation (full -m gpu suite, smoke, default bench)
(time timeout 1800 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zzi_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2zzi_smoke.log 2>&1
(timeout 600 python bench.py) > gpurun_out/r2zzi_bench.json 2> gpurun_out/r2zzi_bench.err
