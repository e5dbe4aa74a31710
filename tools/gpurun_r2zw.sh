# round 2, run zw: end-of-session validation on 1 B200: full -m gpu suite, smoke, default bench, reference arm
(time timeout 1800 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zw_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2zw_smoke.log 2>&1
(timeout 600 python bench.py) > gpurun_out/r2zw_bench.json 2> gpurun_out/r2zw_bench.err
(timeout 600 python bench.py --impl reference) > gpurun_out/r2zw_ref.json 2>> gpurun_out/r2zw_bench.err
