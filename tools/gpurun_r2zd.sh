# round 2, run zd: default k_lamb_p1r / k_lamb_p1 L2 prefetch — full -m gpu suite, smoke, bench N=1, ncu launch list
(time timeout 1500 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zd_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2zd_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2zd_bench1.json 2> gpurun_out/r2zd_bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2zd_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2zd_ncu.log 2>&1
