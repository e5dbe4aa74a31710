# round 2, run zzd: final 1-GPU validation (full -m gpu suite, smoke, default bench) + ncu launch list of the world-4 kernels incl. k_push_posted in the lockstep world (one process)
(time timeout 1800 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2zzd_tests.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/r2zzd_smoke.log 2>&1
(timeout 600 python bench.py) > gpurun_out/r2zzd_bench.json 2> gpurun_out/r2zzd_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_p1w|k_push_posted|k_hopx|k_trust|k_norm_reduce|k_step_final|k_rollback' -c 120 --csv --log-file gpurun_out/r2zzd_launches_world4.csv python bench.py --gpus 4 --steps 2 --warmup 1 > gpurun_out/r2zzd_ncu.log 2>&1
