# round 2, run x: ncu --set full of k_lamb_p1r<4> and k_lamb_p2 (source-level), one bench process
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_lamb_p1r|k_lamb_p2' -s 6 -c 2 -o gpurun_out/r2x_p1r python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2x_ncu.log 2>&1
