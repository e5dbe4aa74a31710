# round 2, run zj: HEAD ncu evidence at N = 1 (BERT-large K = 4 bo_train_step): launch list with DRAM bytes, then one --set full capture of k_lamb_p1r and of k_lamb_p2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_lamb|k_fused' -c 40 --csv --log-file gpurun_out/r2zj_launches_n1.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2zj_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_lamb_p1r|k_lamb_p2' -s 8 -c 2 -o gpurun_out/r2zj_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2zj_ncu_full.log 2>&1
ncu -i gpurun_out/r2zj_full.ncu-rep --page raw --csv > gpurun_out/r2zj_full_raw.csv 2>&1
ncu -i gpurun_out/r2zj_full.ncu-rep --page details --csv > gpurun_out/r2zj_full_details.csv 2>&1
