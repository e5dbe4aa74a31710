# round 2, run h: ncu (one use per call): launch list + DRAM bytes of every
# kernel of the N=1 step, and of the N>1 kernels through the lockstep world-4
# emulation on one GPU (one process, no kernel waits on another: ncu-safe).
export CUDA_VISIBLE_DEVICES=0
B1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
B4="python bench.py --gpus 4 --steps 2 --warmup 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
$B1 > gpurun_out/r2h_plain1.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2h_launches_n1.csv $B1 > gpurun_out/r2h_ncu1.log 2>&1
$B4 > gpurun_out/r2h_plain4.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"k_hopx|k_p1w|k_shard_p2|k_norm_reduce|k_trust|k_step_end" -c 60 --csv --log-file gpurun_out/r2h_launches_w4emu.csv $B4 > gpurun_out/r2h_ncu4.log 2>&1
echo done
