# round 2, run zx: SM-partition probe (few-SM posted-store push concurrent with an HBM stream), 2 and 4 GPUs
(CUDA_VISIBLE_DEVICES=0,1 timeout 300 tools/nvl_partition) > gpurun_out/r2zx_partition_n2.txt 2>&1
(timeout 300 tools/nvl_partition) > gpurun_out/r2zx_partition_n4.txt 2>&1
