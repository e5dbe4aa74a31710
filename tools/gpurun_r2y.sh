# round 2, run y: NVSwitch multicast probe for the parameter all-gather (tools/nvls_probe), 2 and 4 GPUs
CUDA_VISIBLE_DEVICES=0,1 timeout 120 ./tools/nvls_probe > gpurun_out/r2y_nvls_n2.txt 2>&1
timeout 120 ./tools/nvls_probe > gpurun_out/r2y_nvls_n4.txt 2>&1
nvidia-smi -q | grep -i -A3 'fabric' > gpurun_out/r2y_fabric.txt 2>&1
