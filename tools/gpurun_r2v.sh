# round 2, run v: copy-engine push probe (tools/ce_push_bw) at world 2 and 4
nvidia-smi topo -m > gpurun_out/r2v_topo.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 ./tools/ce_push_bw > gpurun_out/r2v_ce_n2.txt 2>&1
timeout 120 ./tools/ce_push_bw > gpurun_out/r2v_ce_n4.txt 2>&1
timeout 120 ./tools/ce_push_bw 25 > gpurun_out/r2v_ce_n4_b25.txt 2>&1
