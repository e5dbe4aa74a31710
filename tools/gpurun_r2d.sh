# round 2, run d: the whole GPU suite on 4 GPUs, the probe, the N=8 reference arm
(time timeout 1500 python -m pytest tests -m gpu -q -rs) > gpurun_out/r2d_tests.log 2>&1
timeout 300 python tools/stage_timing_probe.py > gpurun_out/r2d_probe.json 2> gpurun_out/r2d_probe.err
WORLD_SIZE=8 RANK=0 timeout 900 python bench.py --impl reference --gpus 8 --steps 20 --warmup 5 > gpurun_out/r2d_ref8.json 2> gpurun_out/r2d_ref8.err
