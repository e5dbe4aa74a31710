# round 2, run zm: bench.py with every stage's ms taken as its share of the event-free step (N = 1 default run, and the lockstep world 4)
timeout 600 python bench.py > gpurun_out/r2zm_bench.json 2> gpurun_out/r2zm_bench.err
timeout 600 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2zm_lockstep4.json 2>> gpurun_out/r2zm_bench.err
