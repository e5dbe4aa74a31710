# round 2, run zr: BASELINE config 1 as a bench line (BERT-base, K = 1, one worker) and the reference arm on the same config
timeout 600 python bench.py --model bert-base --accumulation 1 > gpurun_out/r2zr_bench_config1.json 2> gpurun_out/r2zr.err
timeout 600 python bench.py --impl reference --model bert-base --accumulation 1 > gpurun_out/r2zr_ref_config1.json 2>> gpurun_out/r2zr.err
