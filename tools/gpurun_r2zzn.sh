# round 2, run zzn: last 1-GPU check of the whole -m gpu suite at HEAD
(time timeout 1200 python -m pytest tests -m gpu -q -rs -x) > gpurun_out/r2zzn_tests.log 2>&1
