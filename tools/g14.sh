timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/g14_fuzz.log 2>&1
tail -5 gpurun_out/g14_fuzz.log
