timeout 1800 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_spec.py -m gpu -q -p no:cacheprovider > gpurun_out/g18.log 2>&1
tail -3 gpurun_out/g18.log
